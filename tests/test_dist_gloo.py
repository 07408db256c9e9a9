"""N > 1 host logic on CPU: world_size-2 gloo process group (127.0.0.1), no GPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1701_01608_b200 import dist as D


def test_shard_range_covers_disjoint():
    for n in (0, 1, 7, 512, 32768, 110592):
        for size in (1, 2, 3, 8):
            parts = [D.shard_range(n, r, size) for r in range(size)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(size - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)


def test_weak_value_formula():
    # 32^3 cells x 32^3 velocities per rank, 2 ranks, 500 ms slowest rank
    assert D.weak_value(32768, 32768, 2, 500.0) == pytest.approx(32768 * 32768 * 2 / 0.5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=size)
    ws, rk, lr = D.world()
    ms = 100.0 + 50.0 * rank           # rank 1 is the slow one
    mx = D.max_over_ranks(ms)
    a, b = D.shard_range(1001, rk, ws)
    out.put((rk, ws, mx, a, b, D.rank_seed(rk)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_max_and_shards():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2, 2]
    assert all(r[2] == 150.0 for r in res)               # max over ranks seen by every rank
    assert res[0][3:5] == (0, 501) and res[1][3:5] == (501, 1001)
    assert res[0][5] is None and res[1][5] == 1          # rank 0 reproduces the 1-GPU box
