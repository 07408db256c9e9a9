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


# ---------------- slab decomposition of fks_step (NEXT-2): host logic --------------------------------------

@pytest.mark.parametrize("nx,size,H", [(8, 2, 1), (10, 3, 2), (5, 5, 3), (32, 4, 2), (7, 1, 2)])
def test_slab_domain_tables(nx, size, H):
    doms = [D.SlabDomain(nx, 3, 2, r, size) for r in range(size)]
    # the slabs tile the periodic x axis
    owned = sorted(x for d in doms for x in range(d.x0, d.x1))
    assert owned == list(range(nx))
    for d in doms:
        tp = d.table_planes(H)
        assert len(tp) == d.nx_local + 2 * H
        for i, (r, lp) in enumerate(tp):
            gx = (d.x0 - H + i) % nx                      # table entry i is global plane (x0 - H + i) mod nx
            assert doms[r].x0 <= gx < doms[r].x1 and lp == gx - doms[r].x0
        # the interior entries are the rank's own planes, in order
        assert tp[H:H + d.nx_local] == [(d.rank, i) for i in range(d.nx_local)]
        assert d.rank in d.neighbours(H)
    with pytest.raises(ValueError):
        D.SlabDomain(3, 1, 1, 0, 4)


def test_plane_pointers_arithmetic():
    d = D.SlabDomain(10, 2, 2, 1, 3)  # x-planes [4, 7)
    pb = 4 * 2 * 2 * 8
    ptrs = D.plane_pointers(d, 2, [10_000, 20_000, 30_000], pb)
    # planes 2, 3 of rank 0 (x = 2, 3), own 0..2, rank 2's planes 0, 1 (x = 7, 8)
    assert ptrs == [10_000 + 2 * pb, 10_000 + 3 * pb, 20_000, 20_000 + pb, 20_000 + 2 * pb, 30_000, 30_000 + pb]
    with pytest.raises(ValueError):
        D.plane_pointers(d, 2, [None, 20_000, 30_000], pb)


def _slab_worker(rank, size, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=size)
    d = D.SlabDomain(9, 2, 3, rank, size)
    H = 2
    # every rank publishes a fake base address of its buffer, as share_buffer does with IPC handles
    bases = [None] * size
    dist.all_gather_object(bases, 1_000_000 * (rank + 1))
    plane_bytes = 2 * 3 * 8 * 8
    ptrs = D.plane_pointers(d, H, bases, plane_bytes)
    # each table entry must point into the owner's buffer at its local plane
    ok = all(p == 1_000_000 * (r + 1) + lp * plane_bytes for p, (r, lp) in zip(ptrs, d.table_planes(H)))
    out.put((rank, d.x0, d.x1, ok, d.neighbours(H)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_slab_tables():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 5), (5, 9)]
    assert all(r[3] for r in res)
    assert res[0][4] == [0, 1] and res[1][4] == [0, 1]


@pytest.mark.parametrize("nx,size,H", [(64, 2, 2), (96, 3, 2), (256, 8, 2), (40, 4, 3), (12, 4, 2), (8, 2, 5)])
def test_interior_planes_never_read_by_neighbours(nx, size, H):
    """The overlapped slab step computes [H, nx_local - H) before the barrier: those planes must be read by no
    other rank (their sources are this rank's own planes: every table entry within H of a destination plane)."""
    for r in range(size):
        d = D.SlabDomain(nx, 2, 3, r, size)
        a, b = D.interior_planes(d.nx_local, H)
        read = D.planes_read_by_others(d, H)
        assert not (set(range(a, b)) & read), (r, a, b, sorted(read))
        for lx in range(a, b):  # sources of an interior plane are own planes
            for dx in range(-H, H + 1):
                assert 0 <= lx - dx < d.nx_local
        if d.nx_local > 2 * H and size > 1:
            assert read == set(range(0, min(H, d.nx_local))) | set(range(max(0, d.nx_local - H), d.nx_local))
