"""Slab-decomposed fks_step (the paper's MPI FKS) on one GPU.

The gather of each slab reads its neighbours' planes through a pointer table.  (1) Ranks emulated in one process
(tables point into the other slabs' tensors); (2) two real processes sharing buffers through CUDA IPC with a
host barrier per step (one GPU: a correctness test of the peer-pointer path, not a performance claim).  Both
must equal the single-domain fks_transport_step / fks_step bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1701_01608_b200 import binding as B
from paper_1701_01608_b200 import dist as D
from paper_1701_01608_b200 import inputs
from paper_1701_01608_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def _reference(cfg, shape, cfl, f, steps, transport_only):
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    col.transport_setup(shape, *cfl)
    a, b = f.clone(), torch.empty_like(f)
    outs = []
    for _ in range(steps):
        if transport_only:
            col.transport_step(a, b)
        else:
            col.step(a, b, cfg.coll_scale)
        outs.append(b.clone())
        a, b = b, a
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("name,shape,cfl,size", [("c0", (6, 2, 2), (3, 2), 2), ("c0", (7, 1, 2), (3, 2), 3),
                                                 ("c0", (5, 2, 1), (1, 1), 5), ("c2", (4, 2, 1), (1, 1), 2),
                                                 ("c0", (12, 1, 2), (1, 1), 2), ("c2", (10, 1, 1), (1, 1), 2)])
@pytest.mark.parametrize("transport_only", [True, False])
def test_slab_emulated_ranks_bit_exact(cuda_device, name, shape, cfl, size, transport_only):
    """The last two shapes have interior planes (nx_local > 2H): the overlapped step (interior planes before the
    barrier, boundary planes after, fks_step_slab_range) must give the same bits as the single-domain step."""
    cfg = CONFIGS[name]
    nx, ny, nz = shape
    n = nx * ny * nz
    f = inputs.make_f(cfg, device=cuda_device, cells=[c % cfg.n_cells for c in range(n)])
    steps = 3
    ref = _reference(cfg, shape, cfl, f, steps, transport_only)
    per = ny * nz
    doms = [D.SlabDomain(nx, ny, nz, r, size) for r in range(size)]
    bufs_a = [f[d.x0 * per:d.x1 * per].clone() for d in doms]
    bufs_b = [torch.empty_like(x) for x in bufs_a]
    cols = [B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel) for _ in doms]
    steppers = [D.SlabStepper(cols[r], doms[r], bufs_a[r], bufs_b[r], *cfl,
                              ptrs_a=[x.data_ptr() for x in bufs_a], ptrs_b=[x.data_ptr() for x in bufs_b])
                for r in range(size)]
    for s in range(steps):
        outs = [st.step(cfg.coll_scale, transport_only=transport_only) for st in steppers]  # same stream: ordered
        got = torch.cat(outs)
        torch.cuda.synchronize()
        assert torch.equal(got, ref[s]), (s, (got - ref[s]).abs().max().item())


def test_slab_range_checks_and_split(cuda_device):
    """fks_step_slab_range: a step must start with advance = 1; ranges are checked; splitting a step into
    interior-then-boundary ranges equals fks_step_slab bit for bit (one rank owning the whole periodic box)."""
    cfg = CONFIGS["c0"]
    nx, ny, nz = 8, 1, 2
    f = inputs.make_f(cfg, device=cuda_device, cells=[c % cfg.n_cells for c in range(nx * ny * nz)])
    outs = []
    for split in (False, True):
        col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
        B.fks_transport_setup_slab(col.h, nx, ny, nz, 0, nx, 1, 1)
        H = B.fks_slab_halo(col.h)
        table = [f[((x % nx) * ny * nz):((x % nx) + 1) * ny * nz].data_ptr() for x in range(-H, nx + H)]
        g = torch.empty_like(f)
        if not split:
            B.fks_step_slab(col.h, table, g, cfg.coll_scale)
        else:
            with pytest.raises(B.FksError) as ei:
                B.fks_step_slab_range(col.h, table, g, cfg.coll_scale, 0, 2, False)
            assert ei.value.status == B.FKS_ERR_STATE
            with pytest.raises(B.FksError) as ei:
                B.fks_step_slab_range(col.h, table, g, cfg.coll_scale, 3, nx + 1, True)
            assert ei.value.status == B.FKS_ERR_INVALID
            B.fks_step_slab_range(col.h, table, g, cfg.coll_scale, H, nx - H, True)
            B.fks_step_slab_range(col.h, table, g, cfg.coll_scale, 0, H, False)
            B.fks_step_slab_range(col.h, table, g, cfg.coll_scale, nx - H, nx, False)
        torch.cuda.synchronize()
        outs.append(g)
    assert torch.equal(outs[0], outs[1])


def test_slab_argument_checks(cuda_device):
    cfg = CONFIGS["c0"]
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    with pytest.raises(B.FksError):
        B.fks_transport_setup_slab(col.h, 4, 1, 1, 3, 2, 1, 1)  # x0 + nx_local > nx_global
    B.fks_transport_setup_slab(col.h, 4, 1, 1, 1, 2, 1, 1)
    H = B.fks_slab_halo(col.h)
    assert H == 2
    f = torch.zeros(2, cfg.N, cfg.N, cfg.N, dtype=torch.float64, device=cuda_device)
    g = torch.zeros_like(f)
    with pytest.raises(B.FksError):  # the single-domain calls are refused on a slab handle
        col.step(f, g, 0.01)
    with pytest.raises(B.FksError):  # a source plane overlapping f_out
        B.fks_transport_step_slab(col.h, [g.data_ptr()] * (2 + 2 * H), g)
    col.transport_setup((2, 1, 1), 1, 1)  # back to a single domain
    col.step(f, g, 0.01)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, size, port, shape, cfl, steps, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size))
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=size)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = CONFIGS["c0"]
    nx, ny, nz = shape
    d = D.SlabDomain(nx, ny, nz, rank, size)
    cells = [c % cfg.n_cells for c in range(d.x0 * ny * nz, d.x1 * ny * nz)]
    a = inputs.make_f(cfg, device=dev, cells=cells)
    b = torch.empty_like(a)
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    st = D.SlabStepper(col, d, a, b, *cfl, barrier=D.stream_barrier(dev))  # CUDA IPC mapping of a, b
    outs = []
    for _ in range(steps):
        outs.append(st.step(cfg.coll_scale).cpu().numpy())
    torch.cuda.synchronize()
    dist.barrier()  # keep the buffers alive until every rank has read them
    q.put((rank, outs))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_two_processes_cuda_ipc(cuda_device):
    shape, cfl, steps, size = (6, 2, 1), (3, 2), 2, 2
    cfg = CONFIGS["c0"]
    n = shape[0] * shape[1] * shape[2]
    f = inputs.make_f(cfg, device=cuda_device, cells=[c % cfg.n_cells for c in range(n)])
    ref = [r.cpu().numpy() for r in _reference(cfg, shape, cfl, f, steps, False)]
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, size, port, shape, cfl, steps, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for s in range(steps):
        got = np.concatenate([res[r][s] for r in range(size)])
        assert np.array_equal(got, ref[s]), s
