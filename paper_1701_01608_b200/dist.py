"""Host-side plumbing for N > 1 ranks (one process per GPU, torch.distributed).

The collision step shards by cells with no data-path collective (cells are independent): each rank
owns a disjoint cell range (strong split of one batch) or its own box (weak scaling, what bench.py does).
The only collective is the max-over-ranks of the device-measured step time.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous, disjoint, balanced cell range [a, b) of rank `rank` among `size` ranks (covers [0, n))."""
    if size < 1 or not 0 <= rank < size:
        raise ValueError("bad rank/size")
    base, extra = divmod(n, size)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def rank_seed(rank: int) -> int | None:
    """Input seed of a rank's own box under weak scaling (rank 0 reproduces the single-GPU workload)."""
    return None if rank == 0 else rank


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed milliseconds) over all ranks; identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    if dist.get_backend() == "gloo":
        device = None  # host tensor for the CPU backend
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_value(cells_per_rank: int, n_velocity: int, size: int, ms_max: float, steps: int = 1) -> float:
    """Whole-job throughput: cells·velocity-points processed by ALL ranks / slowest rank's time."""
    return cells_per_rank * n_velocity * size * steps / (ms_max / 1e3)


# ---------------------------------------------------------------------------------------------------------------
# Slab decomposition of fks_step in x (the paper's MPI FKS)
#
# Each rank owns the x-planes [x0, x1) of a periodic nx × ny × nz grid (the paper's "subdomains").
# Transport moves particles across the slab boundary; instead of packing and exchanging halo planes, each rank's
# gather kernel reads the source planes it needs directly from the owner's buffer (CUDA IPC mapping, peer loads
# over NVLink): fks_step_slab gets a table of plane pointers covering [x0 − H, x1 + H).  One barrier per step
# orders the ranks (a buffer is overwritten only after every rank finished reading it).
# ---------------------------------------------------------------------------------------------------------------

class SlabDomain:
    """x-slab `rank` of `size` over a periodic nx × ny × nz cell grid (balanced, contiguous, disjoint)."""

    def __init__(self, nx: int, ny: int, nz: int, rank: int, size: int):
        if size > nx:
            raise ValueError("more ranks than x-planes")
        self.nx, self.ny, self.nz, self.rank, self.size = nx, ny, nz, rank, size
        self.x0, self.x1 = shard_range(nx, rank, size)
        self.starts = [shard_range(nx, r, size)[0] for r in range(size)]

    @property
    def nx_local(self) -> int:
        return self.x1 - self.x0

    def owner(self, gx: int) -> tuple[int, int]:
        """(rank, local plane) of global x-plane gx (taken mod nx)."""
        gx %= self.nx
        r = max(i for i, s in enumerate(self.starts) if s <= gx)
        return r, gx - self.starts[r]

    def table_planes(self, H: int) -> list[tuple[int, int]]:
        """(owner rank, local plane) of table entry i = global plane (x0 − H + i) mod nx, i < nx_local + 2H."""
        return [self.owner(self.x0 - H + i) for i in range(self.nx_local + 2 * H)]

    def neighbours(self, H: int) -> list[int]:
        """Ranks whose planes this rank's gather reads (including itself)."""
        return sorted({r for r, _ in self.table_planes(H)})


def interior_planes(nx_local: int, H: int) -> tuple[int, int]:
    """Local destination planes [H, nx_local - H) whose gather reads only this rank's own planes and which no
    neighbour's gather reads ((0, 0) when the slab is too thin): safe to compute before the step's barrier."""
    a, b = H, nx_local - H
    return (a, b) if b > a else (0, 0)


def planes_read_by_others(domain: SlabDomain, H: int) -> set[int]:
    """Local planes of this rank that some other rank's gather table contains (its boundary planes)."""
    out = set()
    for r in range(domain.size):
        if r == domain.rank:
            continue
        other = SlabDomain(domain.nx, domain.ny, domain.nz, r, domain.size)
        out |= {lp for (o, lp) in other.table_planes(H) if o == domain.rank}
    return out


def plane_pointers(domain: SlabDomain, H: int, base_ptrs: list[int], plane_bytes: int) -> list[int]:
    """Device addresses of the table planes, given every rank's buffer base address as mapped in this process."""
    out = []
    for r, lp in domain.table_planes(H):
        if base_ptrs[r] is None:
            raise ValueError(f"plane owned by rank {r} but its buffer is not mapped here")
        out.append(base_ptrs[r] + lp * plane_bytes)
    return out


def share_buffer(t, domain: SlabDomain, H: int, group=None) -> tuple[list, list]:
    """Map the same-named buffer of every rank whose planes this rank reads (CUDA IPC, all_gather of handles).

    Returns (base addresses by rank, keep-alive list).  Without a process group only the local buffer is mapped."""
    import torch
    import torch.distributed as dist
    size = domain.size
    ptrs = [None] * size
    ptrs[domain.rank] = t.data_ptr()
    keep = []
    if size == 1 or not (dist.is_available() and dist.is_initialized()):
        return ptrs, keep
    st = t.untyped_storage()
    handle = st._share_cuda_()
    offset = t.storage_offset() * t.element_size()
    gathered = [None] * size
    dist.all_gather_object(gathered, (handle, offset), group=group)
    for r in domain.neighbours(H):
        if r == domain.rank:
            continue
        h, off = gathered[r]
        peer = torch.UntypedStorage._new_shared_cuda(*h)
        keep.append(peer)
        ptrs[r] = peer.data_ptr() + off
    return ptrs, keep


class SlabStepper:
    """Runs fks_step_slab on this rank's slab with ping-pong buffers (a, b), one barrier per step."""

    def __init__(self, col, domain: SlabDomain, buf_a, buf_b, cfl_num: int, cfl_den: int = 1, barrier=None,
                 ptrs_a=None, ptrs_b=None):
        from . import binding as B
        self.B, self.col, self.domain = B, col, domain
        B.fks_transport_setup_slab(col.h, domain.nx, domain.ny, domain.nz, domain.x0, domain.nx_local, cfl_num,
                                   cfl_den)
        self.H = B.fks_slab_halo(col.h)
        self.bufs = [buf_a, buf_b]
        plane_bytes = domain.ny * domain.nz * buf_a[0].numel() * buf_a.element_size()
        self.keep = []
        if ptrs_a is None:
            ptrs_a, ka = share_buffer(buf_a, domain, self.H)
            ptrs_b, kb = share_buffer(buf_b, domain, self.H)
            self.keep += ka + kb
        self.tables = [plane_pointers(domain, self.H, ptrs_a, plane_bytes),
                       plane_pointers(domain, self.H, ptrs_b, plane_bytes)]
        self.barrier = barrier
        self.i = 0

    def interior(self) -> tuple[int, int]:
        """Local destination planes [H, nx_local - H): their sources are this rank's own planes and no neighbour
        reads them, so they may be computed before the barrier of the step."""
        return interior_planes(self.domain.nx_local, self.H)

    def step(self, coll_scale: float, transport_only: bool = False, overlap: bool = True):
        """Step i reads buffer i % 2 on every rank and writes this rank's buffer (i + 1) % 2.

        overlap: the interior planes are gathered and collided first, then the barrier (every rank finished the
        previous step, so its boundary planes are final and nobody still reads this rank's destination buffer's
        boundary planes), then the boundary planes — the paper's order relaxation -> transport -> communication
        with the exchange hidden behind the interior work.  Bit-identical to the plain step."""
        src, dst = self.i % 2, (self.i + 1) % 2
        a, b = self.interior()
        if transport_only or not overlap or b <= a:
            if self.barrier is not None:
                self.barrier()
            if transport_only:
                self.B.fks_transport_step_slab(self.col.h, self.tables[src], self.bufs[dst])
            else:
                self.B.fks_step_slab(self.col.h, self.tables[src], self.bufs[dst], coll_scale)
        else:
            nx = self.domain.nx_local
            self.B.fks_step_slab_range(self.col.h, self.tables[src], self.bufs[dst], coll_scale, a, b, True)
            if self.barrier is not None:
                self.barrier()
            self.B.fks_step_slab_range(self.col.h, self.tables[src], self.bufs[dst], coll_scale, 0, a, False)
            self.B.fks_step_slab_range(self.col.h, self.tables[src], self.bufs[dst], coll_scale, b, nx, False)
        self.i += 1
        return self.bufs[dst]


def stream_barrier(device):
    """Stream-ordered barrier over the default group: an all-reduce of one element on the current stream (NCCL),
    or a host barrier after a device synchronisation (gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return lambda: None
    if dist.get_backend() == "nccl":
        flag = torch.zeros(1, device=device)
        return lambda: dist.all_reduce(flag)

    def _b():
        torch.cuda.synchronize(device)
        dist.barrier()
    return _b
