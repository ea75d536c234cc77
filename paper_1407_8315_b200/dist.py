"""Multi-GPU: signals shard across ranks, no data-path collective.

Signals are independent: rank r solves signals [lo_r, hi_r) of
a batch on its own GPU; the only communication is control-plane (timing max,
optional gather of host results to rank 0).  One process per GPU, launched by
torchrun; NCCL for the CUDA ranks, gloo works for the host-side helpers.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(total: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of `total` signals for `rank`."""
    if size < 1 or not 0 <= rank < size:
        raise ValueError(f"bad rank {rank} of {size}")
    base, extra = divmod(total, size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    rank, size = world()
    if size == 1:
        return float(value)
    backend = dist.get_backend()
    dev = device if (device is not None and backend == "nccl") else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(obj, root: int = 0):
    """Gather one picklable object per rank to `root` (list on root, None
    elsewhere) -- e.g. each rank's host spectra after a sharded solve."""
    rank, size = world()
    if size == 1:
        return [obj]
    out = [None] * size if rank == root else None
    dist.gather_object(obj, out, dst=root)
    return out


def solve_sharded(X, cfg, solve, device=None):
    """Solve this rank's shard of the (B, n) host batch X with `solve`
    (e.g. paper_1407_8315_b200.solve_noniterative_batch) and gather the
    shard's spectra to rank 0 (ordered by signal index)."""
    rank, size = world()
    lo, hi = shard(X.shape[0], rank, size)
    res = solve(X[lo:hi], cfg, device=device) if hi > lo else None
    mine = (lo, [] if res is None else [s.entries for s in res.spectra()])
    parts = gather_to_root(mine)
    if parts is None:
        return None
    out = []
    for _, entries in sorted(parts, key=lambda p: p[0]):
        out.extend(entries)
    return out
