"""Host-side helpers of bench.py that do not touch the GPU (so they can be tested on CPU with the
gloo backend): max-over-ranks timing, whole-job aggregation, and the sample shard of a rank."""
from __future__ import annotations


def max_over_ranks(ms_local: float, dist=None, device=None) -> float:
    """Max of a per-rank duration over all ranks (all_reduce MAX); identity without dist."""
    if dist is None:
        return ms_local
    import torch
    t = torch.tensor([ms_local], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(steps: int, world: int, ms_max: float) -> float:
    """Whole-job throughput: every rank ran `steps` iterations in at most ms_max milliseconds."""
    return steps * world / (ms_max * 1e-3)


def shard(n_units: int, rank: int, world: int):
    """Contiguous, balanced [lo, hi) shard of n_units independent units (e.g. config-4 samples)."""
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)
