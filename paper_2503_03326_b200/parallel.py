"""Multi-rank plumbing (one process per GPU, torch.distributed): sharding of
independent units and device-time max over ranks. The hot path itself has no
collective except the config-5 tile all-to-all (slab.exchange)."""
from __future__ import annotations


def shard_range(units: int, rank: int, world: int):
    """Contiguous share of `units` independent units (instances) for `rank`."""
    per, extra = divmod(units, world)
    lo = rank * per + min(rank, extra)
    return lo, lo + per + (1 if rank < extra else 0)


def max_over_ranks(x: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return x
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
