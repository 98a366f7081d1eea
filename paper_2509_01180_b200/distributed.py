"""Multi-GPU host logic: one process per GPU, particles sharded in contiguous
blocks, no data-path collective during alignment; the coefficient-space
average numerator is combined with one allreduce (NCCL on GPUs, gloo in the
CPU tests).  SURVEY.md §8(e)."""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [begin, end) of particles owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def allreduce_average(partial_sum, local_count: int, group=None):
    """Sum the per-rank numerators (complex coefficients as (..., 2) real) and the
    particle counts across ranks; returns (average, total_count).  With a single
    process this is the local average."""
    import torch
    import torch.distributed as dist

    count = torch.tensor([float(local_count)], dtype=torch.float64, device=partial_sum.device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(partial_sum, group=group)
        dist.all_reduce(count, group=group)
    total = int(round(count.item()))
    if total == 0:
        raise ArithmeticError("average of zero particles")
    return partial_sum / total, total
