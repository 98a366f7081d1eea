"""Multi-GPU host logic: one process per GPU, particles either sharded in
contiguous blocks or handed out in chunks from a shared counter (dynamic
assignment: per-particle work varies with the fine-window count and the Newton
iterations), no data-path collective during alignment; the coefficient-space
average numerator is combined with one allreduce (NCCL on GPUs, gloo in the
CPU tests).  SURVEY.md §8(e).  The one-process, thread-per-GPU variant with
ncclCommInitAll is MultiDeviceAligner in include/ballmatch_b200.hpp."""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [begin, end) of particles owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


class ChunkScheduler:
    """Dynamic chunk assignment across ranks: every rank pulls the next chunk
    [begin, end) of n_total particles from an atomic counter in the process
    group's key-value store (store.add), until none is left.  Each chunk goes to
    exactly one rank.  `key` names the work queue (one per batch)."""

    def __init__(self, n_total: int, chunk: int, key: str = "bm_chunks", store=None):
        if chunk < 1 or n_total < 0:
            raise ValueError("bad chunk / total")
        self.n_total, self.chunk, self.key = n_total, chunk, key
        if store is None:
            import torch.distributed as dist
            store = dist.distributed_c10d._get_default_store() if dist.is_initialized() else None
        self.store = store
        self._local = 0  # single-process fallback counter

    def next(self):
        if self.store is None:
            begin = self._local
            self._local += self.chunk
        else:
            begin = int(self.store.add(self.key, self.chunk)) - self.chunk
        if begin >= self.n_total:
            return None
        return begin, min(begin + self.chunk, self.n_total)

    def __iter__(self):
        while True:
            span = self.next()
            if span is None:
                return
            yield span


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
