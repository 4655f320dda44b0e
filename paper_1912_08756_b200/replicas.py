"""Query replicas over several GPUs: the in-order
heap loop of a query cannot be split over database shards, and queries are
independent, so every rank holds a full index replica and takes its own
query batches.  No data-path collective; the only exchange is the reduction
of the timings (max over ranks) and of the query counts (sum) for the
whole-job throughput.  Host logic only: used by bench.py under torchrun
(NCCL) and tested on CPU with gloo, world_size 2 (tests/test_replicas.py)."""

from __future__ import annotations


def rank_batch(rank: int, world: int, step: int, nbatches: int) -> int:
    """Index of the query batch rank `rank` runs at step `step`: the ranks of
    one step take `world` consecutive batches (round robin over the set)."""
    if not (0 <= rank < world) or nbatches < 1:
        raise ValueError(f"rank {rank} of {world}, {nbatches} batches")
    return (rank + step * world) % nbatches


def aggregate(dist, device, nq: int, times):
    """Whole-job figures from per-rank ones: (total queries, [max over ranks
    of each time]).  `dist` is torch.distributed (initialised) or None for a
    single process."""
    if dist is None:
        return int(nq), [float(t) for t in times]
    import torch

    tt = torch.tensor([float(t) for t in times], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    nn = torch.tensor([float(nq)], dtype=torch.float64, device=device)
    dist.all_reduce(nn, op=dist.ReduceOp.SUM)
    return int(nn.item()), tt.tolist()
