"""Multi-GPU plumbing for the sequence-parallel decode.

Sequences are independent, so ranks share nothing on the data path: rank r
owns sequences r, r + N, r + 2N, ...  The only collective is a single scalar
MAX over ranks for timing (the whole-job time is the slowest rank's).
"""

from __future__ import annotations

import torch


def shard_sequences(n_sequences: int, world: int, rank: int) -> list[int]:
    """Sequence ids owned by `rank` (round-robin, C4: sequence i on GPU i mod N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_sequences, world))


def max_over_ranks(value: float) -> float:
    """Max of a host scalar over all ranks (identity when not distributed)."""
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: int, world: int, max_seconds: float) -> float:
    """Whole-job units/s: all ranks' units over the slowest rank's time."""
    return units_per_rank * world / max_seconds
