"""Multi-GPU plumbing of the sequence-parallel decode (BASELINE
config 4), used by bench.py's N > 1 path.

Sequences are independent, so ranks share nothing on the data path: rank r
owns sequences r, r + N, r + 2N, ... (sequence i on GPU i mod N) and decodes
them in lockstep in the same launches (their trees side by side).  The only
collective is one scalar MAX over ranks for timing: the whole-job time is the
slowest rank's.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


def shard_sequences(n_sequences: int, world: int, rank: int) -> list[int]:
    """Sequence ids owned by `rank` (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_sequences < world:
        raise ValueError(f"{n_sequences} sequences cannot cover {world} ranks")
    return list(range(rank, n_sequences, world))


@dataclass(frozen=True)
class RankPlan:
    """What one rank decodes: its sequence ids, how many it batches per launch
    and the seed of its synthetic stream."""

    rank: int
    world: int
    sequences: tuple[int, ...]
    seed: int

    @property
    def per_gpu(self) -> int:
        return len(self.sequences)


def plan_rank(n_sequences: int, world: int, rank: int, base_seed: int = 0) -> RankPlan:
    seqs = shard_sequences(n_sequences, world, rank)
    if len({len(shard_sequences(n_sequences, world, r)) for r in range(world)}) != 1:
        raise ValueError("sequences must divide evenly over the ranks (equal-length lockstep decode)")
    # one stream per rank, seeded by its first sequence id: streams never repeat across ranks
    return RankPlan(rank, world, tuple(seqs), base_seed * 1_000_003 + seqs[0])


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host scalar over all ranks (identity when not distributed).
    NCCL needs a device tensor: pass the rank's CUDA device."""
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: float, world: int, max_seconds: float) -> float:
    """Whole-job units/s: all ranks' units over the slowest rank's time."""
    return units_per_rank * world / max_seconds
