"""World-size-2 gloo run of the sequence-parallel plumbing on CPU: each rank
owns a disjoint set of sequences, the timing reduction is a MAX over ranks,
and the aggregate throughput counts every rank's tokens (bench.py's N>1 path)."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_10539_b200.dist import aggregate_throughput, max_over_ranks, plan_rank
    plan = plan_rank(64, world, rank, base_seed=3)     # what bench.py's rank decodes (C4: 64 sequences)
    mine = list(plan.sequences)
    seconds = 1.0 + rank          # rank 1 is the slow one
    tmax = max_over_ranks(seconds)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, plan.seed, plan.per_gpu))
    if rank == 0:
        out.put((tmax, aggregate_throughput(plan.per_gpu, world, tmax), gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sequence_parallel():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, thr, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    assert thr == 32 * 2 / 2.0
    (s0, seed0, n0), (s1, seed1, n1) = gathered
    assert sorted(s0 + s1) == list(range(64)) and not set(s0) & set(s1)
    assert n0 == n1 == 32 and seed0 != seed1


def test_uneven_sequence_split_is_rejected():
    import pytest
    from paper_2604_10539_b200.dist import plan_rank
    with pytest.raises(ValueError):
        plan_rank(63, 2, 0)
    with pytest.raises(ValueError):
        plan_rank(1, 2, 0)
