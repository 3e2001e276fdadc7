"""N>1 path on CPU: world_size-2 gloo processes run the bench's rank logic.

Each rank takes the slots the reference mapping pins to "its" GPU, the shares
partition the workload exactly (no task on two ranks, none dropped), the
timing is a MAX over ranks, and per-rank results gather on rank 0.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2410_22254_b200 import TaskDef
from paper_2410_22254_b200.jobspec import JobSpec
from paper_2410_22254_b200.multigpu import gather_results, max_over_ranks, rank_share, weak_scaling_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = weak_scaling_plan(8, world, lambda i: TaskDef(i, tuple(JobSpec(model="cnn", seed=i).argv())))
    share = rank_share(plan, rank)
    ids = [t.task_id for _, ts in share for t in ts]
    elapsed = max_over_ranks(1.5 + rank)
    allids = gather_results(ids)
    if rank == 0:
        q.put((allids, elapsed, [si for si, _ in share]))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_partition_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allids, elapsed, slots0 = q.get()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert elapsed == 2.5
    assert sorted(allids[0] + allids[1]) == list(range(16))
    assert not set(allids[0]) & set(allids[1])
    # reference mapping: slot s -> GPU s % 2, task i -> slot i
    assert slots0 == [0, 2, 4, 6, 8, 10, 12, 14]
    assert allids[1] == [1, 3, 5, 7, 9, 11, 13, 15]
