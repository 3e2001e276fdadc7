"""Multi-GPU plumbing for packed runs: one process per GPU, no data-path collective.

Jobs are independent, so N GPUs partition the task list by the
reference mapping -- task i -> slot i % S (plan.py:121-123) -> GPU
slot % gpus (core.py:147-153) -- and each rank trains its share as one pack.
The only collectives are host-side: a MAX over ranks of the timed region and
a gather of per-task results (torch.distributed; NCCL on GPUs, gloo on CPU).
"""

from __future__ import annotations

from .core import NodeSpec, TripleSpec
from .plan import LaunchPlan, build_plan


def rank_share(plan: LaunchPlan, rank: int, node_index: int = 0):
    """[(slot_index, [TaskDef, ...])] of the slots pinned to GPU ``rank``."""
    return [(b.slot_index, list(plan.queue_for(node_index, b.slot_index)))
            for b in plan.bindings if b.node_index == node_index and b.gpu_index == rank]


def weak_scaling_plan(tasks_per_gpu: int, world: int, make_task, cores: int = 4096,
                      ntpp: int = 1) -> LaunchPlan:
    """The triples [1, tasks_per_gpu * world, ntpp] plan on a ``world``-GPU node."""
    total = tasks_per_gpu * world
    tasks = [make_task(i) for i in range(total)]
    return build_plan(tasks, TripleSpec(1, total, ntpp),
                      NodeSpec(cores=cores, gpus=world, gpu_mem_mib=183359))


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(obj):
    """All ranks' picklable result objects, in rank order (rank 0 uses them)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
