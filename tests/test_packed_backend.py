"""run_plan(..., backend="packed"): routing, failure conventions, no CPU fallback.

CPU part (here): without a usable GPU the packed lanes fail LOUDLY (exit 1,
reason on the task's stderr) -- never a silent CPU path; opaque argvs keep the
reference mechanism and succeed; the report keeps the reference schema.
GPU part: real packed runs (see test_gpu_packed_backend.py).
"""

import json
import os
import sys

import pytest

from paper_2410_22254_b200 import NodeSpec, TaskDef, TripleSpec, build_plan, run_plan
from paper_2410_22254_b200.jobspec import JobSpec


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_packed_without_gpu_fails_loudly_and_opaque_tasks_still_run(tmp_path):
    job = lambda i: TaskDef(i, tuple(JobSpec(model="mlp", seed=i, steps=2).argv(sys.executable)))
    tasks = [job(0), TaskDef(1, ("sh", "-c", "echo opaque")), job(2), job(3)]
    plan = build_plan(tasks, TripleSpec(1, 2, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=1024))
    report = run_plan(plan, 0, log_dir=tmp_path, backend="packed")
    st = {r.task_id: r.exit_status for r in report.results}
    # slot 0 = tasks 0, 2 (packable) ; slot 1 = tasks 1 (opaque), 3 -> subprocess slot
    assert st[1] == 0
    assert (tmp_path / "task_1.out").read_text() == "opaque\n"
    assert st[0] == 1 and st[2] == 1
    err = (tmp_path / "task_0.err").read_text()
    assert "tlk error" in err or "CUDA" in err or "libtlk" in err
    assert st[3] != 0  # the job entry point itself refuses to run without a GPU
    d = report.to_json_dict()
    assert d["packed"]["backend"] == "packed" and d["packed"]["subprocess_slots"] == 1
    assert [r["task_id"] for r in d["results"]] == [0, 1, 2, 3]


def test_unknown_backend_rejected():
    plan = build_plan([TaskDef(0, ("true",))], TripleSpec(1, 1, 1), NodeSpec(cores=1))
    with pytest.raises(ValueError):
        run_plan(plan, 0, backend="mps")


def test_packed_needs_gpu_slots_else_reference_mechanism(tmp_path):
    # a CPU-only node: no slot has a GPU pin -> every slot uses the subprocess mechanism
    plan = build_plan([TaskDef(i, ("sh", "-c", f"echo {i}")) for i in range(3)], TripleSpec(1, 2, 1),
                      NodeSpec(cores=4))
    report = run_plan(plan, 0, log_dir=tmp_path, backend="packed")
    assert report.failures == 0
    assert (tmp_path / "task_2.out").read_text() == "2\n"
