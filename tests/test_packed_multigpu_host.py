"""Host logic of run_plan(..., backend="packed") across GPUs, without a GPU.

A fake worker stands in for ``python -m paper_2410_22254_b200.worker`` (the
``python=`` hook of run_plan_packed), like the reference's probe children
(test_executor.py:121-132): it reports the device pin it was started with and
plays the worker's event protocol.  Checks:
* one worker per GPU, each started with CUDA_VISIBLE_DEVICES=g (the slot env's
  own pin, core.py:171-179) and given exactly the slots pinned to g;
* TaskResults gathered from all workers, in the reference schema;
* the parent watchdog: a worker that hangs past the task timeout is killed,
  the hung task reports 124 (executor.py:20,116-120) and a fresh worker runs
  the rest of the queues.
"""

import json
import os
import sys

from paper_2410_22254_b200 import NodeSpec, TaskDef, TripleSpec, build_plan, run_plan
from paper_2410_22254_b200.jobspec import JobSpec

FAKE = r'''
import json, os, sys, time
req = json.loads(sys.stdin.read())
out = os.environ["FAKE_OUT"]
with open(os.path.join(out, "worker_%s_%d.json" % (os.environ.get("CUDA_VISIBLE_DEVICES"), os.getpid())), "w") as f:
    json.dump({"dev": os.environ.get("CUDA_VISIBLE_DEVICES"), "argv": sys.argv[1:],
               "slots": [s["slot_index"] for s in req["slots"]], "req": req}, f)
def emit(o):
    sys.stdout.write(json.dumps(o) + "\n"); sys.stdout.flush()
for s in req["slots"]:
    for t in s["tasks"]:
        emit({"ev": "start", "task_id": t["task_id"], "slot_index": s["slot_index"]})
        if "666" in t["argv"]:
            time.sleep(1000)
        emit({"ev": "end", "task_id": t["task_id"], "status": 0, "err": "", "summary": {}})
emit({"ev": "done", "stats": {"dev": os.environ.get("CUDA_VISIBLE_DEVICES")}})
'''


def _fake(tmp_path):
    path = tmp_path / "fakepython"
    path.write_text(f"#!{sys.executable}\n" + FAKE)
    path.chmod(0o755)
    return str(path)


def _job(i, seed=None):
    return TaskDef(i, tuple(JobSpec(model="cnn", seed=i if seed is None else seed, steps=5).argv("python3")))


def test_one_worker_per_gpu_with_its_own_pin(tmp_path, monkeypatch):
    out = tmp_path / "out"
    out.mkdir()
    monkeypatch.setenv("FAKE_OUT", str(out))
    tasks = [_job(i) for i in range(12)]
    plan = build_plan(tasks, TripleSpec(1, 4, 1), NodeSpec(cores=8, gpus=2, gpu_mem_mib=1024))
    report = run_plan(plan, 0, backend="packed", packed_options={"python": _fake(tmp_path)})
    workers = [json.loads(p.read_text()) for p in out.iterdir()]
    assert sorted(w["dev"] for w in workers) == ["0", "1"]
    for w in workers:
        assert w["argv"] == ["-m", "paper_2410_22254_b200.worker"]
        # slots s with s % 2 == gpu (assign_gpu, core.py:147-153)
        assert w["slots"] == [s for s in range(4) if s % 2 == int(w["dev"])]
        for s in w["req"]["slots"]:
            assert [t["task_id"] for t in s["tasks"]] == [t.task_id for t in plan.queue_for(0, s["slot_index"])]
    assert [r.task_id for r in report.results] == list(range(12))
    for r in report.results:
        assert r.exit_status == 0 and r.gpu_index == r.slot_index % 2 and r.slot_index == r.task_id % 4
    d = report.to_json_dict()
    assert d["packed"]["packed_slots"] == 4 and set(d["packed"]["gpus"]) == {"0", "1"}
    assert report.max_observed_concurrency <= 4


def test_watchdog_kills_a_hung_worker_and_the_queue_continues(tmp_path, monkeypatch):
    out = tmp_path / "out"
    out.mkdir()
    monkeypatch.setenv("FAKE_OUT", str(out))
    tasks = [_job(0, seed=666), _job(1), _job(2)]  # slot 0: [0 (hangs), 2]; slot 1: [1]
    plan = build_plan(tasks, TripleSpec(1, 2, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=1024))
    report = run_plan(plan, 0, timeout_s=0.5, log_dir=tmp_path / "logs", backend="packed",
                      packed_options={"python": _fake(tmp_path), "watchdog_grace_s": 0.5})
    st = {r.task_id: r.exit_status for r in report.results}
    assert st[0] == 124
    assert st[2] == 0  # the rest of slot 0's queue ran in a fresh worker
    assert "timeout" in (tmp_path / "logs" / "task_0.err").read_text()
    assert len(list(out.iterdir())) >= 2  # the hung worker was replaced
