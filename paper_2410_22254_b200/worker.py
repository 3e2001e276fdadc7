"""Per-GPU packed worker: ``python -m paper_2410_22254_b200.worker`` (internal).

Started by ``run_plan_packed`` once per GPU with the reference's own device
pin in its environment (CUDA_VISIBLE_DEVICES=<gpu>, core.py:171-179), so it
sees exactly one device.  Reads one JSON request on stdin:

    {"slots": [{"slot_index": s, "tasks": [{"task_id": i, "argv": [...]}, ...]}, ...],
     "timeout_s": float|null, "log_dir": str|null, "chunk": int, "mem_limit_mib": int|null}

and streams JSON lines on stdout: {"ev": "start", "task_id": i} when a task
is loaded into its lane, {"ev": "end", "task_id": i, "status": st, "err": e}
when it finishes, and a final {"ev": "done", "stats": {...}}.  The parent
stamps events with its own monotonic clock (one origin for all TaskResults,
executor.py:187-190).  Task logs are task_<id>.out/.err like the reference's.
"""

from __future__ import annotations

import json
import os
import sys

from .jobspec import parse_task
from .scheduler import LaneScheduler, SlotTask, TlkBackend


def _emit(obj):
    sys.stdout.write(json.dumps(obj) + "\n")
    sys.stdout.flush()


def _tasks(raw):
    out = []
    for t in raw:
        try:
            spec = parse_task(t["argv"])
            err = None if spec is not None else "not a packable job argv"
        except ValueError as exc:
            spec, err = None, f"usage error: {exc}"
        out.append(SlotTask(int(t["task_id"]), spec, err))
    return out


def main() -> int:
    req = json.loads(sys.stdin.read())
    log_dir = req.get("log_dir")
    if log_dir:
        os.makedirs(log_dir, exist_ok=True)

    def on_start(task_id, slot_index):
        _emit({"ev": "start", "task_id": task_id, "slot_index": slot_index})

    def on_end(o):
        if log_dir:
            with open(os.path.join(log_dir, f"task_{o.task_id}.out"), "w") as f:
                if o.summary:
                    f.write(json.dumps(o.summary) + "\n")
            with open(os.path.join(log_dir, f"task_{o.task_id}.err"), "w") as f:
                if o.err:
                    f.write(o.err + "\n")
        _emit({"ev": "end", "task_id": o.task_id, "status": o.status, "err": o.err[-4096:],
               "summary": o.summary})

    slots = [(int(s["slot_index"]), _tasks(s["tasks"])) for s in req["slots"]]
    try:
        mib = req.get("mem_limit_mib")
        backend = TlkBackend(0, int(mib) << 20 if mib else None)
    except Exception as exc:
        # no usable device/library: every task fails loudly (no CPU fallback)
        for si, tasks in slots:
            for t in tasks:
                on_start(t.task_id, si)
                from .scheduler import TaskOutcome

                on_end(TaskOutcome(t.task_id, si, 1, f"{type(exc).__name__}: {exc}"))
        _emit({"ev": "done", "stats": {"error": str(exc)}})
        return 1
    sched = LaneScheduler(backend, slots, timeout_s=req.get("timeout_s"),
                          chunk=int(req.get("chunk", 64)), on_start=on_start, on_end=on_end)
    sched.run()
    _emit({"ev": "done", "stats": sched.stats()})
    backend.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
