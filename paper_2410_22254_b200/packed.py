"""``run_plan_packed``: the packed backend of ``run_plan``.

Same inputs, outputs and failure conventions as the reference's
``run_plan`` (executor.py:162-233).  The node's bindings are grouped by
``gpu_index`` (core.py:147-153); for every GPU g one worker process is
started with the slot env's own device pin (CUDA_VISIBLE_DEVICES=g) and the
slots pinned to g become lanes of that worker's packed runtime.  Slots whose
queue holds any task the packed runtime cannot run (an opaque argv, or a task
whose extra_env overrides the device variable) keep the reference mechanism:
one thread draining the queue with one subprocess per task.

Every task yields exactly one TaskResult with the reference's field meanings:
start/end ms on the run's single monotonic origin (stamped when the worker
reports the lane load/finish), exit status 0 / 1 / 2 / 124, oom_flag from the
same classify_failure on the task's error text.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import threading
from pathlib import Path

from .executor import (
    DEFAULT_OOM_PATTERNS,
    MonotonicClock,
    TaskResult,
    _spawn,
    classify_failure,
    finish_report,
    node_bindings_of,
)
from .jobspec import job_flags_of
from .plan import LaunchPlan

PKG_ROOT = str(Path(__file__).resolve().parent.parent)


def _packable_slot(plan, node_index, binding, device_var) -> bool:
    for task in plan.queue_for(node_index, binding.slot_index):
        if job_flags_of(task.argv) is None:
            return False
        env = dict(task.extra_env)
        if device_var in env and env[device_var] != str(binding.gpu_index):
            return False
    return True


def run_plan_packed(
    plan: LaunchPlan,
    node_index: int = 0,
    *,
    timeout_s: float | None = None,
    log_dir=None,
    oom_patterns=DEFAULT_OOM_PATTERNS,
    base_env: dict | None = None,
    chunk: int = 64,
    python: str | None = None,
):
    mine = node_bindings_of(plan, node_index)
    if log_dir is not None:
        Path(log_dir).mkdir(parents=True, exist_ok=True)
    base = dict(os.environ if base_env is None else base_env)
    device_var = next((k for k, _ in mine[0].env if k == "CUDA_VISIBLE_DEVICES"), None)
    device_var = device_var or "CUDA_VISIBLE_DEVICES"
    results: list[TaskResult] = []
    lock = threading.Lock()
    clock = MonotonicClock()
    stats: dict = {}

    by_gpu: dict[int, list] = {}
    fallback = []
    for b in mine:
        if b.gpu_index is not None and _packable_slot(plan, node_index, b, device_var):
            by_gpu.setdefault(b.gpu_index, []).append(b)
        else:
            fallback.append(b)

    def drain_subprocess(binding):
        """Reference mechanism for slots the packed runtime cannot take."""
        slot_env = {**base, **dict(binding.env)}
        for task in plan.queue_for(node_index, binding.slot_index):
            env = {**slot_env, **dict(task.extra_env)}
            start = clock.now_ms()
            status, tail = _spawn(list(task.argv), env, timeout_s, log_dir, task.task_id)
            end = clock.now_ms()
            oom = status != 0 and classify_failure(status, tail, oom_patterns) == "oom"
            with lock:
                results.append(TaskResult(task.task_id, binding.slot_index, binding.gpu_index,
                                          start, end, status, oom))

    def run_gpu(gpu, bindings):
        env = {**base, **dict(bindings[0].env)}  # the slot env's device pin (same for all)
        env[device_var] = str(gpu)
        env["PYTHONPATH"] = os.pathsep.join(p for p in (PKG_ROOT, env.get("PYTHONPATH")) if p)
        req = {"slots": [{"slot_index": b.slot_index,
                          "tasks": [{"task_id": t.task_id, "argv": list(t.argv)}
                                    for t in plan.queue_for(node_index, b.slot_index)]}
                         for b in bindings],
               "timeout_s": timeout_s, "log_dir": str(log_dir) if log_dir is not None else None,
               "chunk": chunk}
        slot_gpu = {b.slot_index: b.gpu_index for b in bindings}
        starts: dict = {}
        seen_end = set()
        proc = subprocess.Popen([python or sys.executable, "-m", "paper_2410_22254_b200.worker"],
                                stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                env=env, text=True)
        err_lines: list[str] = []
        t_err = threading.Thread(target=lambda: err_lines.extend(proc.stderr), daemon=True)
        t_err.start()
        proc.stdin.write(json.dumps(req))
        proc.stdin.close()
        for line in proc.stdout:
            try:
                ev = json.loads(line)
            except json.JSONDecodeError:
                continue
            now = clock.now_ms()
            if ev.get("ev") == "start":
                starts[ev["task_id"]] = (now, ev["slot_index"])
            elif ev.get("ev") == "end":
                tid = ev["task_id"]
                start, slot = starts.get(tid, (now, None))
                status = int(ev["status"])
                oom = status != 0 and classify_failure(status, ev.get("err", ""), oom_patterns) == "oom"
                with lock:
                    results.append(TaskResult(tid, slot, slot_gpu.get(slot), start, now, status, oom))
                seen_end.add(tid)
            elif ev.get("ev") == "done":
                stats[gpu] = ev.get("stats", {})
        proc.wait()
        t_err.join(timeout=5)
        # a worker that died mid-run: every unfinished task fails loudly
        tail = "".join(err_lines)[-4096:] or f"packed worker exited with {proc.returncode}"
        for b in bindings:
            for t in plan.queue_for(node_index, b.slot_index):
                if t.task_id in seen_end:
                    continue
                now = clock.now_ms()
                start = starts.get(t.task_id, (now, None))[0]
                if log_dir is not None:
                    Path(log_dir, f"task_{t.task_id}.err").write_text(tail + "\n")
                oom = classify_failure(1, tail, oom_patterns) == "oom"
                with lock:
                    results.append(TaskResult(t.task_id, b.slot_index, b.gpu_index, start, now, 1, oom))

    threads = [threading.Thread(target=run_gpu, args=(g, bs), name=f"gpu-{g}") for g, bs in by_gpu.items()]
    threads += [threading.Thread(target=drain_subprocess, args=(b,), name=f"slot-{b.slot_index}")
                for b in fallback]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    elapsed = clock.now_ms()
    extra = {"backend": "packed", "gpus": {str(g): stats.get(g, {}) for g in by_gpu},
             "packed_slots": sum(len(v) for v in by_gpu.values()), "subprocess_slots": len(fallback)}
    return finish_report(plan, node_index, results, elapsed, extra)
