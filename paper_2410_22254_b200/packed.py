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
import queue
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
from .scheduler import TIMEOUT_EXIT_STATUS

WATCHDOG_GRACE_S = 30.0  # worker-side timeout handling gets this long before the kill
MAX_WORKER_RESTARTS = 8
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
    mem_limit_mib: int | None = None,
    watchdog_grace_s: float = None,
):
    """``mem_limit_mib``: admit packed tasks against this much device memory per
    GPU (e.g. the plan's NodeSpec.gpu_mem_mib, as the reference simulator does,
    sim.py:388-402); default: the device's own memory."""
    grace = WATCHDOG_GRACE_S if watchdog_grace_s is None else float(watchdog_grace_s)
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
        """One packed worker per GPU, watched by a deadline.  If the worker
        hangs past the longest per-task timeout (+ grace), it is killed, its
        running tasks get 124 (the reference's timeout status) and a fresh
        worker takes over the rest of every slot's queue."""
        env = {**base, **dict(bindings[0].env)}  # the slot env's device pin (same for all)
        env[device_var] = str(gpu)
        env["PYTHONPATH"] = os.pathsep.join(p for p in (PKG_ROOT, env.get("PYTHONPATH")) if p)
        slot_gpu = {b.slot_index: b.gpu_index for b in bindings}
        pending = {b.slot_index: list(plan.queue_for(node_index, b.slot_index)) for b in bindings}
        starts: dict = {}
        seen_end: set = set()
        restarts = 0

        def record(tid, slot, start, end, status, err):
            oom = status != 0 and classify_failure(status, err, oom_patterns) == "oom"
            if log_dir is not None and err and status != 0:
                Path(log_dir, f"task_{tid}.err").write_text(err + "\n")
            with lock:
                results.append(TaskResult(tid, slot, slot_gpu.get(slot), start, end, status, oom))
            seen_end.add(tid)

        while any(t.task_id not in seen_end for ts in pending.values() for t in ts):
            req = {"slots": [{"slot_index": si,
                              "tasks": [{"task_id": t.task_id, "argv": list(t.argv)}
                                        for t in ts if t.task_id not in seen_end]}
                             for si, ts in pending.items()],
                   "timeout_s": timeout_s, "log_dir": str(log_dir) if log_dir is not None else None,
                   "chunk": chunk, "mem_limit_mib": mem_limit_mib}
            proc = subprocess.Popen([python or sys.executable, "-m", "paper_2410_22254_b200.worker"],
                                    stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                    env=env, text=True)
            err_lines: list[str] = []
            t_err = threading.Thread(target=lambda: err_lines.extend(proc.stderr), daemon=True)
            t_err.start()
            events: queue.Queue = queue.Queue()

            def pump():
                for ln in proc.stdout:
                    events.put(ln)
                events.put(None)

            threading.Thread(target=pump, daemon=True).start()
            proc.stdin.write(json.dumps(req))
            proc.stdin.close()
            running: dict = {}  # task_id -> slot of tasks started, not ended (this worker)
            killed = False
            while True:
                try:
                    line = events.get(timeout=1.0)
                except queue.Empty:
                    line = ""
                if line is None:
                    break
                now = clock.now_ms()
                if line:
                    try:
                        ev = json.loads(line)
                    except json.JSONDecodeError:
                        ev = {}
                    if ev.get("ev") == "start":
                        starts[ev["task_id"]] = (now, ev["slot_index"])
                        running[ev["task_id"]] = ev["slot_index"]
                    elif ev.get("ev") == "end":
                        tid = ev["task_id"]
                        start, slot = starts.get(tid, (now, None))
                        running.pop(tid, None)
                        record(tid, slot, start, now, int(ev["status"]), ev.get("err", ""))
                    elif ev.get("ev") == "done":
                        stats[gpu] = ev.get("stats", {})
                if timeout_s is not None and running:
                    oldest = min(starts[t][0] for t in running)
                    if now - oldest > 1000.0 * (timeout_s + grace):
                        proc.kill()
                        killed = True
                        for tid, slot in list(running.items()):
                            record(tid, slot, starts[tid][0], now, TIMEOUT_EXIT_STATUS,
                                   f"timeout after {timeout_s}s (packed worker killed by the watchdog)")
                        running.clear()
                        break
            proc.wait()
            t_err.join(timeout=5)
            if killed and restarts < MAX_WORKER_RESTARTS:
                restarts += 1
                continue
            # a worker that died mid-run: every unfinished task fails loudly
            tail = "".join(err_lines)[-4096:] or f"packed worker exited with {proc.returncode}"
            for si, ts in pending.items():
                for t in ts:
                    if t.task_id in seen_end:
                        continue
                    now = clock.now_ms()
                    record(t.task_id, si, starts.get(t.task_id, (now, None))[0], now, 1, tail)
            break

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
