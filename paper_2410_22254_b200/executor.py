"""Plan execution: the reference's per-slot subprocess executor plus the
``backend="packed"`` switch into the B200 packed runtime.

``run_plan(plan, node_index, ...)`` keeps the reference signature, result
types and failure conventions (`/root/reference/pkg/src/trilaunch/executor.py:
20-233`):

* one ``TaskResult`` per task, ms timestamps from one monotonic origin taken
  before any slot starts, results sorted by task_id;
* timeout -> 124, spawn failure -> 127, OOM classified from the stderr tail,
  launcher exit = min(failures, 125);
* a failing task never stops its slot's queue.

``backend="subprocess"`` (default) is the reference's mechanism: one thread
per slot, one child process per task.  With K slots pinned to one GPU that is
K CUDA contexts time-sliced by the driver -- the paper's method.

``backend="packed"`` hands the node's share to
``paper_2410_22254_b200.packed.run_plan_packed``: every slot pinned to GPU g
becomes one job lane of a single per-GPU runtime whose forward/backward/
optimizer for all lanes run as grouped sm_100a kernels.
"""

from __future__ import annotations

import json
import os
import re
import subprocess
import threading
import time
from dataclasses import dataclass
from pathlib import Path

from .plan import LaunchPlan, PlanSummary, plan_summary

# Reserved statuses (reference executor.py:20-23).
TIMEOUT_EXIT_STATUS = 124
SPAWN_FAILURE_EXIT_STATUS = 127
MAX_FAILURE_EXIT = 125
STDERR_TAIL_BYTES = 4096

DEFAULT_OOM_PATTERNS = (
    r"out of memory",
    r"cannot allocate memory",
    r"\boom\b",
)

BACKENDS = ("subprocess", "packed")


@dataclass(frozen=True)
class TaskResult:
    """Reference executor.py:32-59."""

    task_id: int
    slot_index: int
    gpu_index: int | None
    start_ms: int
    end_ms: int
    exit_status: int
    oom_flag: bool = False

    @property
    def duration_ms(self) -> int:
        return self.end_ms - self.start_ms

    @property
    def failed(self) -> bool:
        return self.exit_status != 0

    def to_json_dict(self) -> dict:
        keys = ("task_id", "slot_index", "gpu_index", "start_ms", "end_ms", "exit_status", "oom_flag")
        return {k: getattr(self, k) for k in keys}


@dataclass(frozen=True)
class RunReport:
    """Reference executor.py:62-92.  ``extra`` carries packed-runtime metrics
    (samples/s, per-job loss curves) and is only serialised when non-empty."""

    plan: PlanSummary
    node_index: int
    results: tuple[TaskResult, ...]
    elapsed_ms: int
    max_observed_concurrency: int
    extra: dict | None = None

    @property
    def failures(self) -> int:
        return sum(r.failed for r in self.results)

    @property
    def exit_code(self) -> int:
        return min(self.failures, MAX_FAILURE_EXIT)

    def to_json_dict(self) -> dict:
        d = {
            "plan": self.plan.to_json_dict(),
            "node_index": self.node_index,
            "elapsed_ms": self.elapsed_ms,
            "max_observed_concurrency": self.max_observed_concurrency,
            "failures": self.failures,
            "exit_code": self.exit_code,
            "results": [r.to_json_dict() for r in self.results],
        }
        if self.extra:
            d["packed"] = self.extra
        return d

    def write_json(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_json_dict(), indent=2) + "\n")


def classify_failure(exit_status: int, stderr_tail: str, oom_patterns=DEFAULT_OOM_PATTERNS) -> str:
    """'timeout' | 'oom' | 'generic' (reference executor.py:95-102)."""
    if exit_status == TIMEOUT_EXIT_STATUS:
        return "timeout"
    if any(re.search(p, stderr_tail, re.IGNORECASE) for p in oom_patterns):
        return "oom"
    return "generic"


def _tail(data: bytes | None) -> str:
    return (data or b"")[-STDERR_TAIL_BYTES:].decode("utf-8", "replace")


def _spawn(argv, env, timeout_s, log_dir, task_id):
    """Run one task to completion -> (exit_status, stderr_tail).

    The per-task seam of the reference (executor.py:105-141): logs go to
    ``task_<id>.out/.err`` when ``log_dir`` is set, else stdout is dropped and
    stderr captured.
    """
    if log_dir is None:
        try:
            proc = subprocess.run(argv, env=env, stdout=subprocess.DEVNULL,
                                  stderr=subprocess.PIPE, timeout=timeout_s)
        except subprocess.TimeoutExpired as exc:
            return TIMEOUT_EXIT_STATUS, _tail(exc.stderr)
        except OSError as exc:
            return SPAWN_FAILURE_EXIT_STATUS, str(exc)
        return proc.returncode, _tail(proc.stderr)

    out_path = Path(log_dir) / f"task_{task_id}.out"
    err_path = Path(log_dir) / f"task_{task_id}.err"
    try:
        with open(out_path, "wb") as out, open(err_path, "wb") as err:
            status = subprocess.run(argv, env=env, stdout=out, stderr=err,
                                    timeout=timeout_s).returncode
    except subprocess.TimeoutExpired:
        status = TIMEOUT_EXIT_STATUS
    except OSError as exc:
        err_path.write_text(f"{exc}\n")
        return SPAWN_FAILURE_EXIT_STATUS, str(exc)
    try:
        data = err_path.read_bytes()
    except OSError:
        data = b""
    return status, _tail(data)


def _max_overlap(intervals) -> int:
    """Sweep-line peak concurrency; ends sort before starts at equal times
    (reference executor.py:144-159)."""
    events = sorted([(s, 1) for s, _ in intervals] + [(e, -1) for _, e in intervals])
    peak = live = 0
    for _, delta in events:
        live += delta
        if live > peak:
            peak = live
    return peak


class MonotonicClock:
    """Shared ms clock: ``round((monotonic - t0) * 1000)`` (executor.py:187-190)."""

    def __init__(self):
        self.t0 = time.monotonic()

    def now_ms(self) -> int:
        return int(round((time.monotonic() - self.t0) * 1000))


def node_bindings_of(plan: LaunchPlan, node_index: int):
    nb = [b for b in plan.bindings if b.node_index == node_index]
    if not nb:
        raise IndexError(f"node_index {node_index} has no slots in this plan")
    return nb


def finish_report(plan: LaunchPlan, node_index: int, results, elapsed_ms: int,
                  extra: dict | None = None) -> RunReport:
    ordered = tuple(sorted(results, key=lambda r: r.task_id))
    peak = _max_overlap([(r.start_ms, r.end_ms) for r in ordered]) if ordered else 0
    return RunReport(plan_summary(plan), node_index, ordered, elapsed_ms, peak, extra)


def run_plan(
    plan: LaunchPlan,
    node_index: int = 0,
    *,
    timeout_s: float | None = None,
    log_dir=None,
    oom_patterns=DEFAULT_OOM_PATTERNS,
    base_env: dict | None = None,
    backend: str = "subprocess",
    packed_options: dict | None = None,
) -> RunReport:
    """Execute node ``node_index``'s share of ``plan`` (reference executor.py:162-233).

    Env precedence per task: ``base_env`` (default ``os.environ``) < slot env
    < task ``extra_env``.  ``backend="packed"`` routes to the packed runtime
    with identical report semantics.
    """
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")
    if backend == "packed":
        from .packed import run_plan_packed

        return run_plan_packed(plan, node_index, timeout_s=timeout_s, log_dir=log_dir,
                               oom_patterns=oom_patterns, base_env=base_env,
                               **(packed_options or {}))

    mine = node_bindings_of(plan, node_index)
    if log_dir is not None:
        Path(log_dir).mkdir(parents=True, exist_ok=True)
    base = dict(os.environ if base_env is None else base_env)
    results: list[TaskResult] = []
    guard = threading.Lock()
    clock = MonotonicClock()

    def drain(binding):
        slot_env = {**base, **dict(binding.env)}
        for task in plan.queue_for(node_index, binding.slot_index):
            env = {**slot_env, **dict(task.extra_env)}
            start = clock.now_ms()
            status, tail = _spawn(list(task.argv), env, timeout_s, log_dir, task.task_id)
            end = clock.now_ms()
            oom = status != 0 and classify_failure(status, tail, oom_patterns) == "oom"
            res = TaskResult(task.task_id, binding.slot_index, binding.gpu_index,
                             start, end, status, oom)
            with guard:
                results.append(res)

    workers = [threading.Thread(target=drain, args=(b,), name=f"slot-{b.slot_index}") for b in mine]
    for w in workers:
        w.start()
    for w in workers:
        w.join()
    return finish_report(plan, node_index, results, clock.now_ms())
