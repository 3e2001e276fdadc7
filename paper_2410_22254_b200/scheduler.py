"""Per-GPU lane scheduler: the packed replacement of the reference's slot threads.

Reference semantics it keeps (executor.py:162-233, plan.py:100-127):
* every slot drains ITS queue front to back, one task at a time;
* slots pinned to the same GPU run concurrently;
* a failing task never stops its slot's queue;
* timeout -> status 124, bad task -> non-zero status with the reason on the
  task's stderr (OOM text contains "out of memory" -> oom_flag).

What changes: the slots pinned to one GPU are *lanes* of packs (one pack per
(model, batch) kind) inside one context; a slot's current task occupies lane
``slot_local_index`` of the pack of its kind.  Whenever a lane finishes, the
slot's next task is loaded into it (queue refill / job churn, SURVEY §8f
rank 1) between graph-replayed step chunks.

The backend is abstract (``create_pack``) so this logic is unit-tested on CPU
with a fake backend (tests/test_scheduler.py); the real one is libtlk.
"""

from __future__ import annotations

import collections
import time
from dataclasses import dataclass, field

from .jobspec import JobSpec

TIMEOUT_EXIT_STATUS = 124


@dataclass
class SlotTask:
    task_id: int
    spec: JobSpec | None
    error: str | None = None  # argv that failed to parse


@dataclass
class SlotState:
    slot_index: int
    local: int  # lane index inside every pack of this GPU
    queue: collections.deque
    current: object = None


@dataclass
class Running:
    task: SlotTask
    pack: object
    key: tuple
    lane: int
    t_start: float
    steps: int
    done: int = 0


@dataclass
class TaskOutcome:
    task_id: int
    slot_index: int
    status: int
    err: str = ""
    summary: dict = field(default_factory=dict)


class LaneScheduler:
    def __init__(self, backend, slots, timeout_s=None, chunk=64, on_start=None, on_end=None,
                 clock=time.monotonic):
        """slots: [(slot_index, [SlotTask, ...]), ...] in binding order."""
        self.backend = backend
        self.slots = [SlotState(si, k, collections.deque(tasks)) for k, (si, tasks) in enumerate(slots)]
        self.timeout_s = timeout_s
        self.chunk = max(1, int(chunk))
        self.on_start = on_start or (lambda task_id, slot_index: None)
        self.on_end = on_end or (lambda outcome: None)
        self.clock = clock
        self.packs: dict = {}
        self.failed_keys: dict = {}
        self.samples = 0
        self.steps_run = 0
        self.busy_s = 0.0
        self.outcomes: list[TaskOutcome] = []

    # -- pack management ---------------------------------------------------
    def _max_steps(self, key):
        return max((t.spec.steps for s in self.slots for t in list(s.queue)
                    + ([s.current.task] if isinstance(s.current, Running) else [])
                    if t.spec is not None and (t.spec.model, t.spec.batch) == key), default=1)

    def _pack_for(self, key):
        if key in self.failed_keys:
            raise RuntimeError(self.failed_keys[key])
        if key not in self.packs:
            try:
                self.packs[key] = self.backend.create_pack(key[0], key[1], len(self.slots),
                                                           self._max_steps(key))
            except Exception as exc:  # admission failure (e.g. out of memory)
                self.failed_keys[key] = str(exc)
                raise
        return self.packs[key]

    def _finish(self, slot, status, err="", summary=None):
        run = slot.current
        out = TaskOutcome(run.task.task_id if isinstance(run, Running) else run.task_id,
                          slot.slot_index, status, err, summary or {})
        slot.current = None
        self.outcomes.append(out)
        self.on_end(out)

    # -- main loop ----------------------------------------------------------
    def _admit(self):
        for slot in self.slots:
            while slot.current is None and slot.queue:
                task = slot.queue.popleft()
                self.on_start(task.task_id, slot.slot_index)
                if task.spec is None:
                    slot.current = task
                    self._finish(slot, 2, task.error or "not a packable job")
                    continue
                key = (task.spec.model, task.spec.batch)
                try:
                    pack = self._pack_for(key)
                    pack.load(slot.local, task.spec, task_id=task.task_id, slot_index=slot.slot_index)
                except Exception as exc:
                    slot.current = task
                    self._finish(slot, 1, f"{type(exc).__name__}: {exc}")
                    continue
                slot.current = Running(task, pack, key, slot.local, self.clock(), task.spec.steps)

    def run(self):
        while True:
            self._admit()
            running = [s for s in self.slots if isinstance(s.current, Running)]
            if not running:
                break
            n = min(self.chunk, min(s.current.steps - s.current.done for s in running))
            n = max(1, n)
            t0 = self.clock()
            packs = {id(s.current.pack): s.current.pack for s in running}
            for p in packs.values():
                p.run(n)
            for p in packs.values():
                p.sync()
            self.busy_s += self.clock() - t0
            self.steps_run += n
            now = self.clock()
            for s in running:
                r = s.current
                r.done = min(r.steps, r.done + n)
                self.samples += n * r.task.spec.batch
                if r.done >= r.steps:
                    summary = r.pack.summary(r.lane, r.steps)
                    self._finish(s, 0, "", summary)
                elif self.timeout_s is not None and now - r.t_start > self.timeout_s:
                    r.pack.release(r.lane)
                    self._finish(s, TIMEOUT_EXIT_STATUS, f"timeout after {self.timeout_s}s")
        return self.outcomes

    def stats(self) -> dict:
        return {"samples": self.samples, "busy_s": self.busy_s, "step_chunks": self.steps_run,
                "samples_per_s": self.samples / self.busy_s if self.busy_s > 0 else None,
                "packs": {f"{k[0]}/bs{k[1]}": len(self.slots) for k in self.packs}}


class TlkBackend:
    """libtlk-backed packs for LaneScheduler."""

    def __init__(self, device: int = 0):
        from . import runtime as rt

        self.rt = rt
        self.ctx = rt.Context(device)

    def create_pack(self, model, batch, lanes, max_steps):
        return _TlkPack(self, self.ctx.pack(self.rt.MODELS[model], batch, lanes, max_steps))

    def close(self):
        self.ctx.close()


class _TlkPack:
    def __init__(self, be, pack):
        self.be, self.pack = be, pack

    def load(self, lane, spec: JobSpec, task_id=0, slot_index=0):
        rt = self.be.rt
        self.pack.load(lane, seed=spec.seed, steps=spec.steps, optimizer=rt.OPTIMIZERS[spec.optim],
                       lr=spec.lr, beta1=spec.beta1, beta2=spec.beta2, eps=spec.eps,
                       weight_decay=spec.wd, momentum=spec.momentum, task_id=task_id,
                       slot_index=slot_index)

    def release(self, lane):
        self.pack.release(lane)

    def run(self, n):
        self.pack.run(n)

    def sync(self):
        self.be.ctx.sync()

    def summary(self, lane, steps):
        losses = self.pack.losses(lane, steps)
        return {"steps": int(steps), "first_loss": float(losses[0]), "last_loss": float(losses[-1]),
                "min_loss": float(losses.min())}
