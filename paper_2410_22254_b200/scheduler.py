"""Per-GPU lane scheduler: the packed replacement of the reference's slot threads.

Reference semantics it keeps (executor.py:162-233, plan.py:100-127):
* every slot drains ITS queue front to back, one task at a time;
* slots pinned to the same GPU run concurrently;
* a failing task never stops its slot's queue;
* timeout -> status 124, bad task -> non-zero status with the reason on the
  task's stderr (OOM text contains "out of memory" -> oom_flag).

What changes: the slots pinned to one GPU are *lanes* of packs (K co-resident
jobs of one (model, batch) kind inside one context).  A slot's current task
occupies a free lane of a pack of its kind; whenever a lane finishes, the
slot's next task is loaded into a free lane (queue refill / job churn, SURVEY
§8f rank 1) between graph-replayed step chunks.

Admission is per TASK, like the reference simulator's
(sim.py:388-402: a task starts if its memory fits the device's free memory,
else it fails with OOM at once and its slot moves on):
* a task without a free lane of its kind asks for a new pack sized to the
  demand of that admission pass (the slots waiting for that kind);
* if that does not fit, the largest capacity that does is found by bisection
  (device memory or the context budget), idle packs are destroyed first when
  even one lane does not fit, and only a task for which not even a one-lane
  pack fits fails with "out of memory";
* a pack whose lanes are all free is destroyed (its memory returns to the
  device, as a finished process's does in the reference).
Packs of different kinds have their own streams and run concurrently.

The backend is abstract (``create_pack`` / ``destroy_pack``) so this logic is
unit-tested on CPU with a fake backend (tests/test_scheduler.py); the real
one is libtlk.
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
    local: int  # position of the slot among this GPU's slots
    queue: collections.deque
    current: object = None


@dataclass
class PackSlot:
    """One live pack: a (model, batch) kind with `capacity` lanes."""

    key: tuple
    handle: object
    capacity: int
    free: list = field(default_factory=list)  # free lane indices (ascending)

    def __post_init__(self):
        if not self.free:
            self.free = list(range(self.capacity))


@dataclass
class Running:
    task: SlotTask
    pack: PackSlot
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


def _is_oom(exc: Exception) -> bool:
    return bool(getattr(exc, "oom", False)) or "out of memory" in str(exc).lower()


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
        self.packs: list[PackSlot] = []
        # loss-curve capacity per kind: the longest task of that kind anywhere
        # in the plan, so any of them fits any pack of its kind
        self.max_steps: dict = {}
        for s in self.slots:
            for t in s.queue:
                if t.spec is not None:
                    k = (t.spec.model, t.spec.batch)
                    self.max_steps[k] = max(self.max_steps.get(k, 1), int(t.spec.steps))
        self.samples = 0
        self.steps_run = 0
        self.busy_s = 0.0
        self.step_s = None  # measured seconds per step chunk step (caps chunks under a timeout)
        self.packs_created = 0
        self.peak_lanes = 0
        self.outcomes: list[TaskOutcome] = []

    # -- pack management ---------------------------------------------------
    def _create(self, key, lanes):
        handle = self.backend.create_pack(key[0], key[1], lanes, self.max_steps.get(key, 1))
        ps = PackSlot(key, handle, lanes)
        self.packs.append(ps)
        self.packs_created += 1
        return ps

    def _destroy(self, ps: PackSlot):
        self.packs.remove(ps)
        self.backend.destroy_pack(ps.handle)

    def _destroy_idle(self) -> bool:
        idle = [p for p in self.packs if len(p.free) == p.capacity]
        for p in idle:
            self._destroy(p)
        return bool(idle)

    def _try_create(self, key, lanes):
        try:
            return self._create(key, lanes), None
        except Exception as exc:  # noqa: BLE001 -- classified below
            if not _is_oom(exc):
                raise
            return None, exc

    def _new_pack(self, key, want):
        """A pack of `key` with the largest capacity <= want that fits."""
        ps, err = self._try_create(key, want)
        if ps is not None:
            return ps
        if self._destroy_idle():
            ps, err = self._try_create(key, want)
            if ps is not None:
                return ps
        lo, hi = 0, want  # lo fits (0 trivially), hi does not
        while hi - lo > 1:
            mid = (lo + hi) // 2
            ps, e = self._try_create(key, mid)
            if ps is None:
                hi, err = mid, e
            else:
                self._destroy(ps)
                lo = mid
        if lo == 0:
            raise err
        return self._create(key, lo)

    def _place(self, key, demand):
        for ps in self.packs:
            if ps.key == key and ps.free:
                return ps, ps.free.pop(0)
        ps = self._new_pack(key, max(1, demand))
        return ps, ps.free.pop(0)

    def _finish(self, slot, status, err="", summary=None):
        run = slot.current
        if isinstance(run, Running):
            run.pack.free.append(run.lane)
            run.pack.free.sort()
        out = TaskOutcome(run.task.task_id if isinstance(run, Running) else run.task_id,
                          slot.slot_index, status, err, summary or {})
        slot.current = None
        self.outcomes.append(out)
        self.on_end(out)

    # -- main loop ----------------------------------------------------------
    def _admit(self):
        while True:
            waiting = [s for s in self.slots if s.current is None and s.queue]
            if not waiting:
                break
            for k, slot in enumerate(waiting):
                task = slot.queue.popleft()
                self.on_start(task.task_id, slot.slot_index)
                if task.spec is None:
                    slot.current = task
                    self._finish(slot, 2, task.error or "not a packable job")
                    continue
                key = (task.spec.model, task.spec.batch)
                # demand: this slot and the later slots of this pass waiting for the same kind
                demand = 1 + sum(1 for s in waiting[k + 1:]
                                 if s.queue and s.queue[0].spec is not None
                                 and (s.queue[0].spec.model, s.queue[0].spec.batch) == key)
                try:
                    ps, lane = self._place(key, demand)
                except Exception as exc:
                    slot.current = task
                    self._finish(slot, 1, f"{type(exc).__name__}: {exc}")
                    continue
                try:
                    ps.handle.load(lane, task.spec, task_id=task.task_id, slot_index=slot.slot_index)
                except Exception as exc:
                    ps.free.append(lane)
                    ps.free.sort()
                    slot.current = task
                    self._finish(slot, 1, f"{type(exc).__name__}: {exc}")
                    continue
                slot.current = Running(task, ps, key, lane, self.clock(), task.spec.steps)
        self._destroy_idle()

    def _chunk_steps(self, running, now):
        n = min(self.chunk, min(s.current.steps - s.current.done for s in running))
        if self.timeout_s is not None and self.step_s:
            # never run a chunk past the first task's deadline (parent watchdog backs this up)
            left = min(self.timeout_s - (now - s.current.t_start) for s in running)
            n = min(n, int(max(left, 0.0) / self.step_s) + 1)
        return max(1, n)

    def run(self):
        while True:
            self._admit()
            running = [s for s in self.slots if isinstance(s.current, Running)]
            if not running:
                break
            self.peak_lanes = max(self.peak_lanes, len(running))
            t0 = self.clock()
            n = self._chunk_steps(running, t0)
            packs = {id(s.current.pack): s.current.pack for s in running}
            for ps in packs.values():
                ps.handle.run(n)
            for ps in packs.values():
                ps.handle.sync()
            dt = self.clock() - t0
            self.busy_s += dt
            self.step_s = dt / n if self.step_s is None else 0.5 * self.step_s + 0.5 * dt / n
            self.steps_run += n
            now = self.clock()
            for s in running:
                r = s.current
                r.done = min(r.steps, r.done + n)
                self.samples += n * r.task.spec.batch
                if r.done >= r.steps:
                    summary = r.pack.handle.summary(r.lane, r.steps)
                    self._finish(s, 0, "", summary)
                elif self.timeout_s is not None and now - r.t_start > self.timeout_s:
                    r.pack.handle.release(r.lane)
                    self._finish(s, TIMEOUT_EXIT_STATUS, f"timeout after {self.timeout_s}s")
        for ps in list(self.packs):
            self._destroy(ps)
        return self.outcomes

    def stats(self) -> dict:
        return {"samples": self.samples, "busy_s": self.busy_s, "step_chunks": self.steps_run,
                "samples_per_s": self.samples / self.busy_s if self.busy_s > 0 else None,
                "packs_created": self.packs_created, "peak_lanes": self.peak_lanes}


class TlkBackend:
    """libtlk-backed packs for LaneScheduler (one context = one GPU)."""

    def __init__(self, device: int = 0, mem_limit_bytes: int | None = None):
        from . import runtime as rt

        self.rt = rt
        self.ctx = rt.Context(device)
        if mem_limit_bytes:
            self.ctx.set_mem_limit(int(mem_limit_bytes))

    def create_pack(self, model, batch, lanes, max_steps):
        # own stream: packs of different kinds (configs[3] mixes) run concurrently
        return _TlkPack(self, self.ctx.pack(self.rt.MODELS[model], batch, lanes, max_steps,
                                            flags=self.rt.PACK_OWN_STREAM))

    def destroy_pack(self, handle):
        handle.pack.destroy()

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
