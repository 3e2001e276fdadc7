"""CPU tests of the packed lane scheduler (host logic of the packed backend).

A fake backend stands in for libtlk (like the reference's ConstantProvider /
TraceProvider fakes for devices, telemetry.py:152-177) so the run_plan
semantics -- per-slot sequential queues, refill, continue-on-failure,
timeouts, OOM-at-admission -- are checked without a GPU.
"""

import pytest

from paper_2410_22254_b200.executor import classify_failure
from paper_2410_22254_b200.jobspec import JobSpec, parse_task
from paper_2410_22254_b200.scheduler import LaneScheduler, SlotTask


class FakePack:
    def __init__(self, log, lanes, max_steps=10**9):
        self.log, self.lanes, self.max_steps = log, [None] * lanes, max_steps
        self.destroyed = False

    def load(self, lane, spec, task_id=0, slot_index=0):
        assert not self.destroyed
        assert self.lanes[lane] is None or self.lanes[lane]["done"] >= self.lanes[lane]["steps"]
        if not 1 <= spec.steps <= self.max_steps:  # what tlk_lane_load enforces
            raise RuntimeError(f"tlk error -1: steps {spec.steps} outside 1..max_steps={self.max_steps}")
        self.lanes[lane] = {"steps": spec.steps, "done": 0, "task": task_id}
        self.log.append(("load", task_id, lane))

    def release(self, lane):
        self.lanes[lane] = None

    def run(self, n):
        for st in self.lanes:
            if st and st["done"] < st["steps"]:
                st["done"] = min(st["steps"], st["done"] + n)
        self.log.append(("run", n))

    def sync(self):
        pass

    def summary(self, lane, steps):
        return {"steps": steps, "done": self.lanes[lane]["done"]}


class FakeBackend:
    """budget: device capacity in lanes (a pack of L lanes holds L units)."""

    def __init__(self, fail_models=(), budget=None):
        self.log, self.fail = [], set(fail_models)
        self.packs = {}
        self.budget, self.used, self.peak = budget, 0, 0
        self.created, self.destroyed = [], []

    def create_pack(self, model, batch, lanes, max_steps):
        if model in self.fail or (self.budget is not None and self.used + lanes > self.budget):
            raise RuntimeError("tlk error -3: out of memory: pack allocation of 123 bytes failed")
        p = FakePack(self.log, lanes, max_steps)
        p.model, p.n = model, lanes
        self.used += lanes
        self.peak = max(self.peak, self.used)
        self.packs[(model, batch)] = p
        self.created.append((model, lanes))
        return p

    def destroy_pack(self, p):
        assert not p.destroyed
        p.destroyed = True
        self.used -= p.n
        self.destroyed.append((p.model, p.n))


def task(i, steps, model="mlp"):
    return SlotTask(i, JobSpec(model=model, steps=steps, seed=i))


def test_every_task_runs_once_in_slot_order():
    events = []
    slots = [(0, [task(0, 5), task(2, 3), task(4, 7)]), (1, [task(1, 4), task(3, 9)])]
    s = LaneScheduler(FakeBackend(), slots, chunk=100,
                      on_start=lambda t, si: events.append(("start", t, si)),
                      on_end=lambda o: events.append(("end", o.task_id, o.slot_index)))
    outs = s.run()
    assert sorted(o.task_id for o in outs) == [0, 1, 2, 3, 4]
    assert all(o.status == 0 for o in outs)
    for si, ids in ((0, [0, 2, 4]), (1, [1, 3])):
        seq = [e for e in events if e[2] == si]
        assert seq == [x for t in ids for x in (("start", t, si), ("end", t, si))]
    # never more than one task per slot in flight
    live = set()
    for kind, t, si in events:
        if kind == "start":
            assert si not in live
            live.add(si)
        else:
            live.discard(si)


def test_refill_keeps_lanes_busy_and_samples_counted():
    slots = [(0, [task(0, 2), task(2, 2)]), (1, [task(1, 4)])]
    be = FakeBackend()
    s = LaneScheduler(be, slots, chunk=100)
    s.run()
    runs = [e for e in be.log if e[0] == "run"]
    assert sum(n for _, n in runs) == 4  # slot 0: 2+2 steps overlapped with slot 1's 4
    assert s.samples == 64 * (2 + 2 + 4)


def test_bad_task_fails_and_queue_continues():
    slots = [(0, [SlotTask(0, None, "usage error: --batch"), task(1, 2)])]
    outs = LaneScheduler(FakeBackend(), slots).run()
    st = {o.task_id: o.status for o in outs}
    assert st == {0: 2, 1: 0}


def test_admission_oom_is_classified_as_oom_and_other_models_proceed():
    slots = [(0, [task(0, 2, "cnn"), task(1, 2, "mlp")]), (1, [task(2, 2, "cnn")])]
    outs = LaneScheduler(FakeBackend(fail_models={"cnn"}), slots).run()
    by = {o.task_id: o for o in outs}
    assert by[1].status == 0
    for t in (0, 2):
        assert by[t].status == 1 and classify_failure(1, by[t].err) == "oom"


def test_timeout_reports_124():
    t = [0.0]

    def clock():
        t[0] += 1.0
        return t[0]

    slots = [(0, [task(0, 1000), task(1, 1)])]
    outs = LaneScheduler(FakeBackend(), slots, timeout_s=3.0, chunk=10, clock=clock).run()
    st = {o.task_id: o.status for o in outs}
    assert st == {0: 124, 1: 0}


def test_parse_task_recognises_job_argv():
    spec = parse_task(["python3", "-m", "paper_2410_22254_b200.job", "--model", "cnn", "--seed", "3"])
    assert spec.model == "cnn" and spec.seed == 3 and spec.steps == 100
    assert parse_task(["sleep", "1"]) is None
    assert parse_task(["/usr/bin/python", "-m", "other.module"]) is None
    with pytest.raises(ValueError):
        parse_task(["python3", "-m", "paper_2410_22254_b200.job", "--batch", "7"])
    assert JobSpec(model="cnn", seed=5).argv()[2] == "paper_2410_22254_b200.job"
    assert parse_task(JobSpec(model="cnn", seed=5, lr=3e-4).argv()) == JobSpec(model="cnn", seed=5, lr=3e-4)


def test_single_longest_task_fits_its_pack():
    """the pack's step capacity must cover the task being admitted
    (one 200-step task alone on its slot, e.g. --triple 1,8,1 --gpus 8)."""
    outs = LaneScheduler(FakeBackend(), [(0, [task(0, 200, "cnn")])]).run()
    assert [(o.task_id, o.status) for o in outs] == [(0, 0)]
    slots = [(0, [task(0, 3, "cnn"), task(2, 50, "cnn")]), (1, [task(1, 7, "cnn")])]
    outs = LaneScheduler(FakeBackend(), slots).run()
    assert sorted((o.task_id, o.status) for o in outs) == [(0, 0), (1, 0), (2, 0)]


def test_per_task_admission_against_device_capacity():
    """Like sim.py:388-402 (paper: 21 of 48 jobs OOM): the tasks that fit are
    admitted, the others fail with an OOM at once and their slots move on."""
    be = FakeBackend(budget=3)
    slots = [(i, [task(i, 4, "cnn")]) for i in range(8)]
    outs = LaneScheduler(be, slots).run()
    by = {o.task_id: o for o in outs}
    ok = [t for t in by if by[t].status == 0]
    oom = [t for t in by if by[t].status == 1]
    assert ok == [0, 1, 2] and oom == [3, 4, 5, 6, 7]
    assert all(classify_failure(1, by[t].err) == "oom" for t in oom)
    assert be.peak == 3 and be.used == 0  # every pack freed at the end


def test_oom_cascades_through_the_queue_at_the_same_instant():
    be = FakeBackend(budget=2)
    # slot 2's first task cannot fit next to slots 0/1; its second task is
    # admitted after the first wave finished and freed its pack
    slots = [(0, [task(0, 2, "cnn")]), (1, [task(1, 2, "cnn")]), (2, [task(2, 2, "cnn"), task(3, 2, "mlp")])]
    s = LaneScheduler(be, slots)
    outs = {o.task_id: o.status for o in s.run()}
    assert outs[0] == 0 and outs[1] == 0 and outs[2] == 1
    assert outs[3] == 1  # admitted in the same instant as its OOM'd predecessor: still no room


def test_idle_packs_are_destroyed_and_memory_reused_by_another_kind():
    be = FakeBackend(budget=2)
    slots = [(0, [task(0, 2, "resnet18"), task(2, 3, "gpt")]), (1, [task(1, 2, "resnet18"), task(3, 1, "gpt"),
                                                                     task(4, 1, "gpt")])]
    outs = {o.task_id: o.status for o in LaneScheduler(be, slots).run()}
    assert all(v == 0 for v in outs.values()), outs
    assert ("resnet18", 2) in be.destroyed and be.used == 0


def test_pack_capacity_bisects_to_what_fits():
    be = FakeBackend(budget=5)
    slots = [(i, [task(i, 2, "cnn")]) for i in range(8)]
    outs = {o.task_id: o.status for o in LaneScheduler(be, slots).run()}
    assert sum(v == 0 for v in outs.values()) == 5
    assert ("cnn", 5) in be.created  # one pack of the largest capacity that fits


def test_heterogeneous_kinds_get_their_own_packs():
    be = FakeBackend()
    slots = [(0, [task(0, 2, "mlp")]), (1, [task(1, 2, "cnn")]), (2, [task(2, 2, "mlp")]),
             (3, [task(3, 2, "xformer")])]
    outs = LaneScheduler(be, slots).run()
    assert all(o.status == 0 for o in outs)
    assert sorted(be.created) == [("cnn", 1), ("mlp", 2), ("xformer", 1)]
