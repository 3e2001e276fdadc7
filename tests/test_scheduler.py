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
    def __init__(self, log, lanes):
        self.log, self.lanes = log, [None] * lanes

    def load(self, lane, spec, task_id=0, slot_index=0):
        assert self.lanes[lane] is None or self.lanes[lane]["done"] >= self.lanes[lane]["steps"]
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
    def __init__(self, fail_models=()):
        self.log, self.fail = [], set(fail_models)
        self.packs = {}

    def create_pack(self, model, batch, lanes, max_steps):
        if model in self.fail:
            raise RuntimeError("tlk error -3: out of memory: pack allocation of 123 bytes failed")
        p = FakePack(self.log, lanes)
        self.packs[(model, batch)] = p
        return p


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
