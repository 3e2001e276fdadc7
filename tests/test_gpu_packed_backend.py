"""run_plan(..., backend="packed") on a real B200.

* a parametric task list (CNN + MLP jobs, T > S so slots refill) runs through
  the drop-in API; every task exits 0, concurrency <= NPPN, per-slot order and
  TaskResult semantics hold;
* packing invariance: each task's loss curve from the pack is BIT-IDENTICAL to
  the same task trained alone (one-lane pack) -- lanes never interact;
* the job entry point runs standalone as an ordinary process;
* an allocation that cannot fit fails with "out of memory" (oom_flag) and the
  context stays usable.
"""

import json
import subprocess
import sys

import numpy as np
import pytest

from paper_2410_22254_b200 import NodeSpec, TaskDef, TripleSpec, build_plan, run_plan
from paper_2410_22254_b200 import runtime as rt
from paper_2410_22254_b200.executor import classify_failure
from paper_2410_22254_b200.jobspec import JobSpec

pytestmark = pytest.mark.gpu


def _alone(spec):
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODELS[spec.model], spec.batch, 1, spec.steps)
        p.load(0, seed=spec.seed, steps=spec.steps, optimizer=rt.OPTIMIZERS[spec.optim], lr=spec.lr,
               beta1=spec.beta1, beta2=spec.beta2, eps=spec.eps, weight_decay=spec.wd,
               momentum=spec.momentum)
        p.run(spec.steps)
        ctx.sync()
        return p.losses(0, spec.steps)


def test_packed_run_plan_refill_and_packing_invariance(tmp_path):
    specs = [JobSpec(model="cnn" if i % 3 else "mlp", seed=100 + i, steps=4 + (i % 4),
                     lr=1e-3 * (1 + i % 2), optim="sgd" if i == 5 else "adam",
                     momentum=0.9 if i == 5 else 0.0) for i in range(10)]
    tasks = [TaskDef(i, tuple(s.argv(sys.executable))) for i, s in enumerate(specs)]
    plan = build_plan(tasks, TripleSpec(1, 4, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=183359))
    report = run_plan(plan, 0, log_dir=tmp_path, backend="packed", packed_options={"chunk": 3})
    assert report.failures == 0, [(r.task_id, r.exit_status, (tmp_path / f"task_{r.task_id}.err").read_text())
                                  for r in report.results if r.exit_status]
    assert report.max_observed_concurrency <= 4
    assert [r.task_id for r in report.results] == list(range(10))
    for r in report.results:
        assert r.slot_index == r.task_id % 4 and r.gpu_index == 0
    by_slot = {}
    for r in report.results:
        by_slot.setdefault(r.slot_index, []).append(r)
    for rs in by_slot.values():
        for a, b in zip(rs, rs[1:]):
            assert a.end_ms <= b.start_ms
    assert report.to_json_dict()["packed"]["packed_slots"] == 4
    for i, spec in enumerate(specs):
        out = json.loads((tmp_path / f"task_{i}.out").read_text())
        ref = _alone(spec)
        assert out["steps"] == spec.steps
        assert np.float32(out["first_loss"]) == ref[0] and np.float32(out["last_loss"]) == ref[-1], i


def test_job_entry_point_runs_standalone():
    spec = JobSpec(model="mlp", seed=7, steps=5)
    proc = subprocess.run(spec.argv(sys.executable), capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stderr
    out = json.loads(proc.stdout.strip().splitlines()[-1])
    assert np.float32(out["last_loss"]) == _alone(spec)[-1]


def test_admission_oom_is_reported_and_context_survives():
    with rt.Context(0) as ctx:
        with pytest.raises(rt.TlkError) as ei:
            ctx.pack(rt.MODEL_CNN, 64, 4096, 1 << 24)  # ~275 GB loss curves alone
        assert ei.value.oom and classify_failure(1, str(ei.value)) == "oom"
        p = ctx.pack(rt.MODEL_MLP, 64, 1, 2)
        p.load(0, seed=1, steps=2)
        p.run(2)
        ctx.sync()
        assert p.status(0).steps_done == 2


def test_heterogeneous_mix_config4(tmp_path):
    """BASELINE configs[3]: MLP + CNN + 2-layer transformer jobs interleaved in
    one task list on one GPU (here NPPN = 6, T = 12 so slots refill).  The
    packed worker keeps one pack per (model, batch); every task succeeds and
    each loss curve equals the same job trained alone, bit for bit."""
    kinds = ["mlp", "cnn", "xformer"]
    specs = [JobSpec(model=kinds[i % 3], seed=300 + i, steps=3 + (i % 3),
                     batch=8 if kinds[i % 3] == "xformer" else 32, lr=1e-3) for i in range(12)]
    tasks = [TaskDef(i, tuple(s.argv(sys.executable))) for i, s in enumerate(specs)]
    plan = build_plan(tasks, TripleSpec(1, 6, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=183359))
    report = run_plan(plan, 0, log_dir=tmp_path, backend="packed")
    assert report.failures == 0, [(r.task_id, r.exit_status, (tmp_path / f"task_{r.task_id}.err").read_text())
                                  for r in report.results if r.exit_status]
    assert report.max_observed_concurrency <= 6
    for i, spec in enumerate(specs):
        out = json.loads((tmp_path / f"task_{i}.out").read_text())
        ref = _alone(spec)
        assert out["steps"] == spec.steps
        assert np.float32(out["first_loss"]) == ref[0] and np.float32(out["last_loss"]) == ref[-1], i


def test_cli_exec_packed_with_nvml_telemetry(tmp_path):
    """--backend packed --provider nvml: the packed worker's GPU shows up in
    telemetry.csv (reference schema) while a few hundred CNN steps run."""
    from paper_2410_22254_b200 import cli, telemetry as tm
    specs = [JobSpec(model="cnn", seed=300 + i, steps=400, lr=1e-3) for i in range(4)]
    (tmp_path / "jobs.jsonl").write_text("".join(json.dumps({"argv": s.argv(sys.executable)}) + "\n" for s in specs))
    rc = cli.run_cli(["--mode", "exec", "--triple", "1,4,1", "--tasks", str(tmp_path / "jobs.jsonl"), "--gpus", "1",
                      "--backend", "packed", "--provider", "nvml", "--interval", "0.05", "--outdir", str(tmp_path),
                      "--run-name", "r"])
    assert rc == 0
    series = tm.read_series_csv(tmp_path / "r" / "telemetry.csv")
    assert series.samples and all(len(s.gpu) == 1 for s in series.samples)
    assert max(s.gpu[0].mem_mib for s in series.samples) > 0


def test_per_task_admission_against_a_memory_budget(tmp_path):
    """SURVEY §8f rank 2 / the paper's 48-job run (21 of 48 OOM):
    with a device budget that holds only 3 CNN lanes, 16 CNN tasks on 8 slots
    (T > S): the tasks that fit are admitted and train bit-identically to the
    same task alone; the others fail AT ADMISSION with "out of memory"
    (oom_flag), and their slots go on with the next task (admitted as soon as
    memory frees, like sim.py:388-402)."""
    with rt.Context(0) as ctx:
        a = ctx.pack(rt.MODEL_CNN, 64, 1, 6)
        one = ctx.mem_in_use()
        b = ctx.pack(rt.MODEL_CNN, 64, 2, 6)
        per_lane = (ctx.mem_in_use() - one) - one  # 2-lane pack minus 1-lane pack
        fixed = one - per_lane
        a.destroy()
        b.destroy()
        assert ctx.mem_in_use() == 0
    budget_mib = (fixed + 3 * per_lane + per_lane // 2) >> 20
    specs = [JobSpec(model="cnn", seed=700 + i, steps=3 + i % 3, lr=1e-3) for i in range(16)]
    tasks = [TaskDef(i, tuple(s.argv(sys.executable))) for i, s in enumerate(specs)]
    plan = build_plan(tasks, TripleSpec(1, 8, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=budget_mib))
    report = run_plan(plan, 0, log_dir=tmp_path, backend="packed",
                      packed_options={"mem_limit_mib": budget_mib})
    by = {r.task_id: r for r in report.results}
    ok = sorted(t for t, r in by.items() if r.exit_status == 0)
    oom = sorted(t for t, r in by.items() if r.exit_status != 0)
    assert ok == [0, 1, 2, 8, 9, 10], (ok, [(t, (tmp_path / f"task_{t}.err").read_text()) for t in oom])
    for t in oom:
        assert by[t].oom_flag and by[t].exit_status == 1
        assert "out of memory" in (tmp_path / f"task_{t}.err").read_text()
    assert report.max_observed_concurrency <= 8
    for t in ok:
        out = json.loads((tmp_path / f"task_{t}.out").read_text())
        ref = _alone(specs[t])
        assert np.float32(out["last_loss"]) == ref[-1], t


def test_heterogeneous_packs_run_concurrently_on_their_own_streams():
    """configs[3]: packs of different models (own streams) overlap on the
    device -- two packs replayed together finish sooner than back to back --
    and each lane's losses stay bit-identical to running its pack alone."""
    import time

    def make(ctx, flags):
        m = ctx.pack(rt.MODEL_MLP, 64, 4, 200, flags=flags)
        c = ctx.pack(rt.MODEL_CNN, 64, 4, 200, flags=flags)
        for p in (m, c):
            for j in range(4):
                p.load(j, seed=800 + j, steps=200)
        return m, c

    with rt.Context(0) as ctx:
        m, c = make(ctx, rt.PACK_OWN_STREAM)
        assert m.stream_handle != c.stream_handle
        m.run(5), c.run(5)
        ctx.sync()
        t0 = time.perf_counter()
        m.run(100), c.run(100)
        ctx.sync()
        both = time.perf_counter() - t0
        t0 = time.perf_counter()
        m.run(95)
        ctx.sync()
        c.run(95)
        ctx.sync()
        serial = time.perf_counter() - t0
        ctx.sync()
        lm = [m.losses(j, 200) for j in range(4)]
        lc = [c.losses(j, 200) for j in range(4)]
    assert both < serial * 1.02, (both, serial)
    with rt.Context(0) as ctx:
        m2, c2 = make(ctx, 0)
        m2.run(200)
        c2.run(200)
        ctx.sync()
        for j in range(4):
            assert np.array_equal(m2.losses(j, 200), lm[j]) and np.array_equal(c2.losses(j, 200), lc[j])
