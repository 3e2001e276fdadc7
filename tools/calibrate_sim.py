"""Simulator calibration from measured packed runs.

The reference simulator's ``table`` slowdown model (pkg/src/trilaunch/sim.py:
46-70) takes points k -> slowdown(k), the factor by which ONE task's runtime
grows when k tasks share its GPU.  For the packed runtime the bench's NPPN
sweep measures it directly: a step of k packed jobs takes t_k, one job alone
t_1, so slowdown(k) = t_k / t_1 (k time-sliced processes would give ~k).

usage: python tools/calibrate_sim.py profiles/r1d_bench_cnn.json [out.json]
The output holds the reference CLI flags (``--slowdown table --slowdown-table
...``) and the points, so ``--mode sim`` / ``--mode sweep`` of the reference
predict packed B200 runs.
"""
import json
import sys


def calibrate(bench: dict) -> dict:
    sweep = sorted(bench["nppn_sweep"], key=lambda r: r["jobs_per_gpu"])
    t1 = next(r["ms_per_step"] for r in sweep if r["jobs_per_gpu"] == 1)
    points = {int(r["jobs_per_gpu"]): round(r["ms_per_step"] / t1, 4) for r in sweep}
    table = ",".join(f"{k}:{v}" for k, v in sorted(points.items()))
    out = {"model": bench["config"].get("workload"), "source_ms_per_step_alone": t1, "slowdown_points": points,
           "reference_cli": ["--slowdown", "table", "--slowdown-table", table]}
    kp = bench.get("kproc_baseline")
    if kp and bench.get("value"):
        # the K-process time-sliced baseline at the same K, for comparison
        k = int(kp.get("procs", 0))
        per_job_packed = bench["value"] / max(1, bench["config"].get("jobs_per_gpu", k))
        out["kprocess_throughput_ratio_at_k"] = {k: round(bench["value"] / kp["value"], 3)} if k else None
        out["packed_samples_per_s_per_job"] = per_job_packed
    return out


if __name__ == "__main__":
    res = calibrate(json.load(open(sys.argv[1])))
    text = json.dumps(res, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")
    print(text)
