#!/usr/bin/env python
"""Aggregate training samples/s of K co-resident jobs per B200 (packed triples mode).

Workload (BASELINE.json configs[1]): 8 co-resident MNIST-CNN training jobs
per GPU (triples [1, 8*N, 1] -> 8 slots pinned to each GPU), batch 64 per
job, Adam, synthetic on-device data.  One *step* = one optimizer step of all
8 jobs on a GPU (512 samples per GPU).  N>1 (torchrun): every rank runs its
own 8 jobs -- the jobs are independent, so there is no data-path collective
(weak scaling); the only NCCL call is the MAX-reduction of the timings.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl packed|reference]

Prints ONE JSON line (rank 0).  Keys beyond the driver contract:
roofline (dominant kernel), step_roofline (whole step vs max(F/peak_tc,
B/peak_hbm)), cpu_baseline (the oracle CPU path, run through run_plan = the
reference's mechanism), kproc_baseline (K-process time-sliced PyTorch, the
paper's mechanism), kernels (per-kernel device ms of one step).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aggregate samples/sec per B200 vs jobs/GPU (triples NPPN); 1/2/4/8-GPU scaling"
UNIT = "samples/s"
# name -> (model, batch per job, jobs per GPU, description).  The default
# (driver) line is configs[1]; the others are the BASELINE configs' job
# models at their per-GPU packing (a sample = one image / one sequence).
WORKLOADS = {
    "cnn": ("cnn", 64, 8, "configs[1]: 8 co-resident MNIST CNN jobs packed per B200 (triples [1,8,1] per GPU)"),
    "mlp": ("mlp", 64, 4, "configs[0]: 4 MNIST-MLP jobs packed on one device (triples [1,4,1])"),
    "xformer": ("xformer", 32, 32, "configs[3] transformer job (2 layers, d=256, T=128), 32 jobs/GPU"),
    "gpt": ("gpt", 64, 16, "configs[4]: tiny-GPT (6 layers, d=384, T=256) sweep, 16 jobs/GPU"),
    "resnet18": ("resnet18", 128, 8, "configs[2]: ResNet-18/CIFAR-shape sweep, 64 jobs over 8 GPUs = 8 jobs/GPU, "
                                     "bs 128, SGD momentum"),
}
# per-workload optimizer of the synthetic task list
WORKLOAD_OPT = {"resnet18": dict(optim="sgd", lr=0.05, momentum=0.9)}


def rn_kernel_work(name, batch, lanes):
    """FLOPs of all launches of a ResNet conv kernel family in one step."""
    C = (64, 128, 256, 512)
    main = ds = 0
    cin, res = 64, 32
    for s in range(4):
        for b in range(2):
            ci = cin if b == 0 else C[s]
            ho = res // 2 if (b == 0 and s > 0) else res
            main += ho * ho * C[s] * 9 * (ci + C[s])
            if b == 0 and s > 0:
                ds += ho * ho * C[s] * ci
            res = ho
            if b == 1:
                cin = C[s]
    fam = {"conv_fwd": main, "conv_dgrad": main, "conv_wgrad": main,
           "conv_fwd_ds": ds, "conv_dgrad_ds": ds, "conv_wgrad_ds": ds}
    return 2.0 * batch * lanes * fam[name] if name in fam else None
WORKLOAD = WORKLOADS["cnn"][3]
JOBS_PER_GPU = 8
BATCH = 64
MODEL = "cnn"
LAUNCHES_PER_STEP = None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------- dist --------
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    from paper_2410_22254_b200.multigpu import max_over_ranks

    return max_over_ranks(x)


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------- clocks ------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 10 ms; summary() keeps
    the samples stamped inside the timed window (mark_start / mark_end)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.dev = device_index
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"], stdout=self.f,
                stderr=subprocess.DEVNULL)
            time.sleep(0.5)  # let the sampler come up before the measured work
        except OSError:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        import datetime

        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 10:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    ts = None
                rows.append((ts, parts))
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        win = [p for ts, p in rows if ts is not None and self.t0 and self.t1 and
               self.t0 - 0.01 <= ts <= self.t1 + 0.01]
        scope = "timed region"
        if not win:  # region shorter than the sampling period: nearest samples
            win = [p for ts, p in rows if ts is not None and self.t0 and self.t1 and
                   self.t0 - 0.1 <= ts <= self.t1 + 0.1] or [p for _, p in rows]
            scope = "timed region +-100 ms"
        num = lambda s: s.replace(".", "", 1).isdigit()
        sm = [float(r[2]) for r in win if num(r[2])]
        mx = [float(r[3]) for r in win if num(r[3])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in win for i in range(4) if r[6 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(win), "scope": scope}


# ---------------------------------------------------------------- roofline ----
def kernel_work(name, info, lanes, batch):
    """(bound, algorithmic units per launch) for an MLP/CNN-pack kernel; units
    are FLOPs for tensor-bound kernels and bytes for HBM-bound ones."""
    B, L = batch, lanes
    if MODEL == "mlp":
        if B == 64:  # csrc/mlp2.cu: two launches per step
            return {
                # fc1, fc2, fc2 dgrad on tcgen05 (+ inputs, head on CUDA cores): a latency chain
                "mlp_step": ("tensor", 2.0 * B * (784 * 512 + 2 * 512 * 512) * L),
                # fused wgrad + optimizer of fc1.w / fc2.w: p, m, v read + write and the bf16 shadow
                "mlp_wgrad_adam": ("hbm", 26.0 * (784 * 512 + 512 * 512) * L),
            }.get(name, ("hbm", 0.0))
        return {
            "fc1_fwd": ("tensor", 2.0 * B * 784 * 512 * L),
            "fc2_fwd": ("tensor", 2.0 * B * 512 * 512 * L),
            "fc2_wgrad": ("tensor", 2.0 * B * 512 * 512 * L),
            "fc2_dgrad": ("tensor", 2.0 * B * 512 * 512 * L),
            "fc1_wgrad": ("tensor", 2.0 * B * 784 * 512 * L),
            "optimizer": ("hbm", 30.0 * info.param_count * L),
            "inputs": ("hbm", L * B * (784 + 784 * 2 + 4)),
            "head": ("hbm", L * B * 512 * 2),
        }.get(name, ("hbm", 0.0))
    conv2_flops = 2.0 * B * 576 * 64 * 288 * L
    fc1_flops = 2.0 * B * 9216 * 128 * L
    act = {
        # fc1.w (9216x128, 98% of the params) is updated inside its wgrad
        # epilogue: p, m, v read + write and the bf16 shadow (26 B/param); the
        # batched optimizer does the rest (28 B/param + 2 B shadow)
        "fc1_wgrad_adam": ("hbm", 26.0 * 9216 * 128 * L),
        # the other 2%: partial-sum finalisation + update (30 B/param)
        "grad_finalize_opt": ("hbm", L * (30.0 * (info.param_count - 9216 * 128)
                                          + 4.0 * (18 * 288 * 64 + 9216 + B * 320))),
        "conv2_fwd_pool": ("tensor", conv2_flops),
        "conv2_wgrad": ("tensor", conv2_flops),
        "conv2_dgrad": ("tensor", conv2_flops),
        "fc1_fwd_splitk": ("tensor", fc1_flops),
        "fc1_dgrad_unpool": ("tensor", fc1_flops),
        # CUDA-core / bookkeeping kernels: compulsory HBM bytes
        "inputs_conv1_fwd": ("hbm", L * B * (784 + 784 * 2 + 4 + 676 * 32 * 2)),
        "conv1_wgrad": ("hbm", L * B * (784 * 2 + 676 * 32 * 2)),
        "fc1_reduce_head": ("hbm", L * (18 * 128 * 64 * 4 + B * 128 * 2 * 2)),
        "end_step": ("hbm", L * 128),
    }
    return act.get(name, ("hbm", 0.0))


def step_roofline(info, lanes, batch, hbm_gbs, tflops):
    """t_roof = max(F / peak_tc, B / peak_hbm) for one step of all lanes:
    F = 3 x 2 x MACs per sample (libtlk's model table), B = 28 B/param Adam traffic."""
    flops = float(info.flops_per_sample) * batch * lanes
    bytes_ = 28.0 * info.param_count * lanes
    return max(flops / (tflops * 1e12), bytes_ / (hbm_gbs * 1e9)), flops, bytes_


GPT_CFG = {"xformer": (2, 256, 4, 128, 256), "gpt": (6, 384, 6, 256, 65)}


def gpt_kernel_work(name, model, batch, lanes):
    """Algorithmic FLOPs of one launch of a transformer-pack GEMM (per launch =
    one layer's product for all lanes); None for non-GEMM kernels."""
    Lr, d, H, T, V = GPT_CFG[model]
    N = batch * T * lanes
    attn = 2.0 * batch * lanes * H * T * T * 64
    table = {"qkv": 2.0 * N * 3 * d * d, "proj": 2.0 * N * d * d, "fc": 2.0 * N * 4 * d * d,
             "fc2": 2.0 * N * 4 * d * d, "attn_scores": attn, "attn_pv": attn, "attn_dp": attn,
             "attn_dq": attn, "attn_dk": attn, "attn_dv": attn,
             # fused attention (attn.cuh): S and PV forward; dP, dQ, dK, dV backward
             # (the backward's recomputed S is not counted)
             "attn_fwd": 2 * attn, "attn_bwd": 4 * attn,
             "qkv_wgrad": 2.0 * N * 3 * d * d, "qkv_dgrad": 2.0 * N * 3 * d * d,
             "proj_wgrad": 2.0 * N * d * d, "proj_dgrad": 2.0 * N * d * d,
             "fc_wgrad": 2.0 * N * 4 * d * d, "fc_dgrad": 2.0 * N * 4 * d * d,
             "fc2_wgrad": 2.0 * N * 4 * d * d, "fc2_dgrad": 2.0 * N * 4 * d * d,
             "head_ce": 2.0 * N * V * d, "head_dgrad": 2.0 * N * V * d, "head_wgrad": 2.0 * N * V * d}
    return table.get(name)


# ---------------------------------------------------------------- baselines ---
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_launcher():
    """The vendored reference launcher (baseline/_ref/trilaunch, pip-installed
    from /root/reference) when present, else this package's drop-in API."""
    if os.path.isdir(os.path.join(REF_DIR, "trilaunch")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import trilaunch  # noqa: F401

            return trilaunch, "reference trilaunch (baseline/_ref) run_plan"
        except Exception:  # pragma: no cover
            pass
    import paper_2410_22254_b200 as pkg

    return pkg, "paper_2410_22254_b200 run_plan (subprocess backend = the reference mechanism)"


def run_tasks_via_run_plan(argvs, ntpp, timeout, launcher=None):
    """Launch tasks as processes through run_plan (the reference mechanism):
    one slot per task, all concurrent."""
    mod = launcher or reference_launcher()[0]
    tasks = [mod.TaskDef(i, tuple(a)) for i, a in enumerate(argvs)]
    cores = os.cpu_count() or 1
    plan = mod.build_plan(tasks, mod.TripleSpec(1, len(tasks), ntpp), mod.NodeSpec(cores=max(cores, 1)))
    logdir = tempfile.mkdtemp(prefix="tlk_bench_")
    env = dict(os.environ, PYTHONPATH=ROOT)
    report = mod.run_plan(plan, 0, log_dir=logdir, timeout_s=timeout, base_env=env)
    outs = []
    for r in report.results:
        try:
            txt = open(os.path.join(logdir, f"task_{r.task_id}.out")).read().strip().splitlines()
            outs.append(json.loads(txt[-1]))
        except Exception:
            outs.append({"error": f"exit {r.exit_status}"})
    return report, outs


def host_cores():
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        aff = None
    return os.cpu_count() or 1, aff


def cpu_oracle_rate(steps, warmup, jobs=None, batch=None, model=None, launcher=None):
    """The numpy oracle jobs run as `jobs` concurrent processes on the host
    cores (run_plan, OMP_NUM_THREADS = cores // jobs); returns the aggregate
    steady-state samples/s and the thread count used."""
    jobs = JOBS_PER_GPU if jobs is None else jobs
    batch = BATCH if batch is None else batch
    model = MODEL if model is None else model
    cores = os.cpu_count() or 1
    ntpp = max(1, cores // jobs)
    argvs = [[sys.executable, "-m", "oracle.job", "--model", model, "--seed", str(i), "--batch",
              str(batch), "--steps", str(steps + warmup), "--warmup", str(warmup), "--json"]
             for i in range(jobs)]
    report, outs = run_tasks_via_run_plan(argvs, ntpp, timeout=1800, launcher=launcher)
    rates = [o.get("samples_per_s") for o in outs]
    if any(r is None for r in rates):
        return None, ntpp * jobs, outs
    return float(sum(rates)), ntpp * jobs, outs


def kproc_rate(jobs=None, duration=10.0, lead=35.0, fast=0):
    jobs = JOBS_PER_GPU if jobs is None else jobs
    sync = tempfile.mkdtemp(prefix="tlk_kproc_")
    argvs = [[sys.executable, os.path.join(ROOT, "baselines", "kproc_torch.py"), "--model", MODEL,
              "--seed", str(i), "--batch", str(BATCH), "--sync-dir", sync, "--procs", str(jobs),
              "--duration", str(duration), "--fast", str(fast)] for i in range(jobs)]
    report, outs = run_tasks_via_run_plan(argvs, 1, timeout=lead + duration + 600)
    rates = [o.get("samples_per_s") for o in outs]
    if any(r is None for r in rates):
        return None, outs
    return float(sum(rates)), outs


# ---------------------------------------------------------------- arms --------
def reference_arm(a, world, rank):
    """--impl reference: the reference's CPU path for these tasks -- its own
    launcher (vendored trilaunch run_plan) spawning the numpy oracle jobs (the
    reference has no training code of its own), on all host cores."""
    if rank != 0:
        return 0
    # bounded sample: each "step" is one optimizer step of all jobs (~0.2 s
    # for the CNN); steps beyond 40 are not run, and "steps" says so
    timed = max(1, min(a.steps, 40))
    warm = 1
    launcher, lname = reference_launcher()
    value, cores, outs = cpu_oracle_rate(timed, warm, launcher=launcher)
    ncpu, aff = host_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": timed, "requested_steps": a.steps, "warmup": a.warmup,
        "ms_per_step": (JOBS_PER_GPU * BATCH / value * 1e3) if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter RNG, same seeds/shapes as the packed arm)",
        "config": {"workload": WORKLOAD, "jobs": JOBS_PER_GPU, "batch_per_job": BATCH,
                   "optimizer": "adam", "path": f"oracle/ numpy jobs launched by {lname} (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "host_cpu_count": ncpu, "affinity_cpus": aff,
                         "sample": f"{JOBS_PER_GPU} {MODEL.upper()} jobs x {timed} timed steps (+{warm} warm-up), "
                                   f"bs {BATCH}, concurrent processes via {lname}, "
                                   f"OMP_NUM_THREADS={max(1, (os.cpu_count() or 1) // JOBS_PER_GPU)}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "errors": [o for o in outs if "error" in o][:2],
    }
    print(json.dumps(line), flush=True)
    return 0


def packed_arm(a, world, rank, local):
    import numpy as np
    import torch

    from paper_2410_22254_b200 import runtime as rt

    torch.cuda.set_device(local)
    hbm, tc, tc_sus, peak_kind = load_peaks()
    from paper_2410_22254_b200 import TaskDef
    from paper_2410_22254_b200.jobspec import JobSpec, parse_task
    from paper_2410_22254_b200.multigpu import rank_share, weak_scaling_plan

    lanes = a.jobs
    ctx = rt.Context(local)
    total_steps = a.warmup + a.steps + 2 * a.profile_iters + 2  # (+ the CNN full-grid re-profile)
    # the workload as a parametric task list through the triples mapping:
    # triples [1, jobs*world, 1] on a world-GPU node; this rank trains the
    # slots pinned to GPU `rank` (task i -> slot i -> GPU i % world).
    opt = WORKLOAD_OPT.get(MODEL, dict(lr=1e-3))
    plan = weak_scaling_plan(lanes, world, lambda i: TaskDef(i, tuple(
        JobSpec(model=MODEL, seed=i, steps=total_steps, batch=BATCH, **opt).argv())))
    share = rank_share(plan, rank)
    pack = ctx.pack(rt.MODELS[MODEL], BATCH, lanes, total_steps)
    for j, (slot, tasks) in enumerate(share):
        spec = parse_task(tasks[0].argv)
        pack.load(j, seed=spec.seed, steps=spec.steps, optimizer=rt.OPTIMIZERS[spec.optim], lr=spec.lr,
                  beta1=spec.beta1, beta2=spec.beta2, eps=spec.eps, weight_decay=spec.wd,
                  momentum=spec.momentum, task_id=tasks[0].task_id, slot_index=slot)
    stream = torch.cuda.ExternalStream(ctx.stream_handle)

    with ClockSampler(local) as clk:
        pack.run(a.warmup)
        ctx.sync()
        barrier(world)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.mark_start()
        ev0.record(stream)
        pack.run(a.steps)
        ev1.record(stream)
        ev1.synchronize()
        clk.mark_end()
        torch.cuda.synchronize()
        barrier(world)
        ms = ev0.elapsed_time(ev1)
    clocks = clk.summary()
    ms_max = dist_max(ms, world)
    samples = world * lanes * BATCH * a.steps
    value = samples / (ms_max / 1e3)

    # per-kernel device times of one step (CUDA events on the launching stream)
    kernels = pack.profile_step(a.profile_iters)
    step_ms = sum(t for _, t in kernels)
    if MODEL in GPT_CFG:
        # one launch per layer per name: dominant = the GEMM family with the
        # largest total time; roofline per launch of it
        tot, cnt = {}, {}
        for k, v in kernels:
            tot[k] = tot.get(k, 0.0) + v
            cnt[k] = cnt.get(k, 0) + 1
        gem = [k for k in tot if gpt_kernel_work(k, MODEL, BATCH, lanes)]
        top_name = max(gem, key=lambda k: tot[k])
        top_ms = max(tot[top_name] / cnt[top_name], 1e-6)
        bound, work = "tensor", gpt_kernel_work(top_name, MODEL, BATCH, lanes)
        kernels_out = {k: round(v, 5) for k, v in tot.items()}
    elif MODEL == "resnet18":
        # conv families (20 launches each per step, different shapes): the
        # dominant family's total FLOPs over its total device time
        tot = {}
        for k, v in kernels:
            tot[k] = tot.get(k, 0.0) + v
        fams = [k for k in tot if rn_kernel_work(k, BATCH, lanes)]
        top_name = max(fams, key=lambda k: tot[k])
        top_ms = max(tot[top_name], 1e-6)
        bound, work = "tensor", rn_kernel_work(top_name, BATCH, lanes)
        kernels_out = {k: round(v, 5) for k, v in tot.items()}
    else:
        top_name, top_ms = max(kernels, key=lambda kv: kv[1])
        top_ms = max(top_ms, 1e-6)
        bound, work = kernel_work(top_name, pack.info, lanes, BATCH)
        kernels_out = {k: round(v, 5) for k, v in kernels}
    if bound == "tensor":
        achieved = work / (top_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": top_name, "achieved": achieved, "peak": tc,
                "unit": "TFLOP/s", "frac": achieved / tc, "traffic": None,
                "algorithmic_per_launch": work, "ms_per_launch": top_ms,
                "share_of_step": top_ms / step_ms, "peak_source": peak_kind}
    else:
        achieved = work / (top_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": top_name, "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                "algorithmic_per_launch": work, "ms_per_launch": top_ms,
                "share_of_step": top_ms / step_ms, "peak_source": peak_kind}
    # the profile step serialises the kernels on one stream (no graph
    # branches); each kernel runs at its in-graph grid (CNN fc1 wgrad+Adam:
    # the 72 of 148 CTAs it gets on the defer stream, beside the step's tail
    # and the next step's forward)
    roof["timing"] = ("CUDA events around each kernel of a serial (unforked) profile step, "
                      "mean of %d; kernels at their in-graph grids" % a.profile_iters)
    if MODEL == "cnn" and top_name == "fc1_wgrad_adam":
        # the same kernel re-profiled on one CTA per SM (its grid when it runs alone)
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        old = os.environ.get("TLK_FWA_CTAS")
        os.environ["TLK_FWA_CTAS"] = str(sms)
        try:
            full = dict(pack.profile_step(a.profile_iters)).get("fc1_wgrad_adam")
        finally:
            if old is None:
                os.environ.pop("TLK_FWA_CTAS")
            else:
                os.environ["TLK_FWA_CTAS"] = old
        if full:
            ach = work / (full / 1e3) / 1e9
            roof["full_grid"] = {"ctas": sms, "ms_per_launch": full, "achieved": ach, "frac": ach / hbm,
                                 "in_graph_ctas": sms * 72 // 148}
    try:  # dram bytes of this kernel from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(MODEL, {}).get(top_name)
        if tr:
            roof["traffic"] = tr["dram_bytes"]
            roof["traffic_source"] = tr["source"]
    except (OSError, ValueError):
        pass
    t_roof, sflops, sbytes = step_roofline(pack.info, lanes, BATCH, hbm, tc)
    ms_step = ms_max / a.steps

    # end-to-end through the public API with HOST buffers (pinned), per step:
    # H2D of the step's pixels+labels, one packed step, D2H of the losses.
    if MODEL in GPT_CFG or MODEL == "resnet18":
        global LAUNCHES_PER_STEP
        LAUNCHES_PER_STEP = pack.launches_per_step()
        return _finish_gpt_line(a, world, rank, ctx, pack, value, ms_step, clocks, roof, t_roof,
                                sflops, sbytes, lanes, kernels_out)
    e2e_steps = max(3, min(a.steps, 100))
    hpack = ctx.pack(rt.MODELS[MODEL], BATCH, lanes, a.warmup + e2e_steps + 2, host_input=True)
    for j in range(lanes):
        hpack.load(j, seed=rank * lanes + j, steps=a.warmup + e2e_steps + 2)
    rng = np.random.default_rng(rank)
    px = torch.from_numpy(rng.integers(0, 256, (lanes, BATCH, 784), dtype=np.uint8)).pin_memory()
    lb = torch.from_numpy(rng.integers(0, 10, (lanes, BATCH), dtype=np.int32)).pin_memory()
    loss_out = torch.empty(lanes, dtype=torch.float32).pin_memory()
    pxn, lbn = px.numpy(), lb.numpy()
    # two pinned loss buffers: step k's losses are read on the host (after
    # tlk_step_host_wait) while step k+1 -- whose H2D overlaps step k's
    # kernels (tlk_step_host_async) -- is already enqueued
    lons = [torch.empty(lanes, dtype=torch.float32).pin_memory().numpy() for _ in range(2)]
    seen = []

    def run_host_steps(n):
        prev = None
        for k in range(n):
            t = hpack.step_host_async(pxn, lbn, lons[k & 1])
            if prev is not None:
                hpack.step_host_wait(prev)
                seen.append(float(lons[(k - 1) & 1][0]))  # the previous step's result, on the host
            prev = t
        hpack.step_host_wait(prev)
        seen.append(float(lons[(n - 1) & 1][0]))
        ctx.sync()  # the last step's deferred fc1 update (CNN) is inside the timed region

    run_host_steps(max(1, a.warmup))
    barrier(world)
    t0 = time.perf_counter()
    run_host_steps(e2e_steps)
    e2e_s = dist_max(time.perf_counter() - t0, world)
    assert len(seen) == max(1, a.warmup) + e2e_steps and all(math.isfinite(v) for v in seen)
    e2e_value = world * lanes * BATCH * e2e_steps / e2e_s
    h2d = lanes * BATCH * 784 + lanes * BATCH * 4
    d2h = lanes * 4

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (on-device counter RNG MNIST-shaped batches, teacher labels; random-init weights)",
        "config": {"workload": WORKLOAD, "triple": [1, JOBS_PER_GPU * world, 1],
                   "jobs_per_gpu": lanes, "batch_per_job": BATCH, "samples_per_step_per_gpu": lanes * BATCH,
                   "optimizer": "adam (fp32 master, bf16 GEMM operands)",
                   "parallelism": f"independent jobs, {lanes}/GPU x {world} GPU(s), no collective",
                   "l2": "no explicit flush: per-step working set "
                         f"{(16 * pack.info.param_count * lanes + 115e6 / 8 * lanes) / 1e6:.0f} MB > 126 MB L2"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_2410_22254_b200.runtime.Pack.step_host_async/_wait -> tlk_step_host_async "
                       "(pinned host buffers; step k+1's H2D overlaps step k; every step's losses read on the host)",
                "steps": e2e_steps},
        "gpu_launches": pack.launches_per_step() * a.steps,
        "clocks": clocks,
        "roofline": roof,
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "measured_ms": ms_step,
                          "frac": t_roof * 1e3 / ms_step, "flops_per_step": sflops,
                          "compulsory_bytes_per_step": sbytes,
                          "samples_per_s_roof": lanes * BATCH / t_roof},
        "kernels": kernels_out,
    }
    if rank == 0 and world == 1 and a.sweep:
        # the metric's "vs jobs/GPU" axis: packed throughput for NPPN/GPU = 1..32
        line["nppn_sweep"] = nppn_sweep(ctx, stream, (1, 2, 4, 8, 16, 32), 10, 50)
    if rank == 0 and world == 1 and not a.no_baselines:
        launcher, lname = reference_launcher()
        cpu, cores, _ = cpu_oracle_rate(2, 1, launcher=launcher)
        ncpu, aff = host_cores()
        line["cpu_baseline"] = {
            "value": cpu, "unit": UNIT, "cores": cores, "kind": "port", "host_cpu_count": ncpu,
            "affinity_cpus": aff,
            "sample": f"{JOBS_PER_GPU} {MODEL.upper()} jobs x 2 timed steps (+1 warm-up), bs {BATCH}, numpy oracle, "
                      f"concurrent processes via {lname}"}
        for key, fast, mech in (("kproc_baseline", 0, "PyTorch (fp32, cudnn, loss.item() per step) processes"),
                                ("kproc_fast_baseline", 1, "PyTorch (bf16 autocast, fused Adam, host sync every "
                                                           "50 steps) processes")):
            kp, outs = kproc_rate(JOBS_PER_GPU, duration=a.kproc_seconds, fast=fast)
            line[key] = {
                "value": kp, "unit": UNIT, "procs": JOBS_PER_GPU,
                "mechanism": f"{JOBS_PER_GPU} {mech} pinned to one GPU via run_plan, time-sliced",
                "packed_over_kproc": (value / kp) if kp else None,
                "packed_e2e_over_kproc": (e2e_value / kp) if kp else None,
                "errors": [o for o in outs if "error" in o][:2]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def nppn_sweep(ctx, stream, jobs_list, warm, timed):
    """Packed throughput vs co-resident jobs per GPU (the metric's NPPN axis):
    a fresh pack of k lanes per point, `warm` untimed then `timed` timed steps."""
    import torch

    from paper_2410_22254_b200 import runtime as rt

    opt = WORKLOAD_OPT.get(MODEL, dict(lr=1e-3))
    kw = dict(optimizer=rt.OPTIMIZERS[opt.get("optim", "adam")], lr=opt.get("lr", 1e-3),
              momentum=opt.get("momentum", 0.0))
    out = []
    for k in jobs_list:
        sp = ctx.pack(rt.MODELS[MODEL], BATCH, k, warm + timed + 2)
        for jj in range(k):
            sp.load(jj, seed=1000 + jj, steps=warm + timed + 2, **kw)
        sp.run(warm)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sp.run(timed)
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1) / timed
        out.append({"jobs_per_gpu": k, "ms_per_step": t, "samples_per_s": k * BATCH / (t / 1e3)})
        sp.destroy()
    return out


def host_e2e(a, world, ctx, lanes):
    """e2e through the public API with HOST inputs for the ResNet / transformer
    packs: per step, the step's input blob (tokens, or bf16 images + labels)
    is copied from pinned host memory, the step runs, and the per-lane losses
    come back to the host (tlk_step_host_blob)."""
    import numpy as np
    import torch

    from paper_2410_22254_b200 import runtime as rt

    steps = max(3, min(a.steps, 10))
    opt = WORKLOAD_OPT.get(MODEL, dict(lr=1e-3))
    kw = dict(optimizer=rt.OPTIMIZERS[opt.get("optim", "adam")], lr=opt.get("lr", 1e-3),
              momentum=opt.get("momentum", 0.0))
    hp = ctx.pack(rt.MODELS[MODEL], BATCH, lanes, steps + 4, host_input=True)
    for j in range(lanes):
        hp.load(j, seed=2000 + j, steps=steps + 4, **kw)
    nb = hp.host_input_bytes()
    g = np.random.default_rng(0)
    if MODEL in GPT_CFG:
        V = GPT_CFG[MODEL][4]
        host = torch.from_numpy(g.integers(0, V, nb // 4, dtype=np.int32)).pin_memory().numpy().view(np.uint8)
    else:
        n_img = lanes * BATCH * 3072
        img = (g.standard_normal(n_img).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        lab = g.integers(0, 10, lanes * BATCH, dtype=np.int32)
        host = torch.from_numpy(np.concatenate([img.view(np.uint8), lab.view(np.uint8)])).pin_memory().numpy()
    assert host.nbytes == nb
    losses = torch.empty(lanes, dtype=torch.float32).pin_memory().numpy()
    for _ in range(2):
        hp.step_host_blob(host, losses)
    barrier(world)
    t0 = time.perf_counter()
    seen = []
    for _ in range(steps):
        hp.step_host_blob(host, losses)
        seen.append(float(losses[0]))
    e2e_s = dist_max(time.perf_counter() - t0, world)
    assert all(math.isfinite(v) for v in seen)
    hp.destroy()
    return {"value": world * lanes * BATCH * steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nb,
            "d2h_bytes_per_step": lanes * 4, "steps": steps,
            "api": "paper_2410_22254_b200.runtime.Pack.step_host_blob -> tlk_step_host_blob (pinned host blob H2D, "
                   "one packed step, per-lane losses D2H, every step)"}


def _finish_gpt_line(a, world, rank, ctx, pack, value, ms_step, clocks, roof, t_roof, sflops,
                     sbytes, lanes, kernels_out):
    T = GPT_CFG[MODEL][3] if MODEL in GPT_CFG else None
    pack.destroy()
    e2e = host_e2e(a, world, ctx, lanes)
    line = {
        "metric": METRIC, "value": value, "n_gpus": world,
        "unit": "samples/s (sequences)" if T else "samples/s (images)",
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic (on-device order-1 Markov-chain tokens; random-init weights)" if T else
                 "synthetic (on-device ~N(0,1) 3x32x32 images, int4-teacher labels; random-init weights)"),
        "config": {"workload": WORKLOAD, "jobs_per_gpu": lanes, "batch_per_job": BATCH,
                   "optimizer": "sgd momentum 0.9" if MODEL == "resnet18" else "adam",
                   **({"tokens_per_s": value * T} if T else {})},
        "e2e": e2e, "gpu_launches": None, "clocks": clocks,
        "roofline": roof,
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "measured_ms": ms_step,
                          "frac": t_roof * 1e3 / ms_step, "flops_per_step": sflops,
                          "compulsory_bytes_per_step": sbytes},
        "kernels": kernels_out,
    }
    line["gpu_launches"] = LAUNCHES_PER_STEP * a.steps
    if rank == 0 and world == 1 and a.sweep:
        import torch

        stream = torch.cuda.ExternalStream(ctx.stream_handle)
        line["nppn_sweep"] = nppn_sweep(ctx, stream, (1, 2, 4, 8, 16) if MODEL != "xformer" else (1, 4, 16, 32),
                                        3, 5)
    if rank == 0 and world == 1 and not a.no_baselines:
        # CPU path: the numpy oracle jobs on the host cores, a small fixed
        # sample (2 timed steps at a reduced per-job batch; samples/s scale
        # linearly in the batch for these dense models)
        cb = 4 if T else 16
        launcher, lname = reference_launcher()
        cpu, cores, _ = cpu_oracle_rate(2, 1, jobs=min(lanes, 4), batch=cb, launcher=launcher)
        ncpu, aff = host_cores()
        line["cpu_baseline"] = {
            "value": cpu, "unit": line["unit"], "cores": cores, "kind": "port", "host_cpu_count": ncpu,
            "affinity_cpus": aff,
            "sample": f"{min(lanes, 4)} {MODEL} jobs x 2 timed steps (+1 warm-up) at batch {cb}, numpy oracle, "
                      f"concurrent processes via {lname}"}
        kp, outs = kproc_rate(min(lanes, 8), duration=a.kproc_seconds, lead=60.0)
        line["kproc_baseline"] = {"value": kp, "unit": "samples/s", "procs": min(lanes, 8),
                                  "mechanism": "PyTorch processes (bf16 autocast) pinned to one GPU via run_plan",
                                  "packed_over_kproc": (value / kp) if kp else None,
                                  "packed_e2e_over_kproc": (e2e["value"] / kp) if kp else None,
                                  "errors": [o for o in outs if "error" in o][:2]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def _plan_run(tasks, nppn, backend, launcher=None, packed_options=None):
    """One run of a task list at triples [1, nppn, 1] on this GPU; returns the RunReport dict."""
    logdir = tempfile.mkdtemp(prefix="tlk_paper_")
    env = dict(os.environ, PYTHONPATH=ROOT)
    if backend == "packed":
        import paper_2410_22254_b200 as mod

        plan = mod.build_plan(tasks, mod.TripleSpec(1, nppn, 1),
                              mod.NodeSpec(cores=os.cpu_count() or 1, gpus=1, gpu_mem_mib=183359))
        rep = mod.run_plan(plan, 0, log_dir=logdir, base_env=env, backend="packed",
                           packed_options=packed_options or {})
    else:
        mod = launcher
        tl = [mod.TaskDef(t.task_id, t.argv) for t in tasks]
        plan = mod.build_plan(tl, mod.TripleSpec(1, nppn, 1),
                              mod.NodeSpec(cores=os.cpu_count() or 1, gpus=1, gpu_mem_mib=183359))
        rep = mod.run_plan(plan, 0, log_dir=logdir, base_env=env)
    return rep.to_json_dict() if hasattr(rep, "to_json_dict") else json.loads(json.dumps(rep, default=vars))


def paper_arm(a):
    """The paper's own metric (RunReport.elapsed_ms, executor.py:187,223-233):
    a Table-I-style list of 24 MNIST-CNN training tasks (T > S) run at NPPN =
    1, 2, 4, 8, 12, 24 on one GPU, end to end through run_plan -- packed
    backend vs the K-process mechanism (the reference launcher spawning one
    PyTorch process per task, CUDA_VISIBLE_DEVICES-pinned, time-sliced).
    Reports elapsed_ms per NPPN, the speedup elapsed(1) / elapsed(k) of each
    series, and packed vs K-process at every NPPN."""
    from paper_2410_22254_b200 import TaskDef
    from paper_2410_22254_b200.jobspec import JobSpec

    jobs, steps, nppns = a.paper_jobs, a.paper_steps, (1, 2, 4, 8, 12, 24)
    launcher, lname = reference_launcher()
    kp = os.path.join(ROOT, "baselines", "kproc_torch.py")
    series = {
        "packed": (lambda i: tuple(JobSpec(model="cnn", seed=i, steps=steps, batch=BATCH).argv(sys.executable)),
                   "packed"),
        "kproc_torch": (lambda i: (sys.executable, kp, "--model", "cnn", "--seed", str(i), "--batch", str(BATCH),
                                   "--steps", str(steps)), "subprocess"),
        "kproc_torch_fast": (lambda i: (sys.executable, kp, "--model", "cnn", "--seed", str(i), "--batch",
                                        str(BATCH), "--steps", str(steps), "--fast", "1"), "subprocess"),
    }
    out = {}
    for name, (argv_fn, backend) in series.items():
        if a.paper_series and name not in a.paper_series.split(","):
            continue
        rows = []
        for k in nppns:
            tasks = [TaskDef(i, argv_fn(i)) for i in range(jobs)]
            d = _plan_run(tasks, k, backend, launcher)
            el = float(d["elapsed_ms"])
            rows.append({"nppn": k, "elapsed_ms": el, "failures": d["failures"],
                         "max_observed_concurrency": d["max_observed_concurrency"],
                         "samples_per_s": jobs * steps * BATCH / (el / 1e3)})
        base = rows[0]["elapsed_ms"]
        for r in rows:
            r["speedup_vs_nppn1"] = base / r["elapsed_ms"]
        out[name] = rows
    cmp = {}
    if "packed" in out:
        for other in ("kproc_torch", "kproc_torch_fast"):
            if other in out:
                cmp[f"packed_over_{other}"] = [{"nppn": p["nppn"], "elapsed_ratio": o["elapsed_ms"] / p["elapsed_ms"]}
                                               for p, o in zip(out["packed"], out[other])]
    top = out.get("packed", next(iter(out.values())))[-1]
    line = {"metric": METRIC, "value": top["samples_per_s"], "unit": UNIT, "n_gpus": 1, "steps": steps,
            "warmup": 0, "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (on-device counter RNG MNIST batches; random-init weights)",
            "config": {"workload": f"paper metric: {jobs} MNIST-CNN tasks x {steps} steps (bs {BATCH}, Adam), "
                                   f"triples [1, NPPN, 1] on 1 GPU, NPPN in {list(nppns)}, end to end through "
                                   f"run_plan (elapsed_ms, executor.py:187,223)",
                       "subprocess_launcher": lname},
            "e2e": {"value": top["samples_per_s"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "api": "run_plan(plan, backend='packed') elapsed_ms (task list in, RunReport out)"},
            "series": out, "comparison": cmp}
    print(json.dumps(line), flush=True)
    return 0


def mix_arm(a):
    """configs[3]: MLP + CNN + 2-layer transformer tasks interleaved, NPPN =
    1..32 jobs on one GPU.  Steady state: one pack per kind (lanes = that
    kind's share of the NPPN slots), each on its own stream, all replayed
    together (what the packed worker runs between refills), timed after a
    warm-up; plus the same task list end to end through run_plan(backend=
    "packed") (elapsed_ms, worker start-up included)."""
    import torch

    from paper_2410_22254_b200 import TaskDef
    from paper_2410_22254_b200 import runtime as rt
    from paper_2410_22254_b200.jobspec import JobSpec

    kinds = (("mlp", 64), ("cnn", 64), ("xformer", 32))
    rows = []
    ctx = rt.Context(0)
    for k in (1, 2, 4, 8, 16, 32):
        counts = {kd: sum(1 for i in range(k) if i % 3 == n) for n, (kd, _) in enumerate(kinds)}
        packs = []
        for kd, bs in kinds:
            if counts[kd]:
                p = ctx.pack(rt.MODELS[kd], bs, counts[kd], 2 * a.mix_steps + 8, flags=rt.PACK_OWN_STREAM)
                for j in range(counts[kd]):
                    p.load(j, seed=j, steps=2 * a.mix_steps + 8)
                packs.append((p, bs))
        for p, _ in packs:
            p.run(3)
        ctx.sync()
        t0 = time.perf_counter()
        for p, _ in packs:
            p.run(a.mix_steps)
        ctx.sync()
        dt = time.perf_counter() - t0
        samples = sum(p.lanes * bs * a.mix_steps for p, bs in packs)
        for p, _ in packs:
            p.destroy()
        rows.append({"nppn": k, "kinds": counts, "steady_samples_per_s": samples / dt,
                     "steady_ms_per_step": dt * 1e3 / a.mix_steps,
                     "steady_job_steps_per_s": sum(p.lanes for p, _ in packs) * a.mix_steps / dt})
    ctx.close()
    # the paper's metric on configs[3]: ONE fixed list of 32 interleaved tasks
    # (MLP, CNN, transformer, ...) run end to end through run_plan at every
    # NPPN (T >= S; queue refill), elapsed_ms and speedup vs NPPN = 1
    ntask = 32
    specs = [JobSpec(model=kinds[i % 3][0], seed=i, steps=a.mix_steps, batch=kinds[i % 3][1]) for i in range(ntask)]
    tasks = [TaskDef(i, tuple(sp.argv(sys.executable))) for i, sp in enumerate(specs)]
    list_samples = sum(a.mix_steps * kinds[i % 3][1] for i in range(ntask))
    fixed = []
    for k in (1, 2, 4, 8, 16, 32):
        d = _plan_run(tasks, k, "packed", packed_options={"chunk": a.mix_steps})
        el = float(d["elapsed_ms"])
        fixed.append({"nppn": k, "elapsed_ms": el, "failures": d["failures"],
                      "max_observed_concurrency": d["max_observed_concurrency"],
                      "samples_per_s": list_samples / (el / 1e3)})
    for r in fixed:
        r["speedup_vs_nppn1"] = fixed[0]["elapsed_ms"] / r["elapsed_ms"]
    top = rows[-1]
    line = {"metric": METRIC, "value": top["steady_samples_per_s"], "unit": "samples/s (images + sequences)",
            "n_gpus": 1, "steps": a.mix_steps, "warmup": 3, "ms_per_step": top["steady_ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (on-device generators)",
            "config": {"workload": "configs[3]: MLP (bs 64) + CNN (bs 64) + transformer (2L d256 T128, bs 32) tasks "
                                   "interleaved, NPPN 1..32 on 1 GPU; one pack + stream per kind"},
            "e2e": {"value": fixed[-1]["samples_per_s"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0,
                    "api": f"run_plan(plan, backend='packed') elapsed_ms, fixed list of {ntask} tasks at NPPN 32"},
            "nppn_sweep": rows, "fixed_list": {"tasks": ntask, "steps_per_task": a.mix_steps, "rows": fixed}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("packed", "reference"), default="packed")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["paper24", "mix"], default="cnn",
                    help="default cnn = configs[1] (the driver's line); paper24 = the paper's elapsed-time "
                         "speedup over a 24-task list; mix = configs[3]")
    ap.add_argument("--paper-jobs", type=int, default=24)
    ap.add_argument("--paper-steps", type=int, default=938, help="steps per task (938 = one MNIST epoch at bs 64)")
    ap.add_argument("--paper-series", default="", help="comma list of packed,kproc_torch,kproc_torch_fast")
    ap.add_argument("--mix-steps", type=int, default=300)
    ap.add_argument("--jobs", type=int, default=None, help="co-resident jobs per GPU")
    ap.add_argument("--profile-iters", type=int, default=5)
    ap.add_argument("--kproc-seconds", type=float, default=10.0)
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-sweep", dest="sweep", action="store_false",
                    help="skip the jobs/GPU sweep (packed throughput at 1..32 jobs per GPU)")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    global MODEL, BATCH, JOBS_PER_GPU, WORKLOAD
    if a.workload == "paper24":
        return paper_arm(a)
    if a.workload == "mix":
        return mix_arm(a)
    MODEL, BATCH, JOBS_PER_GPU, WORKLOAD = WORKLOADS[a.workload]
    if a.jobs is None:
        a.jobs = JOBS_PER_GPU
    JOBS_PER_GPU = a.jobs
    world, rank, local = dist_setup(a.gpus)
    try:
        if a.impl == "reference":
            return reference_arm(a, world, rank)
        return packed_arm(a, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
