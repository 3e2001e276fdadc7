"""Turn gpurun_out/ ncu artefacts into the tracked summaries under profiles/.

usage: python tools/make_profiles.py <tag> [model]   (e.g. r1 cnn)
writes profiles/<tag>_launches.txt, profiles/<tag>_ncu.txt, profiles/traffic.json
"""
import collections, csv, json, os, re, sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarize  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
# ncu kernel name fragment -> bench.py kernel label
LABELS = {"conv2_tc_kernel<1>": "conv2_fwd_pool", "conv2_tc_kernel<0>": "conv2_dgrad",
          "Fc1WgradOpt": "fc1_wgrad_adam", "Conv2Fwd": "conv2_fwd_pool", "Conv2Dgrad": "conv2_dgrad", "conv2_wgrad_tc": "conv2_wgrad", "conv2_fwd_tc": "conv2_fwd_pool", "conv2_dgrad_tc": "conv2_dgrad",
          "Fc1Dgrad": "fc1_dgrad_unpool", "Fc1Fwd": "fc1_fwd_splitk", "LinWgrad": "fc1_wgrad",
          "optimizer_kernel": "optimizer", "conv1_wgrad": "conv1_wgrad", "conv1_fwd": "inputs_conv1_fwd",
          "head_kernel": "head", "inputs_kernel": "inputs", "cnn_opt": "grad_finalize_opt",
          "fc1_reduce": "fc1_reduce", "end_step": "end_step"}


def label(name):
    for k, v in LABELS.items():
        if k in name:
            return v
    return name.split("(")[0]


def launches(tag):
    lines = open(os.path.join(OUT, "launches.csv")).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    agg = collections.defaultdict(list)
    for r in csv.DictReader(lines[i:]):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        agg[label(r["Kernel Name"])].append(float(r["Metric Value"]) / 1000)
    agg.pop("lane_init_kernel", None)
    tot = sum(sum(v) for v in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)",
           f"# bench.py --steps 3 --warmup 3 --no-baselines ; per-step kernel shares",
           f"{'kernel':24s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:24s} {len(v):8d} {sum(v)/len(v):9.2f} {100*sum(v)/tot:6.1f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(tag, model="cnn"):
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    per_model = traffic.setdefault(model, {})
    lines = ["# ncu --set full --clock-control none, one launch per kernel (bench CNN pack, 8 lanes)"]
    for f in sorted(os.listdir(OUT)):
        if not f.endswith(".ncu-rep"):
            continue
        for d in summarize(os.path.join(OUT, f)):
            lines.append(" | ".join(f"{k}={v}" for k, v in d.items()))
            def mb(s):
                v, u = s.split()
                return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            if "dram_rd" in d and "dram_wr" in d:
                per_model[label(d["kernel"])] = {"dram_bytes": mb(d["dram_rd"]) + mb(d["dram_wr"]),
                                               "source": f"profiles/{tag}_ncu.txt"}
    open(os.path.join(PROF, f"{tag}_ncu.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    full(tag, sys.argv[2] if len(sys.argv) > 2 else "cnn")
