"""Summarise tools/profile_round.sh outputs (gpurun_out/) into profiles/<tag>_*.

usage: python tools/make_round_profiles.py <tag>
  profiles/<tag>_bench_<workload>.json   bench lines (driver contract)
  profiles/<tag>_launches_<workload>.txt per-kernel device time / DRAM GB/s
  profiles/<tag>_ncu_full.txt            --set full summaries of the top kernels
  profiles/traffic.json                  DRAM bytes per launch of the dominant kernels
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_table import table  # noqa: E402
from raw_summary import summarize  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
# capture name -> (model, bench.py kernel label)
CAPS = {"c_fc1_wgrad_adam": ("cnn", "fc1_wgrad_adam"), "c_conv2_fwd": ("cnn", "conv2_fwd_pool"),
        "c_conv2_dgrad": ("cnn", "conv2_dgrad"),
        "c_conv2_wgrad": ("cnn", "conv2_wgrad"), "c_fc1_dgrad": ("cnn", "fc1_dgrad_unpool"),
        "c_cnn_opt": ("cnn", "grad_finalize_opt"), "c_conv1_wgrad": ("cnn", "conv1_wgrad"),
        "c_conv1_fwd": ("cnn", "inputs_conv1_fwd"), "c_cnn_head": ("cnn", "fc1_reduce_head"), "r_fwd_l1_halo": ("resnet18", "conv_fwd"),
        "r_dgrad_l1_halo": ("resnet18", "conv_dgrad"), "r_wgrad_l1_tg": ("resnet18", "conv_wgrad"),
        "r_dgrad_bn256": ("resnet18", "conv_dgrad_bn256"), "r_bn_bwd_apply": ("resnet18", "bn_bwd_apply"),
        "g_scores": ("gpt", "attn_scores"), "g_fc": ("gpt", "fc")}


def main(tag):
    for w in ("cnn", "mlp", "resnet18", "xformer", "gpt", "mix", "reference"):
        f = os.path.join(OUT, f"bench_{w}.json")
        if os.path.exists(f) and os.path.getsize(f):
            try:
                d = json.loads(open(f).read())
            except ValueError:
                continue
            json.dump(d, open(os.path.join(PROF, f"{tag}_bench_{w}.json"), "w"), indent=1)
    for w, how in (("cnn", "bench.py --steps 3 --warmup 3 (10 kernels per step; lane_init_kernel is setup)"),
                   ("resnet18", "tools/pack_step.py resnet18 8 128 1"), ("gpt", "tools/pack_step.py gpt 16 64 1"),
                   ("mlp", "tools/pack_step.py mlp 4 64 1"), ("xformer", "tools/pack_step.py xformer 32 32 1")):
        f = os.path.join(OUT, f"launches_{w}.csv")
        if os.path.exists(f):
            hdr = (f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   f"--clock-control none (cold-cache, serialised); {how}\n")
            open(os.path.join(PROF, f"{tag}_launches_{w}.txt"), "w").write(hdr + table(f) + "\n")
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lines = [f"# ncu --set full --clock-control none, one launch each (tools/profile_round.sh, tag {tag})"]
    for name, (model, label) in CAPS.items():
        f = os.path.join(OUT, f"raw_{name}.csv")
        if not os.path.exists(f) or os.path.getsize(f) < 100:
            continue
        for d in summarize(f):
            lines.append(f"{name} ({model}/{label}) | " + " | ".join(f"{k}={v}" for k, v in d.items()))

            def mb(s):
                v, u = s.split()
                return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            if "dram_rd" in d and "dram_wr" in d:
                traffic.setdefault(model, {})[label] = {"dram_bytes": mb(d["dram_rd"]) + mb(d["dram_wr"]),
                                                        "source": f"profiles/{tag}_ncu_full.txt"}
    open(os.path.join(PROF, f"{tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
