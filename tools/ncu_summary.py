"""Summarise ncu reports (--page raw) into a compact table for profiles/."""
import csv, io, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__t_bytes.sum", "l1_bytes"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")][:70]}
        for m, short in METRICS:
            for cand in (m, m.replace("sm__pipe_tensor_cycles_active", "sm__pipe_tensor_op_hmma_cycles_active")):
                if cand in hdr:
                    d[short] = f"{v[hdr.index(cand)]} {units[hdr.index(cand)]}".strip()
                    break
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarize(p):
            print(p.split("/")[-1], " | ".join(f"{k}={v}" for k, v in d.items()))
