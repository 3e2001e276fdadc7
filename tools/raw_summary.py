"""Summarise ncu --page raw --csv exports (one kernel each) into a table."""
import csv
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        d = {}
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[short] = f"{v[i]} {units[i]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarize(p):
            print(p.split("/")[-1].replace("raw_", "").replace(".csv", ""), "|",
                  " | ".join(f"{k}={v}" for k, v in d.items()))
