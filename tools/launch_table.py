"""Per-kernel table (launches, mean us, share, achieved DRAM GB/s) of an ncu
--csv launch list (gpu__time_duration.sum [+ dram__bytes_read/write.sum])."""
import collections
import csv
import sys


def table(path, skip_first=0):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in list(per.items())[skip_first:]:
        n = names[i].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:48]
        a = agg[n]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':50s} {'n':>4s} {'mean_us':>9s} {'share':>6s} {'GB/s':>8s}"]
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:50s} {a[0]:4d} {a[1] / a[0] / 1e3:9.2f} {100 * a[1] / tot:5.1f}% {a[2] / a[1] if a[1] else 0:8.1f}")
    out.append(f"total {tot / 1e3:.1f} us")
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0))
