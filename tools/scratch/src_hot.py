"""Top SASS lines by warp-stall samples from an ncu --page source --csv export."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ci = hdr.index("Warp Stall Sampling (All Samples)")
    stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[ci]), r))
        except (ValueError, IndexError):
            pass
    tot = sum(v for v, _ in data) or 1
    print("==", path.split("/")[-1], "samples", int(tot))
    for v, r in sorted(data, key=lambda x: -x[0])[:12]:
        top = sorted(((float(r[i] or 0), hdr[i]) for i in stalls), reverse=True)[:2]
        print(f"{100 * v / tot:5.1f}%  {r[1].strip()[:60]:60s} {top}")
