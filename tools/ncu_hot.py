"""Top stall sites of one ncu report (source page, SASS): python tools/ncu_hot.py rep.ncu-rep [n]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))[1:]
h, data = rows[0], rows[1:]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
tot = sum(int(r[iS] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
order = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:n]
for i in sorted(order):
    ctx = " | ".join(data[j][iSrc].strip()[:40] for j in range(max(0, i - 2), i))
    print(f"{int(data[i][iS]):6d} {int(data[i][iE] or 0):9d} {data[i][0][-5:]} {data[i][iSrc].strip()[:60]:60s}  <- {ctx}")
