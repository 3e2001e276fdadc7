"""Timestamps inside persistent-kernel items (TLK_PERSIST_PROBE=1), 1 launch.
    python tools/persist_probe.py LANES STEPS"""
import os, sys
os.environ["TLK_PERSIST_PROBE"] = "1"
import numpy as np
sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt

PH = ["C1F", "C2F", "F1F", "HR", "HD", "F1D", "C2D", "C2W", "FWA", "C1W", "OPT"]
lanes, steps = int(sys.argv[1]), int(sys.argv[2])
B = 64
n = [B, 36, 18, 8, 1, 72, 36, 18, 72, B, 36]
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_CNN, B, lanes, 10 + steps, flags=rt.PACK_PERSISTENT)
    for j in range(lanes):
        p.load(j, seed=j, steps=10 + steps)
    p.run(3)
    ctx.sync()
    p.run(steps)
    ctx.sync()
    pr = p.named("persist.probe", "f4").cpu().numpy().view(np.uint64)
per = sum(n) * lanes
tot = per * steps
pr = pr[: tot * 16].reshape(tot, 16).astype(np.int64)
ph = np.zeros(tot, int)
for i in range(tot):
    s, r = divmod(i, per)
    for k in range(len(PH)):
        m = lanes * n[k]
        if r < m:
            ph[i] = k
            break
        r -= m
for k in (PH.index("C2W"), PH.index("FWA"), PH.index("HD"), PH.index("C2F"), PH.index("F1D")):
    m = np.where(ph == k)[0]
    rows = pr[m]
    st = rows[:, 13:14]
    rel = np.where(rows > 0, (rows - st) / 1000.0, np.nan)
    print(PH[k], "probe k: mean us after item start (k=13), n =", len(m))
    print("  ", " ".join(f"{kk}:{np.nanmean(rel[:, kk]):.1f}" for kk in range(16) if np.isfinite(np.nanmean(rel[:, kk]))))
