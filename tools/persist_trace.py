"""Per-item timeline of the CNN persistent scheduler kernel (TLK_PERSIST_TRACE=1).

    python tools/persist_trace.py LANES STEPS OUT.npz
Records [fetched, deps ready, started, ended] per queue item of one launch of
STEPS steps (after a warm-up launch) and prints per-phase summaries."""
import os, sys
os.environ["TLK_PERSIST_TRACE"] = "1"
import numpy as np
sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt

PH = ["C1F", "C2F", "F1F", "HR", "HD", "F1D", "C2D", "C2W", "FWA", "C1W", "OPT"]
lanes, steps = int(sys.argv[1]), int(sys.argv[2])
out = sys.argv[3] if len(sys.argv) > 3 else None
B = 64
n = [B, 36, 18, 8, 1, 72, 36, 18, 72, B, 36]
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_CNN, B, lanes, 10 + steps, flags=rt.PACK_PERSISTENT)
    for j in range(lanes):
        p.load(j, seed=j, steps=10 + steps)
    p.run(5)
    ctx.sync()
    p.run(steps)
    ctx.sync()
    tr = p.named("persist.trace", "f4").cpu().numpy().view(np.uint64)
per = sum(n) * lanes
tot = per * steps
tr = tr[: tot * 5].reshape(tot, 5).astype(np.int64)
sm = tr[:, 4]
t = tr[:, :4]
t0 = t[:, 0].min()
t = (t - t0) / 1000.0  # us
ph = np.zeros(tot, int); lane = np.zeros(tot, int); step = np.zeros(tot, int)
for i in range(tot):
    s, r = divmod(i, per)
    for k in range(len(PH)):
        m = lanes * n[k]
        if r < m:
            ph[i], lane[i], step[i] = k, r // n[k], s
            break
        r -= m
span = t[:, 3].max()
print(f"lanes {lanes} steps {steps}: launch span {span:.1f} us = {span / steps:.1f} us/step")
work = t[:, 3] - t[:, 2]
dep = t[:, 1] - t[:, 0]
gap = t[:, 2] - t[:, 1]
print(f"{'phase':5s} {'items':>6s} {'work_us':>8s} {'sum_work':>9s} {'depwait':>8s} {'gap':>7s}")
for k, name in enumerate(PH):
    m = ph == k
    print(f"{name:5s} {m.sum():6d} {work[m].mean():8.2f} {work[m].sum():9.1f} {dep[m].mean():8.2f} {gap[m].mean():7.2f}")
busy = np.zeros(sm.max() + 1)
for i in range(tot):
    busy[sm[i]] += work[i]
print(f"group busy fraction: mean {busy[busy > 0].mean() / span:.3f} over {int((busy > 0).sum())} groups")
for s in range(min(steps, 3)):
    for j in range(min(lanes, 2)):
        row = []
        for k, name in enumerate(PH):
            m = (ph == k) & (lane == j) & (step == s)
            row.append(f"{name}:{t[m, 2].min():.0f}-{t[m, 3].max():.0f}")
        print(f"step {s} lane {j}: " + " ".join(row))
if out:
    np.savez(out, t=t, sm=sm, ph=ph, lane=lane, step=step)
