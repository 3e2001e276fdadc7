"""One warm-up launch + one measured launch of the CNN pack (for ncu captures).
    python tools/persist_run.py LANES STEPS [graph]"""
import sys
sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt

lanes, steps = int(sys.argv[1]), int(sys.argv[2])
flags = 0 if len(sys.argv) > 3 and sys.argv[3] == "graph" else rt.PACK_PERSISTENT
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_CNN, 64, lanes, 4 * steps + 4, flags=flags)
    for j in range(lanes):
        p.load(j, seed=j, steps=4 * steps + 4)
    p.run(steps)
    ctx.sync()
    p.run(steps)
    ctx.sync()
print("ok")
