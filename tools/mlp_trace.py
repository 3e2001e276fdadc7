"""Phase timeline of the MLP step kernel (cluster of lane 0, clock64 cycles): python tools/mlp_trace.py [lanes]"""
import os
import sys

os.environ["TLK_MLP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2410_22254_b200 import runtime as rt  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 4
NAMES = {0: "start", 1: "inputs+sync", 2: "M:fc1 issued", 3: "M:h1 all", 4: "M:fc2 issued", 5: "M:dz2 all",
         6: "M:dgrad issued", 7: "labels", 8: "E:fc1 done", 9: "E:h1 sent", 10: "E:fc2 done", 11: "E:plog sent",
         12: "E:plog all", 13: "E:dz2 sent", 14: "E:dgrad done", 15: "end", 16: "cluster exit",
         17: "cluster.sync", 18: "teacher", 19: "words done",
         **{20 + i: f"M:w1 tile {i}" for i in range(12)}}
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_MLP, 64, lanes, 8)
    for j in range(lanes):
        p.load(j, seed=j, steps=8)
    p.run(5)
    ctx.sync()
    tr = p.named("mlp.trace", "f4").cpu().numpy().view(np.uint64).astype(np.int64).reshape(4, 32)
t0 = tr[tr > 0].min()
for k in sorted(NAMES):
    print(f"{NAMES[k]:>15s} " + " ".join(f"{(tr[c, k] - t0) if tr[c, k] else -1:8d}" for c in range(4)))
