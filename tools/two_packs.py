"""Throughput of 8 CNN lanes as ONE pack vs TWO 4-lane packs on their own
streams (lane groups overlapping on the device)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt

mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
flags = 0 if mode == "graph" else rt.PACK_PERSISTENT
with rt.Context(0) as ctx:
    one = ctx.pack(rt.MODEL_CNN, 64, 8, 400, flags=flags)
    halves = [ctx.pack(rt.MODEL_CNN, 64, 4, 400, flags=flags | rt.PACK_OWN_STREAM) for _ in range(2)]
    for p in [one] + halves:
        for j in range(p.lanes):
            p.load(j, seed=j, steps=400)
    for p in [one] + halves:
        p.run(5)
    ctx.sync()
    t0 = time.perf_counter()
    one.run(100)
    ctx.sync()
    t1 = time.perf_counter()
    for p in halves:
        p.run(100)
    ctx.sync()
    t2 = time.perf_counter()
    print(mode, "one pack of 8: %.1f us/step; two packs of 4 concurrently: %.1f us/step" % ((t1 - t0) * 1e4, (t2 - t1) * 1e4))
