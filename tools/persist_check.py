"""Quick A/B of the CNN persistent scheduler kernel vs the per-phase graph path
(bit-identical losses / params) and their step times.  Used under gpurun."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
with rt.Context(0) as ctx:
    packs = {}
    for name, flags in (("graph", 0), ("persist", rt.PACK_PERSISTENT)):
        p = ctx.pack(rt.MODEL_CNN, 64, lanes, steps + 60, flags=flags)
        for j in range(lanes):
            p.load(j, seed=11 + j, steps=steps + 60, optimizer=rt.OPT_ADAM if j % 2 == 0 else rt.OPT_SGD,
                   lr=1e-3 if j % 2 == 0 else 0.02, momentum=0.0 if j % 2 == 0 else 0.9)
        t0 = time.perf_counter()
        p.run(steps)
        ctx.sync()
        print(name, "first run s", time.perf_counter() - t0, flush=True)
        packs[name] = p
    for j in range(lanes):
        a, b = packs["graph"].losses(j, steps), packs["persist"].losses(j, steps)
        pa, pb = packs["graph"].params(j), packs["persist"].params(j)
        print("lane", j, "loss eq", np.array_equal(a, b), a[:3], b[:3], "params eq", np.array_equal(pa, pb),
              "maxdiff", float(np.abs(pa - pb).max()), flush=True)
    for name, p in packs.items():
        st = torch.cuda.ExternalStream(ctx.stream_handle)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        p.run(40)
        e1.record(st)
        e1.synchronize()
        print(name, "ms/step", e0.elapsed_time(e1) / 40, flush=True)
