"""ms/step of the CNN pack, kernel graph vs the persistent scheduler kernel,
over lane counts: python tools/persist_vs_graph.py [lanes ...]"""
import sys
import time

sys.path.insert(0, ".")
from paper_2410_22254_b200 import runtime as rt  # noqa: E402

lanes_list = [int(x) for x in sys.argv[1:]] or [1, 8, 16, 32, 64]
with rt.Context(0) as ctx:
    for lanes in lanes_list:
        row = []
        for flags in (0, rt.PACK_PERSISTENT):
            p = ctx.pack(rt.MODEL_CNN, 64, lanes, 200, flags=flags)
            for j in range(lanes):
                p.load(j, seed=j, steps=200)
            p.run(10)
            ctx.sync()
            t0 = time.perf_counter()
            p.run(100)
            ctx.sync()
            row.append((time.perf_counter() - t0) * 10.0)
            p.destroy()
        print(f"lanes {lanes:3d}: graph {row[0]:.3f} ms/step, persistent {row[1]:.3f} ms/step", flush=True)
