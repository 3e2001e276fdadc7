import sys, os
sys.path.insert(0, os.getcwd())
from paper_2410_22254_b200 import runtime as rt
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 1
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_MLP, 64, lanes, 4)
    print("packed", flush=True)
    for j in range(lanes):
        p.load(j, seed=j, steps=4)
    ctx.sync()
    print("loaded", flush=True)
    p.run(1)
    print("run issued", flush=True)
    ctx.sync()
    print("losses", [p.losses(j, 1).tolist() for j in range(lanes)], flush=True)
    p.run(2)
    ctx.sync()
    print("losses", [p.losses(j, 3).tolist() for j in range(lanes)], flush=True)
