"""Run a few steps of a pack (ncu captures): python tools/pack_step.py <model> <lanes> <batch> <steps> [opt]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_22254_b200 import runtime as rt  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "gpt"
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 16
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 64
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
ctx = rt.Context(0)
pack = ctx.pack(rt.MODELS[model], batch, lanes, steps + 1)
opt = dict(optimizer=rt.OPT_SGD, lr=0.05, momentum=0.9) if model == "resnet18" else {}
for j in range(lanes):
    pack.load(j, seed=j, steps=steps + 1, **opt)
pack.run(steps)
ctx.sync()
print("ok", [pack.losses(j, steps).tolist() for j in range(min(2, lanes))])
