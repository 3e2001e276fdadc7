"""Same ResNet step with the tap-group wgrad / halo convs on and off: every
weight gradient must agree to fp32 summation-order noise (run on the GPU)."""
import os
import numpy as np
from paper_2410_22254_b200 import runtime as rt
from oracle import resnet as orn


def run(env):
    os.environ.update(env)
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_RESNET18, 16, 1, 1, flags=rt.PACK_SNAPSHOTS)
        p.load(0, seed=60, steps=1, optimizer=rt.OPT_SGD, lr=0.02, momentum=0.9)
        p.run(1)
        ctx.sync()
        return p.tensor(rt.BUF_GRADS).cpu().numpy()[:p.info.param_stride].copy()


base = run({"TLK_NO_TAPGROUP": "1", "TLK_NO_HALO": "1"})
tg = run({"TLK_NO_TAPGROUP": "0", "TLK_NO_HALO": "1"})
both = run({"TLK_NO_TAPGROUP": "0", "TLK_NO_HALO": "0"})
lay, _, _ = orn.layout()
for name, shape, off in lay:
    n = int(np.prod(shape))
    b = base[off:off + n]
    nb = np.linalg.norm(b) + 1e-30
    r1 = np.linalg.norm(tg[off:off + n] - b) / nb
    r2 = np.linalg.norm(both[off:off + n] - b) / nb
    if name.endswith(".w"):
        print(f"{name:16s} tg {r1:.2e}  halo+tg {r2:.2e}")
