"""Per-tensor rel-L2 gradient error of the ResNet pack vs the oracle (1 step)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import resnet as orn  # noqa: E402
from paper_2410_22254_b200 import runtime as rt  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_RESNET18, B, 1, 1)
    p.load(0, seed=50, steps=1, optimizer=rt.OPT_SGD, lr=0.01)
    p.run(1)
    ctx.sync()
    G = p.tensor(rt.BUF_GRADS).cpu().numpy()
    x, y = orn.batch(50, 0, B)
    loss, g = orn.resnet_step(orn.init_params(50), x, y, bf16=True)
    print("loss gpu", p.losses(0, 1)[0], "oracle", loss)
    for name, shape, off in orn.layout()[0]:
        n = int(np.prod(shape))
        a, b = G[off:off + n], g[name].reshape(-1)
        print(f"{name:16s} rel {np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.4f}  "
              f"|gpu| {np.linalg.norm(a):.4e} |ref| {np.linalg.norm(b):.4e}")
