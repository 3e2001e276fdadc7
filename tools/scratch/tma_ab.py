"""A/B of the TMA-staged GEMM epilogue (TLK_TMA_EPI=1) vs the per-element one:
first-step losses and gradients of a pack, compared element-wise."""
import json, os, subprocess, sys, tempfile
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_22254_b200 import runtime as rt
model, lanes, batch, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODELS[model], batch, lanes, 2)
    for j in range(lanes):
        p.load(j, seed=11 + j, steps=2, lr=3e-3)
    p.run(1)
    ctx.sync()
    np.savez(out, loss=np.array([p.losses(j, 1) for j in range(lanes)]), g=p.tensor(rt.BUF_GRADS).cpu().numpy())
""" % ROOT
for model, lanes, batch in [("gpt", 2, 8), ("xformer", 3, 8)]:
    res = {}
    with tempfile.TemporaryDirectory() as d:
        for v in ("0", "1"):
            f = os.path.join(d, v + ".npz")
            r = subprocess.run([sys.executable, "-c", CODE, model, str(lanes), str(batch), f], capture_output=True,
                               text=True, env=dict(os.environ, TLK_TMA_EPI=v), timeout=600)
            if r.returncode:
                print(model, v, "FAILED", r.stderr[-2000:])
                break
            res[v] = dict(np.load(f))
    if len(res) < 2:
        continue
    a, b = res["0"], res["1"]
    ga, gb = a["g"].ravel(), b["g"].ravel()
    print(model, "loss equal", np.array_equal(a["loss"], b["loss"]), a["loss"].ravel()[:3], b["loss"].ravel()[:3],
          "grad elems equal %.6f" % np.mean(ga == gb), "rel-L2 %.3e" % (np.linalg.norm(ga - gb) / np.linalg.norm(ga)),
          "nan", np.isnan(gb).sum())
