"""TMA-staged dense GEMM epilogues (sgemm.cuh `EpiOps::tile_tma`, default)
against the per-element transpose epilogues (`TLK_TMA_EPI=0`).

Both compute the same per-element FMA chains (the TMA path on f32x2 pairs,
which round per lane exactly like the scalar ops), so the forward -- every
loss of the first step -- is bit-identical.  The backward differs only in
summation order: bias-gradient column partials (rows summed per column pair
instead of per 4-column group) and, with fused attention, the softmax-
backward row term D taken from the proj-dgrad epilogue (two accumulators per
head instead of one).  Those feed bf16 roundings of dS, so first-step
gradients agree to GRAD_TOL rel-L2 and short loss curves to LOSS_TOL.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_22254_b200 import runtime as rt
model, lanes, batch, steps, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODELS[model], batch, lanes, steps + 1)
    for j in range(lanes):
        p.load(j, seed=11 + j, steps=steps + 1, lr=3e-3)
    p.run(1)
    ctx.sync()
    g = p.tensor(rt.BUF_GRADS).cpu().numpy()
    p.run(steps - 1)
    ctx.sync()
    np.savez(out, loss=np.array([p.losses(j, steps) for j in range(lanes)]), g=g)
""" % ROOT
GRAD_TOL = 1e-2
LOSS_TOL = 2e-3


def _run(model, lanes, batch, steps, tma):
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "o.npz")
        r = subprocess.run([sys.executable, "-c", CODE, model, str(lanes), str(batch), str(steps), f],
                           capture_output=True, text=True, timeout=900, env=dict(os.environ, TLK_TMA_EPI=tma))
        assert r.returncode == 0, r.stderr[-3000:]
        return dict(np.load(f))


@pytest.mark.parametrize("model,lanes,batch", [("gpt", 2, 8), ("xformer", 3, 8)])
def test_tma_epilogue_matches_per_element(model, lanes, batch):
    a, b = _run(model, lanes, batch, 4, "0"), _run(model, lanes, batch, 4, "1")
    assert np.array_equal(a["loss"][:, 0], b["loss"][:, 0])  # forward: bit-identical
    assert np.all(np.isfinite(b["g"]))
    for j in range(lanes):
        ga, gb = a["g"].reshape(lanes, -1)[j], b["g"].reshape(lanes, -1)[j]
        assert np.linalg.norm(ga - gb) <= GRAD_TOL * np.linalg.norm(ga), j
    assert np.all(np.abs(a["loss"] - b["loss"]) <= LOSS_TOL * np.maximum(1.0, np.abs(a["loss"])))
