"""Fused causal attention (csrc/attn.cuh) against the unfused P / dS GEMM chain.

The fused kernels restate the unfused path operation for operation (same SFU
exponentials, P and dS rounded to bf16 at the same points, the same ascending
k-order of every product); only the softmax row sum is added in a different
order (four column quarters with four accumulators each, instead of two
sequential halves).  So a run with TLK_ATTN_FUSED=0 and one with the fused
kernels agree to fp32 rounding: first-step gradients within GRAD_TOL rel-L2
(rare 1-ulp bf16 flips of P), loss curves within LOSS_TOL, at T = 256
(tiny-GPT layout: the causal off-diagonal tile and the diagonal masks) and
T = 128 (configs[3]'s transformer).  The oracle comparisons of the fused path
itself are the GPT tests (tests/test_gpu_gpt.py, test_gpu_baseline_shapes.py),
which run it by default.
"""
import json
import os
import tempfile
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
from paper_2410_22254_b200 import runtime as rt
model, lanes, batch, steps, cfg = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), json.loads(sys.argv[5])
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODELS[model], batch, lanes, steps, **cfg)
    for j in range(lanes):
        p.load(j, seed=300 + j, steps=steps, lr=3e-3)
    p.run(steps)
    ctx.sync()
    out = {"losses": [p.losses(j, steps).tolist() for j in range(lanes)],
           "params": [hashlib.sha256(p.params(j).tobytes()).hexdigest() for j in range(lanes)],
           "grads": hashlib.sha256(p.tensor(rt.BUF_GRADS).cpu().numpy().tobytes()).hexdigest()}
    if len(sys.argv) > 6:
        import numpy as np
        np.save(sys.argv[6], p.tensor(rt.BUF_GRADS).cpu().numpy())
    print(json.dumps(out))
""" % ROOT


GRAD_TOL = 1e-2
LOSS_TOL = 2e-3


def _run(env, model, lanes, batch, steps, cfg, save=None):
    extra = [save] if save else []
    out = subprocess.run([sys.executable, "-c", CODE, model, str(lanes), str(batch), str(steps), json.dumps(cfg),
                          *extra],
                         capture_output=True, text=True, env=dict(os.environ, **env), timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("model,lanes,batch,cfg", [
    ("gpt", 3, 4, dict(layers=2, d_model=128, heads=2, seq_len=256, vocab=65)),
    ("gpt", 2, 2, dict(layers=1, d_model=384, heads=6, seq_len=256, vocab=65)),
    ("xformer", 3, 8, {}),
])
def test_fused_attention_matches_unfused(model, lanes, batch, cfg):
    with tempfile.TemporaryDirectory() as d:
        f1 = _run({"TLK_ATTN_FUSED": "1"}, model, lanes, batch, 1, cfg, os.path.join(d, "f.npy"))
        f0 = _run({"TLK_ATTN_FUSED": "0"}, model, lanes, batch, 1, cfg, os.path.join(d, "u.npy"))
        g1, g0 = np.load(os.path.join(d, "f.npy")), np.load(os.path.join(d, "u.npy"))
    l1, l0 = np.array(f1["losses"]), np.array(f0["losses"])
    assert np.all(np.abs(l1 - l0) <= 1e-4 * np.abs(l0))
    for j in range(lanes):
        a, b = g1.reshape(lanes, -1)[j], g0.reshape(lanes, -1)[j]
        assert np.linalg.norm(a - b) <= GRAD_TOL * np.linalg.norm(b), j
    steps = 4
    fused = _run({"TLK_ATTN_FUSED": "1"}, model, lanes, batch, steps, cfg)
    plain = _run({"TLK_ATTN_FUSED": "0"}, model, lanes, batch, steps, cfg)
    lf, lp = np.array(fused["losses"]), np.array(plain["losses"])
    assert np.all(np.isfinite(lf))
    assert np.all(np.abs(lf - lp) <= LOSS_TOL * np.maximum(1.0, np.abs(lp)))


def test_fused_attention_skips_inactive_lanes():
    """A finished lane in the middle of the pack (fewer steps) leaves the
    other lanes' numbers unchanged (the work list skips it in every role)."""
    cfg = dict(layers=1, d_model=128, heads=2, seq_len=256, vocab=65)
    code = CODE.replace("p.load(j, seed=300 + j, steps=steps, lr=3e-3)",
                        "p.load(j, seed=300 + j, steps=(1 if j == 1 else steps), lr=3e-3)")
    out = subprocess.run([sys.executable, "-c", code, "gpt", "3", "4", "3", json.dumps(cfg)], capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    mixed = json.loads(out.stdout.strip().splitlines()[-1])
    full = _run({}, "gpt", 3, 4, 3, cfg)
    assert mixed["losses"][0] == full["losses"][0] and mixed["losses"][2] == full["losses"][2]
    assert mixed["params"][0] == full["params"][0] and mixed["params"][2] == full["params"][2]
