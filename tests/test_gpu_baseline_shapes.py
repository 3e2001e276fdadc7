"""Parity at the shapes BASELINE.json's configs (and bench.py) actually run.

* configs[1] -- the headline: 8 CNN lanes x bs 64 in ONE pack.  Teacher-forced
  layer-wise outputs / gradients for every lane (oracle fed the GPU's own layer
  inputs), the optimizer update bit-exact, then free-running loss curves and
  final weights of all 8 lanes vs independent oracle runs.
* configs[4] -- tiny-GPT at its real layout (6 layers, d 384, 6 heads, T 256,
  vocab 65), 2 lanes: bit-exact tokens and init, every parameter's first-step
  gradient within GRAD_TOL of the bf16-emulating oracle (this is the shape
  whose attention-score / dP GEMMs take the 256-wide causal row epilogues),
  and a 4-step loss curve per lane.
(configs[2], ResNet-18 at bs 128 x 2 lanes: tests/test_gpu_resnet.py.)
"""

import numpy as np
import pytest

from oracle import gpt as ogpt
from oracle import job as ojob
from oracle import models as omodels
from oracle import optim as ooptim
from paper_2410_22254_b200 import runtime as rt
from tests.test_gpu_pack import _check_lane, _teacher_forced

pytestmark = pytest.mark.gpu

GPT = ogpt.CFGS[ogpt.MODEL_GPT]
GRAD_TOL = 5e-2
LOSS_TOL = 5e-3


def _cnn_jobs(base):
    kinds = [(ooptim.ADAM, dict(lr=1e-3)), (ooptim.ADAMW, dict(lr=2e-3, weight_decay=0.01)),
             (ooptim.SGD, dict(lr=0.02, momentum=0.9)), (ooptim.ADAM, dict(lr=5e-4, beta1=0.8))]
    return [(base + i, *kinds[i % 4]) for i in range(8)]


def test_cnn_8_lanes_bs64_teacher_forced():
    _teacher_forced(omodels.MODEL_CNN, _cnn_jobs(400), steps=2, batch=64)


def test_cnn_8_lanes_bs64_trajectories():
    steps, batch = 10, 64
    jobs = _cnn_jobs(500)
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_CNN, batch, len(jobs), steps)
        for lane, (seed, opt, kw) in enumerate(jobs):
            pack.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
        pack.run(steps)
        ctx.sync()
        for lane, (seed, opt, kw) in enumerate(jobs):
            _check_lane(omodels.MODEL_CNN, pack, lane, seed, steps, batch, opt, **kw)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_tiny_gpt_default_layout_first_step():
    batch, lanes = 4, 2
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_GPT, batch, lanes, 1)  # 0 = the model's default layout
        for lane in range(lanes):
            p.load(lane, seed=610 + lane, steps=1, optimizer=rt.OPT_ADAMW, lr=3e-4, weight_decay=0.1)
        ctx.sync()
        S = p.info.param_stride
        _, _, stride = ogpt.layout(GPT)
        assert S == stride
        for lane in range(lanes):
            assert np.array_equal(p.params(lane), ogpt.flatten(GPT, ogpt.init_params(GPT, 610 + lane)))
        p.run(1)
        ctx.sync()
        raw = p.tensor(rt.BUF_ACTS).cpu().numpy().view(np.int32)
        G = p.tensor(rt.BUF_GRADS).cpu().numpy()
        lay, _, _ = ogpt.layout(GPT)
        bad = []
        for lane in range(lanes):
            toks = ogpt.tokens(GPT, 610 + lane, 0, batch)
            T1 = GPT.T + 1
            assert np.array_equal(raw[lane * batch * T1:(lane + 1) * batch * T1].reshape(batch, T1), toks)
            params = ogpt.init_params(GPT, 610 + lane)
            loss, g = ogpt.gpt_step(GPT, params, toks, bf16=True)
            got = p.losses(lane, 1)[0]
            assert abs(got - loss) <= LOSS_TOL * max(1.0, abs(loss)), (lane, got, loss)
            gl = G[lane * S:(lane + 1) * S]
            for name, shape, off in lay:
                n = int(np.prod(shape))
                r = _rel(gl[off:off + n], g[name].reshape(-1))
                if r > GRAD_TOL:
                    bad.append((lane, name, round(r, 4)))
        assert not bad, bad


def test_tiny_gpt_default_layout_loss_curve():
    steps, batch = 4, 4
    jobs = [(620, ooptim.ADAMW, dict(lr=1e-3, weight_decay=0.1)), (621, ooptim.ADAM, dict(lr=3e-4))]
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_GPT, batch, len(jobs), steps)
        for lane, (seed, opt, kw) in enumerate(jobs):
            p.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
        p.run(steps)
        ctx.sync()
        for lane, (seed, opt, kw) in enumerate(jobs):
            ref, _, _ = ojob.train_gpt(GPT, seed, steps, ooptim.OptState(kind=opt, **kw), bf16=True, batch=batch)
            got = p.losses(lane, steps)
            assert np.all(np.abs(got - ref) <= LOSS_TOL * np.maximum(1, np.abs(ref))), (lane, got, ref)
