"""Transformer packs (configs 4/5 model family) vs the numpy oracle (oracle/gpt.py).

* Markov-chain tokens and init weights: bit-exact;
* one step from init: every parameter gradient within rel-L2 GRAD_TOL of the
  oracle's bf16-emulating gradient (fp32 summation-order + bf16 flips);
* free-running loss curves within LOSS_TOL; packing invariance (a lane's
  losses are bit-identical alone and packed).
"""

import numpy as np
import pytest

from oracle import gpt as ogpt
from oracle import job as ojob
from oracle import optim as ooptim
from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu

SMALL = dict(layers=2, d_model=128, heads=2, seq_len=64, vocab=65)
SMALL_CFG = ogpt.GptCfg(2, 128, 2, 64, 65, 8)
GRAD_TOL = 5e-2
LOSS_TOL = 5e-3


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _pack(ctx, lanes, steps, batch=8, model=rt.MODEL_GPT, **cfg):
    return ctx.pack(model, batch, lanes, steps, **(cfg or SMALL))


def test_tokens_and_init_bit_exact():
    with rt.Context(0) as ctx:
        p = _pack(ctx, 2, 1)
        for lane in range(2):
            p.load(lane, seed=70 + lane, steps=1)
        ctx.sync()
        for lane in range(2):
            ref = ogpt.flatten(SMALL_CFG, ogpt.init_params(SMALL_CFG, 70 + lane))
            assert np.array_equal(p.params(lane), ref)
        p.run(1)
        ctx.sync()
        raw = p.tensor(rt.BUF_ACTS).cpu().numpy().view(np.int32)  # tokens are the first buffer
        B, T = 8, SMALL_CFG.T
        for lane in range(2):
            got = raw[lane * B * (T + 1):(lane + 1) * B * (T + 1)].reshape(B, T + 1)
            assert np.array_equal(got, ogpt.tokens(SMALL_CFG, 70 + lane, 0, B))


@pytest.mark.parametrize("model,cfg,ocfg,batch", [
    (rt.MODEL_GPT, SMALL, SMALL_CFG, 8),
    (rt.MODEL_XFORMER, {}, ogpt.CFGS[ogpt.MODEL_XFORMER], 8),
])
def test_first_step_gradients_match_oracle(model, cfg, ocfg, batch):
    with rt.Context(0) as ctx:
        p = ctx.pack(model, batch, 2, 1, **cfg)
        for lane in range(2):
            p.load(lane, seed=80 + lane, steps=1)
        p.run(1)
        ctx.sync()
        G = p.tensor(rt.BUF_GRADS).cpu().numpy()
        S = p.info.param_stride
        for lane in range(2):
            params = ogpt.init_params(ocfg, 80 + lane)
            loss, g = ogpt.gpt_step(ocfg, params, ogpt.tokens(ocfg, 80 + lane, 0, batch), bf16=True)
            assert abs(p.losses(lane, 1)[0] - loss) <= LOSS_TOL * max(1.0, abs(loss))
            lay, _, _ = ogpt.layout(ocfg)
            gl = G[lane * S:(lane + 1) * S]
            for name, shape, off in lay:
                n = int(np.prod(shape))
                r = _rel(gl[off:off + n], g[name].reshape(-1))
                assert r <= GRAD_TOL, (lane, name, r)


def test_loss_curve_and_packing_invariance():
    steps = 6
    jobs = [(90, ooptim.ADAMW, dict(lr=3e-3, weight_decay=0.1)), (91, ooptim.ADAM, dict(lr=1e-3))]
    with rt.Context(0) as ctx:
        p = _pack(ctx, len(jobs), steps)
        for lane, (seed, opt, kw) in enumerate(jobs):
            p.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
        p.run(steps)
        ctx.sync()
        alone = _pack(ctx, 1, steps)
        alone.load(0, seed=91, steps=steps, optimizer=ooptim.ADAM, lr=1e-3)
        alone.run(steps)
        ctx.sync()
        assert np.array_equal(alone.losses(0, steps), p.losses(1, steps))
        for lane, (seed, opt, kw) in enumerate(jobs):
            ref, _, _ = ojob.train_gpt(SMALL_CFG, seed, steps, ooptim.OptState(kind=opt, **kw), bf16=True)
            got = p.losses(lane, steps)
            assert np.all(np.abs(got - ref) <= LOSS_TOL * np.maximum(1, np.abs(ref))), (lane, got, ref)
