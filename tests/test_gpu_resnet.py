"""ResNet-18 packs (BASELINE configs[2] model family) vs the numpy oracle
(oracle/resnet.py, itself pinned to torch float64 in test_oracle_golden.py).

* synthetic images, teacher labels and init weights: bit-exact;
* layer-local parity from one step: every forward stage recomputed by the
  oracle from the GPU's own stage inputs (one bf16 ulp), and every block's
  backward from the GPU's forward tensors and incoming-gradient snapshot
  (rel-L2 2e-2).  End-to-end gradients are not comparable at init: the
  oracle's own bf16 and fp32 modes differ by ~35% on early layers;
* loss curves within LOSS_TOL; packing invariance (a lane's losses are
  bit-identical alone and packed).
"""

import numpy as np
import pytest

from oracle import job as ojob
from oracle import optim as ooptim
from oracle import resnet as orn
from oracle.bf16 import to_bf16_bits
from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu

GRAD_TOL = 5e-2
LOSS_TOL = 1e-2


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_inputs_and_init_bit_exact():
    B = 8
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_RESNET18, B, 2, 1)
        for lane in range(2):
            p.load(lane, seed=40 + lane, steps=1, optimizer=rt.OPT_SGD, lr=0.01)
        ctx.sync()
        for lane in range(2):
            assert np.array_equal(p.params(lane), orn.flatten(orn.init_params(40 + lane)))
        p.run(1)
        ctx.sync()
        raw = p.tensor(rt.BUF_ACTS).cpu().numpy()
        labels = p.tensor(rt.BUF_LABELS).cpu().numpy()
        for lane in range(2):
            x, y = orn.batch(40 + lane, 0, B)
            got = raw[lane * B * 3072:(lane + 1) * B * 3072]
            assert np.array_equal(got, to_bf16_bits(x).reshape(-1))
            assert np.array_equal(labels[lane * B:(lane + 1) * B], y)


def _bf(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _ulp_frac(got, ref):
    """fraction of elements further apart than one bf16 ulp of the larger."""
    tol = np.maximum(np.abs(got), np.abs(ref)) * 2.0 ** -7 + 1e-6
    return float(np.mean(np.abs(got - ref) > tol))


def _conv_index():
    """oracle block prefix -> (c1, c2, cd) libtlk conv indices (0 = stem)."""
    idx, out = 1, {}
    for q, stride in orn.blocks():
        ds = q.endswith(".0.") and not q.startswith("l1.")
        out[q] = (idx, idx + 1, idx + 2 if ds else None)
        idx += 3 if ds else 2
    return out


@pytest.fixture(scope="module", params=[(16, 1, 0), (128, 2, 1)], ids=["bs16x1", "bs128x2-lane1"])
def snap(request):
    """One step of a pack with gradient snapshots; every named buffer of ONE
    lane copied to host.  (16, 1 lane) and the BASELINE configs[2] shape
    (bs 128, 2 lanes, checking lane 1: the per-lane offsets and the
    batch-dependent wgrad split-K / partial-buffer sizing of resnet.cu)."""
    B, lanes, lane = request.param
    seed = 55
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_RESNET18, B, lanes, 1, flags=rt.PACK_SNAPSHOTS)
        for j in range(lanes):
            p.load(j, seed=seed - lane + j, steps=1, optimizer=rt.OPT_SGD, lr=0.01)
        p.run(1)
        ctx.sync()
        names = ["xin", "a0", "stem.G"] + [f"conv{i}.{k}" for i in range(20) for k in ("y", "stats")]
        names += [f"blk{i}.{k}" for i in range(8) for k in ("a1", "o", "G")]
        out = {}
        for n in names:
            kind = "f4" if n.endswith((".stats", ".G")) else "u2"
            v = p.named(n, kind).cpu().numpy()
            per = v.size // lanes
            v = v[lane * per:(lane + 1) * per]
            out[n] = _bf(v) if kind == "u2" else v
        S = p.info.param_stride
        out["grads"] = p.tensor(rt.BUF_GRADS).cpu().numpy()[lane * S:(lane + 1) * S]
        out["labels"] = p.tensor(rt.BUF_LABELS).cpu().numpy()[lane * B:(lane + 1) * B]
        out["loss"] = p.losses(lane, 1)[0]
    out["B"], out["seed"] = B, seed
    return out


def _stats(v, C):
    return v[:C], v[C:2 * C]


def test_layerwise_forward(snap):
    """Each forward stage from the GPU's own inputs: conv outputs within one
    bf16 ulp (fp32 summation order), BN statistics to fp32 precision, BN-ReLU
    (+ shortcut) outputs within one ulp."""
    B = snap["B"]
    p = orn.init_params(snap["seed"])
    W = orn.conv_weights(p)
    x = snap["xin"].reshape(B, 32, 32, 3)
    y0 = snap["conv0.y"].reshape(B, 32, 32, 64)
    assert _ulp_frac(y0, orn.round_bf16(orn.conv_fwd(x, W["stem.w"], 1))) < 1e-3
    st0 = _stats(snap["conv0.stats"], 64)
    mu, rs = orn.bn_stats(y0)
    np.testing.assert_allclose(st0[0], mu, rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(st0[1], rs, rtol=1e-4)
    a0 = snap["a0"].reshape(B, 32, 32, 64)
    assert _ulp_frac(a0, orn.round_bf16(np.maximum(orn.bn_apply(y0, st0, p["bn0.g"], p["bn0.b"]), 0))) < 1e-3
    ci = _conv_index()
    xin, res = a0, 32
    for i, (q, stride) in enumerate(orn.blocks()):
        c1, c2, cd = ci[q]
        C = W[q + "conv1.w"].shape[0]
        ho = res // stride
        y1 = snap[f"conv{c1}.y"].reshape(B, ho, ho, C)
        assert _ulp_frac(y1, orn.round_bf16(orn.conv_fwd(xin, W[q + "conv1.w"], stride))) < 1e-3, (q, "conv1")
        s1 = _stats(snap[f"conv{c1}.stats"], C)
        mu, rs = orn.bn_stats(y1)
        np.testing.assert_allclose(s1[1], rs, rtol=1e-4, err_msg=q)
        a1 = snap[f"blk{i}.a1"].reshape(B, ho, ho, C)
        assert _ulp_frac(a1, orn.round_bf16(np.maximum(orn.bn_apply(y1, s1, p[q + "bn1.g"], p[q + "bn1.b"]), 0))) < 1e-3
        y2 = snap[f"conv{c2}.y"].reshape(B, ho, ho, C)
        assert _ulp_frac(y2, orn.round_bf16(orn.conv_fwd(a1, W[q + "conv2.w"], 1))) < 1e-3, (q, "conv2")
        s2 = _stats(snap[f"conv{c2}.stats"], C)
        short = xin
        if cd is not None:
            yd = snap[f"conv{cd}.y"].reshape(B, ho, ho, C)
            assert _ulp_frac(yd, orn.round_bf16(orn.conv_fwd(xin, W[q + "ds.w"], stride))) < 1e-3, (q, "ds")
            short = orn.bn_apply(yd, _stats(snap[f"conv{cd}.stats"], C), p[q + "dsbn.g"], p[q + "dsbn.b"])
        o = snap[f"blk{i}.o"].reshape(B, ho, ho, C)
        ref = orn.round_bf16(np.maximum(orn.bn_apply(y2, s2, p[q + "bn2.g"], p[q + "bn2.b"]) + short, 0))
        assert _ulp_frac(o, ref) < 1e-3, (q, "out")
        xin, res = o, ho


def test_layerwise_backward(snap):
    """Head and every block's backward from the GPU's own forward tensors and
    incoming gradient (snapshots): the block's parameter gradients and its
    input gradient within rel-L2 BWD_TOL (bf16 rounding of dy inside one block
    only); the end-to-end gradient is chaotic at init (oracle bf16 vs fp32
    differ by ~35% on early layers) and is not a usable parity signal."""
    B = snap["B"]
    BWD_TOL = 2e-2
    p = orn.init_params(snap["seed"])
    W = orn.conv_weights(p)
    lay = {n: (s, o) for n, s, o in orn.layout()[0]}
    grads = snap["grads"]

    def gpu_grad(n):
        s, o = lay[n]
        return grads[o:o + int(np.prod(s))]

    ci = _conv_index()
    res_of, r = {}, 32
    for q, stride in orn.blocks():
        r //= stride
        res_of[q] = r
    qs = orn.blocks()
    o_last = snap["blk7.o"].reshape(B, 4, 4, 512)
    loss, G, gh = orn.head(p, o_last, snap["labels"])
    assert abs(loss - snap["loss"]) < 1e-4 * max(1, abs(loss))
    np.testing.assert_allclose(snap["blk7.G"], G.reshape(-1), rtol=1e-4, atol=1e-7)
    for n in ("fc.w", "fc.b"):
        assert _rel(gpu_grad(n), gh[n].reshape(-1)) < 1e-4, n
    bad = []
    for i in reversed(range(8)):
        q, stride = qs[i]
        c1, c2, cd = ci[q]
        C, ho = W[q + "conv1.w"].shape[0], res_of[q]
        hi = ho * stride
        cin = W[q + "conv1.w"].shape[3]
        xin = (snap["a0"] if i == 0 else snap[f"blk{i - 1}.o"]).reshape(B, hi, hi, cin)
        cache = (xin, snap[f"conv{c1}.y"].reshape(B, ho, ho, C), _stats(snap[f"conv{c1}.stats"], C),
                 snap[f"blk{i}.a1"].reshape(B, ho, ho, C), snap[f"conv{c2}.y"].reshape(B, ho, ho, C),
                 _stats(snap[f"conv{c2}.stats"], C),
                 None if cd is None else snap[f"conv{cd}.y"].reshape(B, ho, ho, C),
                 None if cd is None else _stats(snap[f"conv{cd}.stats"], C), snap[f"blk{i}.o"].reshape(B, ho, ho, C))
        Gin = snap[f"blk{i}.G"].reshape(B, ho, ho, C)
        Gx, gb = orn.block_backward(p, W, q, cache, Gin, stride)
        Gnext = snap["stem.G"] if i == 0 else snap[f"blk{i - 1}.G"]
        r = _rel(Gnext, Gx.reshape(-1))
        if r > BWD_TOL:
            bad.append((q, "dX", round(r, 4)))
        for n, v in gb.items():
            r = _rel(gpu_grad(n), v.reshape(-1))
            if r > BWD_TOL:
                bad.append((n, round(r, 4)))
    y0 = snap["conv0.y"].reshape(B, 32, 32, 64)
    gs = orn.stem_backward(p, snap["xin"].reshape(B, 32, 32, 3), y0, _stats(snap["conv0.stats"], 64),
                           snap["a0"].reshape(B, 32, 32, 64), snap["stem.G"].reshape(B, 32, 32, 64))
    for n, v in gs.items():
        r = _rel(gpu_grad(n), v.reshape(-1))
        if r > BWD_TOL:
            bad.append((n, round(r, 4)))
    assert not bad, bad


def test_loss_curve_and_packing_invariance():
    steps, B = 4, 16
    jobs = [(60, dict(lr=0.02, momentum=0.9)), (61, dict(lr=0.01, momentum=0.0))]
    with rt.Context(0) as ctx:
        packed = ctx.pack(rt.MODEL_RESNET18, B, 3, steps)
        for lane, (seed, kw) in enumerate(jobs):
            packed.load(lane, seed=seed, steps=steps, optimizer=rt.OPT_SGD, **kw)
        packed.load(2, seed=62, steps=2, optimizer=rt.OPT_SGD, lr=0.01)  # a shorter neighbour
        packed.run(steps)
        ctx.sync()
        for lane, (seed, kw) in enumerate(jobs):
            got = packed.losses(lane, steps)
            ref, _, _ = ojob.train_resnet(seed, steps, B, ooptim.OptState(kind=ooptim.SGD, **kw), bf16=True)
            ref32, _, _ = ojob.train_resnet(seed, steps, B, ooptim.OptState(kind=ooptim.SGD, **kw), bf16=False)
            # first step: forward only (bf16 rounding flips through 20 BN layers
            # move the loss by ~1e-3); later steps drift with the chaotic
            # bf16 gradients (see test_layerwise_backward): the bound per step
            # is 0.05 or 3x the oracle's own bf16-vs-fp32 spread, whichever is
            # larger (any change of fp32 summation order -- e.g. the halo conv
            # tap order -- moves step 4 by a few 1e-2 at batch 16)
            assert abs(got[0] - ref[0]) < 5e-3 * abs(ref[0])
            tol = np.maximum(0.05, 3.0 * np.abs(ref - ref32))
            assert np.all(np.abs(got - ref) <= tol), (got, ref, ref32)
            alone = ctx.pack(rt.MODEL_RESNET18, B, 1, steps)
            alone.load(0, seed=seed, steps=steps, optimizer=rt.OPT_SGD, **kw)
            alone.run(steps)
            ctx.sync()
            assert np.array_equal(alone.losses(0, steps), got)


def test_loss_curve_bs128_bench_shape():
    """configs[2] shape: 2 lanes x bs 128, SGD-momentum, 3 steps vs the oracle
    (same per-step bound as test_loss_curve_and_packing_invariance)."""
    steps, B = 3, 128
    jobs = [(64, dict(lr=0.02, momentum=0.9)), (65, dict(lr=0.05, momentum=0.9, weight_decay=5e-4))]
    with rt.Context(0) as ctx:
        p = ctx.pack(rt.MODEL_RESNET18, B, len(jobs), steps)
        for lane, (seed, kw) in enumerate(jobs):
            p.load(lane, seed=seed, steps=steps, optimizer=rt.OPT_SGD, **kw)
        p.run(steps)
        ctx.sync()
        for lane, (seed, kw) in enumerate(jobs):
            got = p.losses(lane, steps)
            ref, _, _ = ojob.train_resnet(seed, steps, B, ooptim.OptState(kind=ooptim.SGD, **kw), bf16=True)
            ref32, _, _ = ojob.train_resnet(seed, steps, B, ooptim.OptState(kind=ooptim.SGD, **kw), bf16=False)
            assert abs(got[0] - ref[0]) < 5e-3 * abs(ref[0]), (lane, got, ref)
            tol = np.maximum(0.05, 3.0 * np.abs(ref - ref32))
            assert np.all(np.abs(got - ref) <= tol), (lane, got, ref, ref32)
