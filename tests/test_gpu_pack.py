"""Packed training parity: K lanes trained by libtlk vs the numpy oracle.

Each lane of a pack is compared with an independent oracle run of the same
task (same seed -> same init and data, same optimizer).  The oracle runs in
its bf16-emulation mode (rounds exactly the tensors the GPU rounds), so the
only differences are fp32 summation order.  Stated tolerances:

* init weights and synthetic data: bit-exact;
* teacher-forced step: layer-wise (oracle fed the GPU's own layer inputs)
  bf16 outputs equal up to rare 1-ulp midpoint flips and grads rel-L2 <= 1e-5;
  whole-step grads from the GPU's pre-step params rel-L2 <= 3e-2 (one flip of
  a large activation perturbs the whole sample downstream); optimizer update
  BIT-EXACT given the GPU's grads;
* free-running trajectories: per-step loss |d| <= 5e-3 * max(1, |L|);
  final weights rel-L2 per tensor <= 1e-2 for SGD and <= 6e-2 for Adam/AdamW.
  (Adam's m/sqrt(v) maps the sign of near-zero gradients to +-lr, so
  summation-order noise on those elements is amplified into whole-step
  differences; SGD is near-linear and shows the arithmetic agreement.)
"""

import numpy as np
import pytest
import torch

from oracle import job as ojob
from oracle import models as omodels
from oracle import optim as ooptim
from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu

LOSS_TOL = 5e-3
W_TOL = {ooptim.SGD: 1e-2, ooptim.ADAM: 6e-2, ooptim.ADAMW: 6e-2}
GRAD_TOL = 3e-2


def _oracle(model, seed, steps, batch, opt, **kw):
    st = ooptim.OptState(kind=opt, **kw)
    return ojob.train(model, seed, steps, batch, st, bf16=True)


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _check_lane(model, pack, lane, seed, steps, batch, opt, **kw):
    losses_ref, flat_ref, _ = _oracle(model, seed, steps, batch, opt, **kw)
    got = pack.losses(lane, steps)
    tol = LOSS_TOL * np.maximum(1.0, np.abs(losses_ref))
    assert np.all(np.abs(got - losses_ref) <= tol), (lane, got[:5], losses_ref[:5])
    params = pack.params(lane)
    lay, _, _ = omodels.layout(model)
    for t, off in lay:
        r = _rel_l2(params[off:off + t.count], flat_ref[off:off + t.count])
        assert r <= W_TOL[opt], (lane, t.name, r)


@pytest.mark.parametrize("model", [omodels.MODEL_MLP, omodels.MODEL_CNN])
def test_init_bit_exact(model):
    with rt.Context(0) as ctx:
        pack = ctx.pack(model, 64, 2, 4)
        for lane, seed in enumerate((5, 2**33 + 1)):
            pack.load(lane, seed=seed, steps=1)
        ctx.sync()
        for lane, seed in enumerate((5, 2**33 + 1)):
            ref = omodels.flatten_params(model, omodels.init_params(model, seed))
            assert np.array_equal(pack.params(lane), ref)


def test_mlp_pack_matches_oracle():
    steps, batch = 12, 64
    jobs = [
        (0, ooptim.ADAM, dict(lr=1e-3)),
        (1, ooptim.ADAM, dict(lr=3e-3, beta1=0.8)),
        (2, ooptim.ADAMW, dict(lr=2e-3, weight_decay=0.05)),
        (3, ooptim.SGD, dict(lr=0.05, momentum=0.9, weight_decay=1e-4)),
    ]
    names = {"beta1": "beta1", "beta2": "beta2", "weight_decay": "weight_decay", "momentum": "momentum"}
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_MLP, batch, len(jobs), steps)
        for lane, (seed, opt, kw) in enumerate(jobs):
            pack.load(lane, seed=seed, steps=steps, optimizer=opt, **{names.get(k, k): v for k, v in kw.items()})
        pack.run(steps)
        ctx.sync()
        for lane, (seed, opt, kw) in enumerate(jobs):
            st = pack.status(lane)
            assert st.steps_done == steps and st.active == 0
            _check_lane(omodels.MODEL_MLP, pack, lane, seed, steps, batch, opt, **kw)


def test_mlp_lanes_with_different_lengths_stop_independently():
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_MLP, 64, 3, 10)
        for lane, steps in enumerate((3, 10, 6)):
            pack.load(lane, seed=lane, steps=steps)
        pack.run(10)
        ctx.sync()
        for lane, steps in enumerate((3, 10, 6)):
            s = pack.status(lane)
            assert (s.steps_done, s.active) == (steps, 0)
            _check_lane(omodels.MODEL_MLP, pack, lane, lane, steps, 64, ooptim.ADAM, lr=1e-3)


def test_host_input_step_matches_device_generated():
    from oracle import rng

    lanes, batch = 2, 64
    with rt.Context(0) as ctx:
        dev = ctx.pack(omodels.MODEL_MLP, batch, lanes, 4)
        host = ctx.pack(omodels.MODEL_MLP, batch, lanes, 4, host_input=True)
        for p in (dev, host):
            for lane in range(lanes):
                p.load(lane, seed=lane + 10, steps=4)
        dev.run(4)
        for t in range(4):
            px = np.stack([rng.batch(lane + 10, t, batch)[0] for lane in range(lanes)])
            lb = np.stack([rng.batch(lane + 10, t, batch)[1] for lane in range(lanes)])
            out = host.step_host(px, lb)
            assert out.shape == (lanes,)
        ctx.sync()
        for lane in range(lanes):
            assert np.array_equal(dev.losses(lane, 4), host.losses(lane, 4))
            assert np.array_equal(dev.params(lane), host.params(lane))


@pytest.mark.parametrize("model", [omodels.MODEL_MLP, omodels.MODEL_CNN])
def test_pipelined_host_steps_match_device_generated(model):
    """tlk_step_host_async (double-buffered inputs, H2D overlapping the previous
    step): every step's losses equal the device-generated run, bit for bit."""
    from oracle import rng

    lanes, batch, steps = 3, 64, 6
    with rt.Context(0) as ctx:
        dev = ctx.pack(model, batch, lanes, steps)
        host = ctx.pack(model, batch, lanes, steps, host_input=True)
        for p in (dev, host):
            for lane in range(lanes):
                p.load(lane, seed=lane + 40, steps=steps)
        dev.run(steps)
        bufs = []
        for t in range(steps):
            px = np.ascontiguousarray(np.stack([rng.batch(lane + 40, t, batch)[0] for lane in range(lanes)]))
            lb = np.ascontiguousarray(np.stack([rng.batch(lane + 40, t, batch)[1] for lane in range(lanes)])
                                      .astype(np.int32))
            bufs.append((px, lb, np.zeros(lanes, np.float32)))
        tickets = []
        for t in range(steps):
            tickets.append(host.step_host_async(*bufs[t]))
            if t >= 1:
                host.step_host_wait(tickets[t - 1])
        host.step_host_wait(tickets[-1])
        ctx.sync()
        for t in range(steps):
            assert np.array_equal(bufs[t][2], np.array([dev.losses(j, steps)[t] for j in range(lanes)], np.float32))
        for lane in range(lanes):
            assert np.array_equal(dev.params(lane), host.params(lane))


def test_zero_copy_tensor_view():
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_MLP, 64, 2, 2)
        pack.load(0, seed=9, steps=2)
        ctx.sync()
        t = pack.tensor(rt.BUF_PARAMS)
        assert t.is_cuda and t.numel() == 2 * pack.info.param_stride
        ref = omodels.flatten_params(omodels.MODEL_MLP, omodels.init_params(omodels.MODEL_MLP, 9))
        assert np.array_equal(t[: pack.info.param_stride].cpu().numpy(), ref)


def _bf(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _ulp_close(gpu, ref, what, frac=2e-3):
    """bf16 tensors equal except for rare 1-ulp rounding flips (values that sit
    on a rounding midpoint within fp32 summation-order noise)."""
    diff = gpu != ref
    n = int(diff.sum())
    assert n <= max(2, frac * gpu.size), (what, n, gpu.size)
    if n:
        # one bf16 ulp, plus an absolute floor for values produced by heavy
        # cancellation (tensor-core fp32 accumulation noise relative to the
        # terms, not to the small result)
        bound = 2.0**-7 * np.abs(ref[diff]) + 2.0**-12 * np.abs(ref).max()
        excess = np.abs(gpu[diff] - ref[diff]) - bound
        assert excess.max() <= 0, (what, excess.max())


def _mlp_layerwise(pack, lane, seed, t, p0, g, batch):
    """Oracle fed the GPU's own layer inputs (TLK_BUF_ACTS = h1, h2, dz1, dz2)."""
    from oracle import rng
    from oracle.bf16 import round_bf16 as r

    L, n = pack.lanes, batch * 512
    acts = pack.tensor(rt.BUF_ACTS).cpu().numpy().astype(np.uint16)
    h1, h2, dz1, dz2 = [_bf(acts[(k * L + lane) * n:(k * L + lane + 1) * n]).reshape(batch, 512)
                        for k in range(4)]
    prm = omodels.unflatten(omodels.MODEL_MLP, p0)
    px, y = rng.batch(seed, t, batch)
    x = px.astype(np.float32) / np.float32(256)
    w1, w2 = r(prm["fc1.w"]), r(prm["fc2.w"])
    _ulp_close(h1, r(np.maximum(x @ w1.T + prm["fc1.b"], 0)), "h1")
    _ulp_close(h2, r(np.maximum(h1 @ w2.T + prm["fc2.b"], 0)), "h2")
    loss, g3w, g3b, dh2 = omodels.head(h2, prm["fc3.w"], prm["fc3.b"], y)
    _ulp_close(dz2, r(dh2 * (h2 > 0)), "dz2")
    _ulp_close(dz1, r((dz2 @ w2) * (h1 > 0)), "dz1")
    ref = {"fc3.w": g3w, "fc3.b": g3b, "fc2.w": dz2.T @ h1, "fc2.b": dz2.sum(0),
           "fc1.w": dz1.T @ x, "fc1.b": dz1.sum(0)}
    for tt, off in omodels.layout(omodels.MODEL_MLP)[0]:
        got = g[off:off + tt.count]
        assert _rel_l2(got, ref[tt.name].reshape(-1)) <= 1e-5, (t, lane, tt.name)


def _p28_to_nhwc(planes, B, size, off):
    """P28 chunk planes [C][npos][8] -> NHWC [B, size, size, 8*C] (interior at +off)."""
    C = planes.shape[0]
    img = planes[:, 32:32 + B * 784, :].reshape(C, B, 28, 28, 8)
    border = img.copy()
    border[:, :, off:off + size, off:off + size, :] = 0
    assert not border.any(), "P28 border/padding must stay zero"
    x = img[:, :, off:off + size, off:off + size, :]
    return np.ascontiguousarray(x.transpose(1, 2, 3, 0, 4).reshape(B, size, size, 8 * C))


def _cnn_acts(pack, lane, B, t=0):
    """Split TLK_BUF_ACTS (csrc/cnn.cu layout) into this lane's NHWC fp32 tensors
    of the lane's step t (p2 of odd steps is the second p2 buffer, after dz1)."""
    L = pack.lanes
    npos = 32 + B * 784 + 64
    raw = pack.tensor(rt.BUF_ACTS).cpu().numpy().view(np.uint8)
    sizes = [("h1", 4 * npos * 16), ("p2", B * 9216 * 2), ("idx", B * 9216), ("h3", B * 128 * 2),
             ("dz3", B * 128 * 2), ("dz2", 8 * npos * 16), ("dz1", 4 * npos * 16), ("p2_alt", B * 9216 * 2)]
    out, off = {}, 0
    for name, per in sizes:
        blob = raw[off + lane * per: off + (lane + 1) * per]
        out[name] = blob.copy() if name == "idx" else _bf(blob.view(np.uint16))
        off += (L * per + 15) // 16 * 16
    if t & 1:
        out["p2"] = out["p2_alt"]
    out["h1"] = _p28_to_nhwc(out["h1"].reshape(4, npos, 8), B, 26, 1)
    out["p2"] = out["p2"].reshape(B, 12, 12, 64)
    out["live"] = (out["idx"].reshape(B, 12, 12, 64) & 4) != 0
    out["idx"] = out["idx"].reshape(B, 12, 12, 64) & 3
    out["h3"] = out["h3"].reshape(B, 128)
    out["dz3"] = out["dz3"].reshape(B, 128)
    out["dz2"] = _p28_to_nhwc(out["dz2"].reshape(8, npos, 8), B, 24, 2)
    dz1 = out["dz1"].reshape(4, npos, 8)[:, 32:32 + B * 784, :].reshape(4, B, 28, 28, 8)
    out["dz1"] = np.ascontiguousarray(dz1[:, :, 1:27, 1:27, :].transpose(1, 2, 3, 0, 4).reshape(B, 26, 26, 32))
    return out


def _cnn_layerwise(pack, lane, seed, t, p0, g, batch):
    from oracle import rng
    from oracle.bf16 import round_bf16 as r

    B = batch
    a = _cnn_acts(pack, lane, B, t)
    prm = omodels.unflatten(omodels.MODEL_CNN, p0)
    px, y = rng.batch(seed, t, B)
    x = (px.astype(np.float32) / np.float32(256)).reshape(B, 28, 28, 1)
    cols1 = omodels._taps(x, 26)
    _ulp_close(a["h1"], r(np.maximum(cols1 @ prm["conv1.w"].T + prm["conv1.b"], 0)), "h1")
    w2 = r(prm["conv2.w"])
    cols2 = omodels._taps(a["h1"], 24)
    a2 = np.maximum(cols2 @ w2.T + prm["conv2.b"], 0)
    win = a2.reshape(B, 12, 2, 12, 2, 64).transpose(0, 1, 3, 2, 4, 5).reshape(B, 12, 12, 4, 64)
    _ulp_close(a["p2"], r(win.max(axis=3)), "p2")
    srt = np.sort(win, axis=3)
    clear = (srt[:, :, :, 3] - srt[:, :, :, 2]) > 1e-4 * np.maximum(srt[:, :, :, 3], 1e-3)
    assert (a["idx"] == np.argmax(win, axis=3))[clear & (srt[:, :, :, 3] > 0)].all(), "argmax"
    assert np.array_equal(a["live"], a["p2"] > 0), "live bit"
    flat = a["p2"].reshape(B, 9216)
    w3 = r(prm["fc1.w"])
    _ulp_close(a["h3"], r(np.maximum(flat @ w3.T + prm["fc1.b"], 0)), "h3")
    loss, g4w, g4b, dh3 = omodels.head(a["h3"], prm["fc2.w"], prm["fc2.b"], y)
    _ulp_close(a["dz3"], r(dh3 * (a["h3"] > 0)), "dz3")
    dp2 = (a["dz3"] @ w3).reshape(B, 12, 12, 64)
    onehot = np.arange(4)[None, None, None, :, None] == a["idx"][:, :, :, None, :]
    dwin = np.where(onehot & (a["p2"][:, :, :, None, :] > 0), dp2[:, :, :, None, :], np.float32(0))
    ref_dz2 = r(dwin.reshape(B, 12, 12, 2, 2, 64).transpose(0, 1, 3, 2, 4, 5).reshape(B, 24, 24, 64))
    _ulp_close(a["dz2"], ref_dz2, "dz2")
    dz2 = a["dz2"]
    dpad = np.pad(dz2, ((0, 0), (2, 2), (2, 2), (0, 0)))
    w2t = w2.reshape(64, 9, 32)
    dh1 = np.zeros((B, 26, 26, 32), np.float32)
    for kh in range(3):
        for kw in range(3):
            dh1 += dpad[:, 2 - kh:2 - kh + 26, 2 - kw:2 - kw + 26, :] @ w2t[:, kh * 3 + kw, :]
    _ulp_close(a["dz1"], r(dh1 * (a["h1"] > 0)), "dz1")
    dz1 = a["dz1"]
    ref = {"fc2.w": g4w, "fc2.b": g4b, "fc1.w": a["dz3"].T @ flat, "fc1.b": a["dz3"].sum(0),
           "conv2.w": dz2.reshape(-1, 64).T @ cols2.reshape(-1, 288),
           "conv2.b": dz2.reshape(-1, 64).sum(0),
           "conv1.w": dz1.reshape(-1, 32).T @ cols1.reshape(-1, 9),
           "conv1.b": dz1.reshape(-1, 32).sum(0)}
    for tt, off in omodels.layout(omodels.MODEL_CNN)[0]:
        got = g[off:off + tt.count]
        assert _rel_l2(got, ref[tt.name].reshape(-1)) <= 1e-5, (t, lane, tt.name,
                                                               _rel_l2(got, ref[tt.name].reshape(-1)))


LAYERWISE = {omodels.MODEL_MLP: _mlp_layerwise, omodels.MODEL_CNN: _cnn_layerwise}


def _teacher_forced(model, lanes_cfg, steps, batch=64):
    """Per step: (1) layer-wise -- the oracle fed the GPU's own inputs of each
    layer reproduces its outputs (bf16: up to rare 1-ulp flips) and its
    gradients (rel-L2 <= 1e-5); (2) whole-step grads from the GPU's pre-step
    params within GRAD_TOL (flips cascade); (3) the optimizer update on the
    GPU's grads is BIT-EXACT with oracle.optim."""
    from oracle import rng

    step_fn = omodels.STEP_FNS[model]
    with rt.Context(0) as ctx:
        pack = ctx.pack(model, batch, len(lanes_cfg), steps, flags=rt.PACK_WRITE_ALL_GRADS)
        for lane, (seed, opt, kw) in enumerate(lanes_cfg):
            pack.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
        P, G = pack.tensor(rt.BUF_PARAMS), pack.tensor(rt.BUF_GRADS)
        M1, M2 = pack.tensor(rt.BUF_MOM1), pack.tensor(rt.BUF_MOM2)
        S = pack.info.param_stride
        states = [ooptim.OptState(kind=opt, **kw) for _, opt, kw in lanes_cfg]
        for t in range(steps):
            ctx.sync()
            before = [(P[l * S:(l + 1) * S].cpu().numpy(), M1[l * S:(l + 1) * S].cpu().numpy(),
                       M2[l * S:(l + 1) * S].cpu().numpy()) for l in range(len(lanes_cfg))]
            pack.run(1)
            ctx.sync()
            for lane, (seed, opt, kw) in enumerate(lanes_cfg):
                p0, m0, v0 = before[lane]
                g = G[lane * S:(lane + 1) * S].cpu().numpy()
                LAYERWISE[model](pack, lane, seed, t, p0, g, batch)
                px, y = rng.batch(seed, t, batch)
                _, gref = step_fn(omodels.unflatten(model, p0), px, y, bf16=True)
                gflat = omodels.flatten_params(model, gref)
                for tt, off in omodels.layout(model)[0]:
                    sl = slice(off, off + tt.count)
                    assert _rel_l2(g[sl], gflat[sl]) <= GRAD_TOL, (t, lane, tt.name)
                st = states[lane]
                st.m, st.v = m0.copy(), v0.copy()
                p1 = ooptim.step(st, p0, g)
                got = P[lane * S:(lane + 1) * S].cpu().numpy()
                assert np.array_equal(got, p1), (t, lane, np.abs(got - p1).max())
                assert np.array_equal(M1[lane * S:(lane + 1) * S].cpu().numpy(), st.m)
                assert np.array_equal(M2[lane * S:(lane + 1) * S].cpu().numpy(), st.v)


def test_mlp_teacher_forced_grads_and_bit_exact_update():
    _teacher_forced(omodels.MODEL_MLP, [
        (21, ooptim.ADAM, dict(lr=1e-3)),
        (22, ooptim.ADAMW, dict(lr=2e-3, weight_decay=0.1)),
        (23, ooptim.SGD, dict(lr=0.05, momentum=0.9, weight_decay=1e-4)),
        (24, ooptim.ADAM, dict(lr=1e-3, weight_decay=1e-2, beta2=0.99)),
    ], steps=4)


def test_cnn_teacher_forced_grads_and_bit_exact_update():
    _teacher_forced(omodels.MODEL_CNN, [
        (31, ooptim.ADAM, dict(lr=1e-3)),
        (32, ooptim.SGD, dict(lr=0.02, momentum=0.9)),
        (33, ooptim.ADAMW, dict(lr=1e-3, weight_decay=0.01)),
    ], steps=3)


def test_cnn_pack_matches_oracle():
    steps, batch = 8, 64
    jobs = [(40 + i, ooptim.ADAM, dict(lr=1e-3 * (1 + i % 2))) for i in range(4)]
    jobs.append((50, ooptim.SGD, dict(lr=0.02, momentum=0.9)))
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_CNN, batch, len(jobs), steps)
        for lane, (seed, opt, kw) in enumerate(jobs):
            pack.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
        pack.run(steps)
        ctx.sync()
        for lane, (seed, opt, kw) in enumerate(jobs):
            _check_lane(omodels.MODEL_CNN, pack, lane, seed, steps, batch, opt, **kw)


@pytest.mark.parametrize("batch", [8, 32])
def test_cnn_small_batches(batch):
    with rt.Context(0) as ctx:
        pack = ctx.pack(omodels.MODEL_CNN, batch, 2, 3)
        for lane in range(2):
            pack.load(lane, seed=60 + lane, steps=3)
        pack.run(3)
        ctx.sync()
        for lane in range(2):
            _check_lane(omodels.MODEL_CNN, pack, lane, 60 + lane, 3, batch, ooptim.ADAM, lr=1e-3)
