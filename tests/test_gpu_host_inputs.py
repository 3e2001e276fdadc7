"""End-to-end host-input steps (tlk_step_host_blob) for every model family:
a pack fed each step from a HOST blob built by the oracle's data generators
trains bit-identically to the pack that synthesises the same data on the
device.  This is the e2e path bench.py times for the ResNet / transformer
lines (host -> device inputs and device -> host losses every step)."""

import numpy as np
import pytest

from oracle import gpt as ogpt
from oracle import resnet as orn
from oracle import rng as orng
from oracle.bf16 import to_bf16_bits
from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _run_pair(model, batch, lanes, steps, blob_fn, **cfg):
    with rt.Context(0) as ctx:
        dev = ctx.pack(model, batch, lanes, steps, **cfg)
        host = ctx.pack(model, batch, lanes, steps, host_input=True, **cfg)
        kw = dict(optimizer=rt.OPT_SGD, lr=0.02, momentum=0.9) if model == rt.MODEL_RESNET18 else {}
        for p in (dev, host):
            for lane in range(lanes):
                p.load(lane, seed=500 + lane, steps=steps, **kw)
        dev.run(steps)
        for t in range(steps):
            blob = blob_fn(t)
            assert blob.nbytes == host.host_input_bytes()
            out = host.step_host_blob(blob)
            assert out.shape == (lanes,)
        ctx.sync()
        for lane in range(lanes):
            assert np.array_equal(dev.losses(lane, steps), host.losses(lane, steps)), lane
            assert np.array_equal(dev.params(lane), host.params(lane)), lane
        return out


def test_gpt_host_tokens():
    cfg = ogpt.GptCfg(2, 128, 2, 64, 65, 4)
    lanes, B = 2, 4
    blob = lambda t: np.concatenate([ogpt.tokens(cfg, 500 + j, t, B).reshape(-1) for j in range(lanes)]).astype(np.int32)
    _run_pair(rt.MODEL_GPT, B, lanes, 3, blob, layers=2, d_model=128, heads=2, seq_len=64, vocab=65)


def test_resnet_host_images():
    lanes, B = 2, 16

    def blob(t):
        xs, ys = zip(*(orn.batch(500 + j, t, B) for j in range(lanes)))
        img = np.concatenate([to_bf16_bits(x).reshape(-1) for x in xs]).astype(np.uint16)
        lab = np.concatenate(ys).astype(np.int32)
        return np.concatenate([img.view(np.uint8), lab.view(np.uint8)])

    _run_pair(rt.MODEL_RESNET18, B, lanes, 2, blob)


def test_cnn_host_blob():
    lanes, B = 3, 64

    def blob(t):
        px = np.stack([orng.batch(500 + j, t, B)[0] for j in range(lanes)]).astype(np.uint8)
        lb = np.stack([orng.batch(500 + j, t, B)[1] for j in range(lanes)]).astype(np.int32)
        return np.concatenate([px.reshape(-1), lb.reshape(-1).view(np.uint8)])

    _run_pair(rt.MODEL_CNN, B, lanes, 3, blob)


def test_cnn_host_async_then_params_without_sync():
    """Pipelined host steps (tlk_step_host_async) leave the CNN's deferred fc1
    wgrad + Adam of the last step in flight; tlk_lane_params must settle it
    without an explicit tlk_sync: the parameters then equal those of the
    device-input pack after the same steps, bit for bit."""
    lanes, B, steps = 3, 64, 4
    with rt.Context(0) as ctx:
        dev = ctx.pack(rt.MODEL_CNN, B, lanes, steps)
        host = ctx.pack(rt.MODEL_CNN, B, lanes, steps, host_input=True)
        for p in (dev, host):
            for lane in range(lanes):
                p.load(lane, seed=700 + lane, steps=steps)
        dev.run(steps)
        outs = [np.zeros(lanes, np.float32) for _ in range(2)]
        keep = []  # the host buffers of a step stay alive until its wait
        prev = None
        for t in range(steps):
            px = np.ascontiguousarray(np.stack([orng.batch(700 + j, t, B)[0] for j in range(lanes)])
                                      .astype(np.uint8).reshape(lanes, B, 784))
            lb = np.ascontiguousarray(np.stack([orng.batch(700 + j, t, B)[1] for j in range(lanes)]).astype(np.int32))
            keep.append((px, lb))
            tk = host.step_host_async(px, lb, outs[t & 1])
            if prev is not None:
                host.step_host_wait(prev)
            prev = tk
        host.step_host_wait(prev)
        for lane in range(lanes):  # no ctx.sync(): the lane call settles the deferred update
            assert np.array_equal(dev.params(lane), host.params(lane)), lane
            assert np.array_equal(dev.losses(lane, steps), host.losses(lane, steps)), lane
