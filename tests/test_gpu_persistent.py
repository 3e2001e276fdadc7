"""The persistent per-GPU scheduler kernel (csrc/cnn_persist.cu, TLK_PACK_PERSISTENT)
against the per-phase kernel graph of the same CNN pack.

Both run the same arithmetic in the same order, so every check is BIT-EXACT:
* 8 lanes x bs 64 (the configs[1] shape), mixed optimizers and task lengths
  (lanes go inactive in the middle of a multi-step launch), losses and final
  params / m / v identical to the graph path;
* chunking: run(7) + run(5) on the persistent pack equals run(12);
* the pipelined host-input path (tlk_step_host_async) on a persistent pack;
* one kernel launch per chunk of steps (tlk_pack_launches_per_step == 1).
"""

import numpy as np
import pytest

from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu

JOBS = [(700 + i, (rt.OPT_ADAM, rt.OPT_ADAMW, rt.OPT_SGD, rt.OPT_ADAM)[i % 4],
         dict(lr=(1e-3, 2e-3, 0.02, 5e-4)[i % 4], momentum=0.9 if i % 4 == 2 else 0.0,
              weight_decay=0.01 if i % 4 == 1 else 0.0), (12, 5, 9, 12, 3, 12, 7, 10)[i])
        for i in range(8)]


def _make(ctx, flags, lanes=8, cap=12):
    p = ctx.pack(rt.MODEL_CNN, 64, lanes, cap, flags=flags)
    for lane, (seed, opt, kw, steps) in enumerate(JOBS[:lanes]):
        p.load(lane, seed=seed, steps=steps, optimizer=opt, **kw)
    return p


def _state(p, lane):
    S = p.info.param_stride
    sl = slice(lane * S, (lane + 1) * S)
    return (p.params(lane), p.tensor(rt.BUF_MOM1)[sl].cpu().numpy(), p.tensor(rt.BUF_MOM2)[sl].cpu().numpy())


def test_persistent_matches_graph_bit_exact():
    with rt.Context(0) as ctx:
        g = _make(ctx, 0)
        q = _make(ctx, rt.PACK_PERSISTENT)
        assert q.launches_per_step() == 1 and g.launches_per_step() == 10
        g.run(12)
        q.run(12)
        ctx.sync()
        for lane, (_, _, _, steps) in enumerate(JOBS):
            assert q.status(lane).steps_done == steps and q.status(lane).active == 0
            assert np.array_equal(g.losses(lane, steps), q.losses(lane, steps)), lane
            for a, b in zip(_state(g, lane), _state(q, lane)):
                assert np.array_equal(a, b), lane


def test_persistent_chunking_is_invisible():
    with rt.Context(0) as ctx:
        a = _make(ctx, rt.PACK_PERSISTENT)
        b = _make(ctx, rt.PACK_PERSISTENT)
        a.run(12)
        b.run(7)
        b.run(5)
        ctx.sync()
        for lane, (_, _, _, steps) in enumerate(JOBS):
            assert np.array_equal(a.losses(lane, steps), b.losses(lane, steps))
            assert np.array_equal(a.params(lane), b.params(lane))


def test_persistent_host_input_pipeline():
    from oracle import rng

    lanes, steps = 3, 5
    with rt.Context(0) as ctx:
        dev = ctx.pack(rt.MODEL_CNN, 64, lanes, steps)
        host = ctx.pack(rt.MODEL_CNN, 64, lanes, steps, host_input=True, flags=rt.PACK_PERSISTENT)
        for p in (dev, host):
            for lane in range(lanes):
                p.load(lane, seed=lane + 90, steps=steps)
        dev.run(steps)
        bufs = []
        for t in range(steps):
            px = np.ascontiguousarray(np.stack([rng.batch(lane + 90, t, 64)[0] for lane in range(lanes)]))
            lb = np.ascontiguousarray(np.stack([rng.batch(lane + 90, t, 64)[1] for lane in range(lanes)])
                                      .astype(np.int32))
            bufs.append((px, lb, np.zeros(lanes, np.float32)))
        tickets = []
        for t in range(steps):
            tickets.append(host.step_host_async(*bufs[t]))
            if t:
                host.step_host_wait(tickets[t - 1])
        host.step_host_wait(tickets[-1])
        ctx.sync()
        for lane in range(lanes):
            assert np.array_equal(dev.losses(lane, steps), host.losses(lane, steps))
            assert np.array_equal(dev.params(lane), host.params(lane))
