"""numpy restatement of the packed ResNet-18 jobs (oracle; test infrastructure).

BASELINE.json configs[2] / SURVEY.md Appendix B: ResNet-18, CIFAR variant
(3x3 stride-1 stem, no max-pool), BasicBlocks [2, 2, 2, 2] with widths 64,
128, 256, 512, stride 2 and a 1x1 stride-2 conv + BN shortcut at the first
block of stages 2-4, global average pool, fc 512 -> 10.  BatchNorm in
training mode (batch statistics over N*H*W, biased variance, eps 1e-5); the
running averages do not influence training and are not kept.  Convolutions
have no bias.  11,173,962 parameters.  Activations are NHWC.

Data (restated bit-exactly by csrc/resnet.cu rn_inputs_kernel): sample s of
step t, element i = (h*32 + w)*3 + c of the 32x32x3 image uses
word = bits(key(seed, RDATA, t), s*3072 + i); S = sum of its four 16-bit
chunks (Irwin-Hall(4), mean 131070); x = bf16(f32(S - 131070) * f32(1/37837.227)),
approximately N(0, 1).  Label = argmax_k sum_i T[k, i] (S_i - 131070) in
exact integers (first max wins), T[k, i] = ((bits(key(TEACHER_SEED,
RTEACHER, 0), k*3072 + i) >> 60) & 15) - 8.

Parameter tensors (64-float aligned, restating csrc/resnet.cu): stem.w
[64,3,3,3] (co, kh, kw, ci), bn0.g, bn0.b; per stage s = 1..4 and block
b = 0, 1: conv1.w [C,3,3,Cin], bn1.g, bn1.b, conv2.w [C,3,3,C], bn2.g, bn2.b,
and for (s > 1, b = 0) ds.w [C,1,1,Cin], dsbn.g, dsbn.b; fc.w [10,512],
fc.b [10].  Conv / fc weights U(-1/sqrt(fan_in), +) (= torch's default
kaiming_uniform(a=sqrt 5) bound), BN gains 1, biases 0.

bf16=True rounds where the CUDA path rounds: conv weight operands (bf16
shadow), conv outputs y (stored bf16; BN statistics are taken from the
stored values), BN-ReLU outputs and block outputs, and the BN-backward
outputs dy that feed the dgrad / wgrad convolutions.  The BN statistics,
the pooled features, the fc head (fp32 weights), every gradient that is
not a conv operand and all weight gradients stay fp32.
"""

from __future__ import annotations

import numpy as np

from . import rng
from .bf16 import round_bf16

MODEL_RESNET18 = 5
STREAM_RDATA = 4
STREAM_RTEACHER = 5
BN_EPS = np.float32(1e-5)
X_SCALE = np.float32(1.0 / 37837.227)  # 1 / std of Irwin-Hall(4) over 16-bit chunks
STAGES = ((64, 1), (128, 2), (256, 2), (512, 2))
IMG = 3072


def tensors():
    """[(name, shape, fan_in, kind)] kind: 'u' uniform, 'one', 'zero'."""
    out = [("stem.w", (64, 3, 3, 3), 27, "u"), ("bn0.g", (64,), 27, "one"), ("bn0.b", (64,), 27, "zero")]
    cin = 64
    for s, (C, stride) in enumerate(STAGES):
        for b in range(2):
            p = f"l{s + 1}.{b}."
            ci = cin if b == 0 else C
            out += [(p + "conv1.w", (C, 3, 3, ci), 9 * ci, "u"), (p + "bn1.g", (C,), 9 * ci, "one"),
                    (p + "bn1.b", (C,), 9 * ci, "zero"), (p + "conv2.w", (C, 3, 3, C), 9 * C, "u"),
                    (p + "bn2.g", (C,), 9 * C, "one"), (p + "bn2.b", (C,), 9 * C, "zero")]
            if b == 0 and s > 0:
                out += [(p + "ds.w", (C, 1, 1, ci), ci, "u"), (p + "dsbn.g", (C,), ci, "one"),
                        (p + "dsbn.b", (C,), ci, "zero")]
        cin = C
    out += [("fc.w", (10, 512), 512, "u"), ("fc.b", (10,), 512, "u")]
    return out


def layout():
    lay, off = [], 0
    for name, shape, fan, kind in tensors():
        n = int(np.prod(shape))
        lay.append((name, shape, off))
        off = (off + n + 63) // 64 * 64
    return lay, sum(int(np.prod(s)) for _, s, _, _ in tensors()), off


def init_params(seed: int) -> dict:
    out = {}
    for i, (name, shape, fan, kind) in enumerate(tensors()):
        n = int(np.prod(shape))
        if kind == "one":
            out[name] = np.ones(shape, np.float32)
        elif kind == "zero":
            out[name] = np.zeros(shape, np.float32)
        else:
            out[name] = rng.init_uniform(seed, i, n, fan).reshape(shape)
    return out


def flatten(params):
    lay, _, stride = layout()
    flat = np.zeros(stride, np.float32)
    for name, shape, off in lay:
        flat[off:off + int(np.prod(shape))] = params[name].reshape(-1)
    return flat


def unflatten(flat):
    lay, _, _ = layout()
    return {n: flat[o:o + int(np.prod(s))].reshape(s).copy() for n, s, o in lay}


_TEACHER = None


def teacher() -> np.ndarray:
    """int64 [10, 3072] in [-8, 7]."""
    global _TEACHER
    if _TEACHER is None:
        w = rng.bits(rng.key(rng.TEACHER_SEED, STREAM_RTEACHER, 0), np.arange(10 * IMG))
        _TEACHER = (((w >> np.uint64(60)) & np.uint64(15)).astype(np.int64) - 8).reshape(10, IMG)
    return _TEACHER


def batch(seed: int, step: int, B: int):
    """(x bf16-valued float32 [B,32,32,3] NHWC, labels int32 [B])."""
    w = rng.bits(rng.key(seed, STREAM_RDATA, step), np.arange(B * IMG)).reshape(B, IMG)
    m = np.uint64(0xFFFF)
    S = sum(((w >> np.uint64(16 * q)) & m).astype(np.int64) for q in range(4)) - 131070
    x = round_bf16(S.astype(np.float32) * X_SCALE).reshape(B, 32, 32, 3)
    score = S @ teacher().T                     # exact int64
    return x, np.argmax(score, axis=1).astype(np.int32)


# ------------------------------------------------------------------ pieces --
def _r(x, on):
    return round_bf16(x) if on else x.astype(np.float32, copy=False)


def _pad(x, p):
    return np.pad(x, ((0, 0), (p, p), (p, p), (0, 0))) if p else x


def conv_fwd(x, w, stride):
    """x [B,H,W,Ci], w [Co,k,k,Ci] -> [B,Ho,Wo,Co] (fp32 accumulate)."""
    B, H, W, Ci = x.shape
    Co, k = w.shape[0], w.shape[1]
    p = (k - 1) // 2
    Ho, Wo = H // stride, W // stride
    xp = _pad(x, p)
    cols = np.empty((B, Ho, Wo, k, k, Ci), np.float32)
    for kh in range(k):
        for kw in range(k):
            cols[:, :, :, kh, kw] = xp[:, kh:kh + stride * Ho:stride, kw:kw + stride * Wo:stride]
    return (cols.reshape(-1, k * k * Ci) @ w.reshape(Co, -1).T).reshape(B, Ho, Wo, Co)


def conv_dgrad(dy, w, stride, H, W):
    B, Ho, Wo, Co = dy.shape
    k, Ci = w.shape[1], w.shape[3]
    p = (k - 1) // 2
    dxp = np.zeros((B, H + 2 * p, W + 2 * p, Ci), np.float32)
    d2 = dy.reshape(-1, Co)
    for kh in range(k):
        for kw in range(k):
            dxp[:, kh:kh + stride * Ho:stride, kw:kw + stride * Wo:stride] += (d2 @ w[:, kh, kw, :]).reshape(
                B, Ho, Wo, Ci)
    return dxp[:, p:p + H, p:p + W] if p else dxp


def conv_wgrad(dy, x, k, stride):
    B, Ho, Wo, Co = dy.shape
    Ci = x.shape[3]
    p = (k - 1) // 2
    xp = _pad(x, p)
    d2 = dy.reshape(-1, Co).T
    g = np.empty((Co, k, k, Ci), np.float32)
    for kh in range(k):
        for kw in range(k):
            g[:, kh, kw] = d2 @ xp[:, kh:kh + stride * Ho:stride, kw:kw + stride * Wo:stride].reshape(-1, Ci)
    return g


def bn_stats(y):
    C = y.shape[-1]
    y2 = y.reshape(-1, C).astype(np.float32)
    M = np.float32(y2.shape[0])
    mu = (y2.sum(axis=0, dtype=np.float32) / M).astype(np.float32)
    # two-pass (centred) variance: E[y^2] - mu^2 cancels catastrophically for
    # channels with |mu| >> sigma; the CUDA path combines per-32-row centred
    # partials with Chan's formula (equally stable)
    var = (np.square(y2 - mu).sum(axis=0, dtype=np.float32) / M).astype(np.float32)
    rstd = (np.float32(1.0) / np.sqrt(var + BN_EPS)).astype(np.float32)
    return mu, rstd


def bn_apply(y, st, g, b):
    mu, rstd = st
    return (y - mu) * rstd * g + b


def bn_bwd(gy, y, st, gamma):
    """gy fp32 [.., C] (already ReLU-masked) -> (dy fp32, dgamma, dbeta)."""
    mu, rstd = st
    C = y.shape[-1]
    xh = ((y - mu) * rstd).reshape(-1, C)
    g2 = gy.reshape(-1, C)
    M = np.float32(g2.shape[0])
    sg = g2.sum(axis=0, dtype=np.float32)
    sgx = (g2 * xh).sum(axis=0, dtype=np.float32)
    dy = gamma * rstd * (g2 - sg / M - xh * (sgx / M))
    return dy.reshape(y.shape).astype(np.float32), sgx, sg


# ------------------------------------------------------------ the pieces --
def conv_weights(p, bf16=True):
    return {n: _r(p[n], bf16) for n, _, _, _ in tensors() if n.endswith(".w") and n != "fc.w"}


def stem_forward(p, W, x, bf16=True):
    y0 = _r(conv_fwd(x, W["stem.w"], 1), bf16)
    st0 = bn_stats(y0)
    a0 = _r(np.maximum(bn_apply(y0, st0, p["bn0.g"], p["bn0.b"]), 0), bf16)
    return y0, st0, a0


def block_forward(p, W, q, xin, stride, bf16=True):
    """BasicBlock q ('l<s>.<b>.'); returns its cache (xin, y1, s1, a1, y2, s2, yd, sd, o)."""
    y1 = _r(conv_fwd(xin, W[q + "conv1.w"], stride), bf16)
    s1 = bn_stats(y1)
    a1 = _r(np.maximum(bn_apply(y1, s1, p[q + "bn1.g"], p[q + "bn1.b"]), 0), bf16)
    y2 = _r(conv_fwd(a1, W[q + "conv2.w"], 1), bf16)
    s2 = bn_stats(y2)
    if q + "ds.w" in W:
        yd = _r(conv_fwd(xin, W[q + "ds.w"], stride), bf16)
        sd = bn_stats(yd)
        short = bn_apply(yd, sd, p[q + "dsbn.g"], p[q + "dsbn.b"])
    else:
        yd = sd = None
        short = xin
    o = _r(np.maximum(bn_apply(y2, s2, p[q + "bn2.g"], p[q + "bn2.b"]) + short, 0), bf16)
    return (xin, y1, s1, a1, y2, s2, yd, sd, o)


def head(p, o, labels):
    """avg-pool + fc + mean CE -> (loss, G = dL/do fp32, {fc.w, fc.b} grads)."""
    B = o.shape[0]
    h = o.reshape(B, 16, 512).mean(axis=1, dtype=np.float32)
    logits = h @ p["fc.w"].T + p["fc.b"]
    lm = logits.max(axis=1, keepdims=True)
    le = np.exp(logits - lm)
    ls = le.sum(axis=1, keepdims=True)
    loss = np.float32((((lm + np.log(ls))[:, 0] - logits[np.arange(B), labels])).sum() / np.float32(B))
    dl = le / ls
    dl[np.arange(B), labels] -= np.float32(1.0)
    dl = (dl / np.float32(B)).astype(np.float32)
    dh = dl @ p["fc.w"]
    G = np.broadcast_to((dh / np.float32(16.0))[:, None, None, :], (B, 4, 4, 512)).astype(np.float32)
    return loss, G, {"fc.w": dl.T @ h, "fc.b": dl.sum(axis=0)}


def block_backward(p, W, q, cache, G, stride, bf16=True):
    """G = dL/d(block output) fp32 -> (dL/d(block input) fp32, grads of the block)."""
    xin, y1, s1, a1, y2, s2, yd, sd, o = cache
    g = {}
    go = G * (o > 0)
    dy2, g[q + "bn2.g"], g[q + "bn2.b"] = bn_bwd(go, y2, s2, p[q + "bn2.g"])
    dy2 = _r(dy2, bf16)
    g[q + "conv2.w"] = conv_wgrad(dy2, a1, 3, 1)
    da1 = conv_dgrad(dy2, W[q + "conv2.w"], 1, a1.shape[1], a1.shape[2])
    ga1 = da1 * (a1 > 0)
    dy1, g[q + "bn1.g"], g[q + "bn1.b"] = bn_bwd(ga1, y1, s1, p[q + "bn1.g"])
    dy1 = _r(dy1, bf16)
    g[q + "conv1.w"] = conv_wgrad(dy1, xin, 3, stride)
    Gx = conv_dgrad(dy1, W[q + "conv1.w"], stride, xin.shape[1], xin.shape[2])
    if yd is not None:
        dyd, g[q + "dsbn.g"], g[q + "dsbn.b"] = bn_bwd(go, yd, sd, p[q + "dsbn.g"])
        dyd = _r(dyd, bf16)
        g[q + "ds.w"] = conv_wgrad(dyd, xin, 1, stride)
        Gx = Gx + conv_dgrad(dyd, W[q + "ds.w"], stride, xin.shape[1], xin.shape[2])
    else:
        Gx = Gx + go
    return Gx, g


def stem_backward(p, x, y0, st0, a0, G, bf16=True):
    g = {}
    g0 = G * (a0 > 0)
    dy0, g["bn0.g"], g["bn0.b"] = bn_bwd(g0, y0, st0, p["bn0.g"])
    dy0 = _r(dy0, bf16)
    g["stem.w"] = conv_wgrad(dy0, x, 3, 1)
    return g


def blocks():
    """[(prefix, stride)] in forward order."""
    return [(f"l{s + 1}.{b}.", stride if b == 0 else 1) for s, (C, stride) in enumerate(STAGES) for b in range(2)]


# --------------------------------------------------------------- the step --
def resnet_step(params: dict, x, labels, bf16: bool = True):
    """One forward + backward. Returns (mean CE loss, grads dict)."""
    p = params
    W = conv_weights(p, bf16)
    y0, st0, a0 = stem_forward(p, W, x, bf16)
    caches, a = [], a0
    for q, stride in blocks():
        caches.append(block_forward(p, W, q, a, stride, bf16))
        a = caches[-1][-1]
    loss, G, g = head(p, a, labels)
    for (q, stride), cache in reversed(list(zip(blocks(), caches))):
        G, gb = block_backward(p, W, q, cache, G, stride, bf16)
        g.update(gb)
    g.update(stem_backward(p, x, y0, st0, a0, G, bf16))
    return loss, g
