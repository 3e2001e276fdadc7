"""numpy restatement of the packed transformer jobs (oracle; test infrastructure).

SURVEY.md Appendix B / BASELINE.json configs 4 and 5:
  XFORMER  2 layers, d=256, 4 heads, FFN 1024, T=128, byte vocab 256, batch 32
  GPT      6 layers, d=384, 6 heads, FFN 1536, T=256, vocab 65, batch 64 (nanoGPT char)
Pre-LN decoder blocks (x += Wo attn(LN1 x); x += W2 gelu(W1 LN2 x)), learned
token + position embeddings, final LN, untied LM head, mean next-token CE.
GELU is the tanh approximation; LayerNorm eps 1e-5, biased variance.

Tokens come from a seeded order-1 Markov chain (restated bit-exactly by the
CUDA data kernel): token_0 = bits(key, s*(T+1)) mod V and
token_{i+1} = (token_i * A[k] + C[k]) mod V with k = bits(key, s*(T+1)+i+1) >> 61
(8 successors per token, a learnable distribution with entropy ln 8).

Parameter tensors (each starting at a 64-float boundary, restating
csrc/gpt.cu): wte [V,d], wpe [T,d], then per layer ln1.g, ln1.b [d],
attn.w [3d,d], attn.b [3d], proj.w [d,d], proj.b [d], ln2.g, ln2.b [d],
fc.w [4d,d], fc.b [4d], fc2.w [d,4d], fc2.b [d]; then lnf.g, lnf.b [d],
head.w [V,d].  LayerNorm gains init to 1 and biases to 0; matrices and
embeddings U(-1/sqrt(fan_in), 1/sqrt(fan_in)) from the shared counter RNG
(fan_in of an embedding = d).

bf16=True rounds where the CUDA path rounds: GEMM weight operands (bf16
shadow), LayerNorm outputs, q/k/v, attention probabilities, attention
outputs, GELU outputs and the stored GELU pre-activation (GELU' is evaluated
at bf16(z)), and every gradient fed to a GEMM; the residual stream
and its gradient, softmax / LayerNorm statistics, the logits and the GEMM
outputs consumed by LayerNorm backward stay fp32.  The attention backward
uses the stored bf16 probabilities (ds = P (dP - D) / sqrt(dh), with
D = rowsum(dY o Y), equal to rowsum(P o dP) in exact arithmetic).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import rng
from .bf16 import round_bf16

MODEL_XFORMER = 3
MODEL_GPT = 4
STREAM_TOKENS = 3
MARKOV_A = (1, 3, 5, 7, 11, 13, 17, 19)
MARKOV_C = (1, 2, 3, 5, 8, 13, 21, 34)
LN_EPS = np.float32(1e-5)
GELU_C = np.float32(0.7978845608028654)  # sqrt(2/pi)
GELU_K = np.float32(0.044715)


@dataclass(frozen=True)
class GptCfg:
    layers: int
    d: int
    heads: int
    T: int
    V: int
    batch: int

    @property
    def dh(self) -> int:
        return self.d // self.heads


CFGS = {
    MODEL_XFORMER: GptCfg(2, 256, 4, 128, 256, 32),
    MODEL_GPT: GptCfg(6, 384, 6, 256, 65, 64),
}


def tensors(cfg: GptCfg):
    """[(name, shape, fan_in, kind)] kind: 'u' uniform, 'one', 'zero'."""
    d, V, T = cfg.d, cfg.V, cfg.T
    out = [("wte", (V, d), d, "u"), ("wpe", (T, d), d, "u")]
    for l in range(cfg.layers):
        p = f"h{l}."
        out += [
            (p + "ln1.g", (d,), d, "one"), (p + "ln1.b", (d,), d, "zero"),
            (p + "attn.w", (3 * d, d), d, "u"), (p + "attn.b", (3 * d,), d, "u"),
            (p + "proj.w", (d, d), d, "u"), (p + "proj.b", (d,), d, "u"),
            (p + "ln2.g", (d,), d, "one"), (p + "ln2.b", (d,), d, "zero"),
            (p + "fc.w", (4 * d, d), d, "u"), (p + "fc.b", (4 * d,), d, "u"),
            (p + "fc2.w", (d, 4 * d), 4 * d, "u"), (p + "fc2.b", (d,), 4 * d, "u"),
        ]
    out += [("lnf.g", (d,), d, "one"), ("lnf.b", (d,), d, "zero"), ("head.w", (V, d), d, "u")]
    return out


def layout(cfg: GptCfg):
    lay, off = [], 0
    for name, shape, fan, kind in tensors(cfg):
        n = int(np.prod(shape))
        lay.append((name, shape, off))
        off = (off + n + 63) // 64 * 64
    return lay, sum(int(np.prod(s)) for _, s, _, _ in tensors(cfg)), off


def init_params(cfg: GptCfg, seed: int) -> dict:
    out = {}
    for i, (name, shape, fan, kind) in enumerate(tensors(cfg)):
        n = int(np.prod(shape))
        if kind == "one":
            out[name] = np.ones(shape, np.float32)
        elif kind == "zero":
            out[name] = np.zeros(shape, np.float32)
        else:
            out[name] = rng.init_uniform(seed, i, n, fan).reshape(shape)
    return out


def flatten(cfg, params):
    lay, _, stride = layout(cfg)
    flat = np.zeros(stride, np.float32)
    for name, shape, off in lay:
        flat[off:off + int(np.prod(shape))] = params[name].reshape(-1)
    return flat


def unflatten(cfg, flat):
    lay, _, _ = layout(cfg)
    return {n: flat[o:o + int(np.prod(s))].reshape(s).copy() for n, s, o in lay}


def tokens(cfg: GptCfg, seed: int, step: int, batch: int | None = None) -> np.ndarray:
    """int32 [batch, T+1] Markov-chain sequences (inputs = [:, :-1], targets = [:, 1:])."""
    B = cfg.batch if batch is None else batch
    T1 = cfg.T + 1
    h = rng.bits(rng.key(seed, STREAM_TOKENS, step), np.arange(B * T1)).reshape(B, T1)
    out = np.zeros((B, T1), np.int64)
    out[:, 0] = (h[:, 0] % np.uint64(cfg.V)).astype(np.int64)
    A = np.array(MARKOV_A, np.int64)
    C = np.array(MARKOV_C, np.int64)
    ks = (h >> np.uint64(61)).astype(np.int64)
    for i in range(cfg.T):
        k = ks[:, i + 1]
        out[:, i + 1] = (out[:, i] * A[k] + C[k]) % cfg.V
    return out.astype(np.int32)


# ------------------------------------------------------------------ pieces --
def _r(x, on):
    return round_bf16(x) if on else x.astype(np.float32, copy=False)


def ln_fwd(x, g, b):
    mu = x.mean(axis=-1, keepdims=True, dtype=np.float32)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True, dtype=np.float32)
    rstd = np.float32(1.0) / np.sqrt(var + LN_EPS)
    xh = xc * rstd
    return xh * g + b, xh, rstd


def ln_bwd(dy, xh, rstd, g):
    """dy [N, d] fp32 -> dx, dg, db (biased-variance LayerNorm)."""
    d = xh.shape[-1]
    dxh = dy * g
    m1 = dxh.mean(axis=-1, keepdims=True, dtype=np.float32)
    m2 = (dxh * xh).mean(axis=-1, keepdims=True, dtype=np.float32)
    dx = (dxh - m1 - xh * m2) * rstd
    return dx, (dy * xh).sum(axis=0), dy.sum(axis=0)


def gelu(x):
    u = GELU_C * (x + GELU_K * x * x * x)
    t = np.tanh(u)
    return np.float32(0.5) * x * (np.float32(1.0) + t), t


def gelu_bwd(x, t):
    du = GELU_C * (np.float32(1.0) + np.float32(3.0) * GELU_K * x * x)
    return np.float32(0.5) * (np.float32(1.0) + t) + np.float32(0.5) * x * (np.float32(1.0) - t * t) * du


def gpt_step(cfg: GptCfg, p: dict, toks: np.ndarray, bf16: bool = True):
    """One forward+backward on [B, T+1] tokens; returns (loss, grads)."""
    B, T, d, H, dh, V = toks.shape[0], cfg.T, cfg.d, cfg.heads, cfg.dh, cfg.V
    inp, tgt = toks[:, :-1], toks[:, 1:]
    N = B * T
    x = (p["wte"][inp] + p["wpe"][None, :T]).reshape(N, d).astype(np.float32)
    scale = np.float32(1.0 / np.sqrt(dh))
    causal = np.tril(np.ones((T, T), bool))
    cache = []
    for l in range(cfg.layers):
        q_ = f"h{l}."
        a, xh1, rs1 = ln_fwd(x, p[q_ + "ln1.g"], p[q_ + "ln1.b"])
        a = _r(a, bf16)
        wqkv = _r(p[q_ + "attn.w"], bf16)
        qkv = _r(a @ wqkv.T + p[q_ + "attn.b"], bf16).reshape(B, T, 3, H, dh)
        q, k, v = (qkv[:, :, i].transpose(0, 2, 1, 3) for i in range(3))  # [B,H,T,dh]
        s = (q @ k.transpose(0, 1, 3, 2)) * scale
        s = np.where(causal, s, np.float32(-np.inf))
        m = s.max(axis=-1, keepdims=True)
        e = np.exp(s - m)
        pr = e / e.sum(axis=-1, keepdims=True)
        pb = _r(pr, bf16)
        y = _r(pb @ v, bf16)                                            # [B,H,T,dh]
        yf = y.transpose(0, 2, 1, 3).reshape(N, d)
        wo = _r(p[q_ + "proj.w"], bf16)
        x = x + (yf @ wo.T + p[q_ + "proj.b"])
        mm, xh2, rs2 = ln_fwd(x, p[q_ + "ln2.g"], p[q_ + "ln2.b"])
        mm = _r(mm, bf16)
        w1 = _r(p[q_ + "fc.w"], bf16)
        z = mm @ w1.T + p[q_ + "fc.b"]
        f, tz = gelu(z)
        f = _r(f, bf16)
        w2 = _r(p[q_ + "fc2.w"], bf16)
        x = x + (f @ w2.T + p[q_ + "fc2.b"])
        cache.append((a, xh1, rs1, q, k, v, pb, pr, yf, mm, xh2, rs2, z, tz, f))
    xf, xhf, rsf = ln_fwd(x, p["lnf.g"], p["lnf.b"])
    xf = _r(xf, bf16)
    wh = _r(p["head.w"], bf16)
    logits = xf @ wh.T                                                  # [N, V]
    lm = logits.max(axis=1, keepdims=True)
    le = np.exp(logits - lm)
    ls = le.sum(axis=1, keepdims=True)
    y_ = tgt.reshape(-1)
    loss = np.float32((((lm + np.log(ls))[:, 0] - logits[np.arange(N), y_])).sum() / np.float32(N))
    dl = le / ls
    dl[np.arange(N), y_] -= np.float32(1.0)
    dl = _r((dl / np.float32(N)).astype(np.float32), bf16)
    g = {"head.w": dl.T @ xf}
    dxf = dl @ wh             # gradient into LN_f output (fp32, feeds LN backward)
    dx, g["lnf.g"], g["lnf.b"] = ln_bwd(dxf, xhf, rsf, p["lnf.g"])
    for l in reversed(range(cfg.layers)):
        q_ = f"h{l}."
        a, xh1, rs1, q, k, v, pb, pr, yf, mm, xh2, rs2, z, tz, f = cache[l]
        w2, w1 = _r(p[q_ + "fc2.w"], bf16), _r(p[q_ + "fc.w"], bf16)
        dxb = _r(dx, bf16)
        g[q_ + "fc2.w"] = dxb.T @ f
        g[q_ + "fc2.b"] = dxb.sum(axis=0)
        df = dxb @ w2
        if bf16:  # the CUDA path stores z as bf16 and evaluates GELU' there
            zb = round_bf16(z)
            dz = _r(df * gelu_bwd(zb, np.tanh(GELU_C * (zb + GELU_K * zb * zb * zb))), bf16)
        else:
            dz = df * gelu_bwd(z, tz)
        g[q_ + "fc.w"] = dz.T @ mm
        g[q_ + "fc.b"] = dz.sum(axis=0)
        dmm = dz @ w1
        dx2, g[q_ + "ln2.g"], g[q_ + "ln2.b"] = ln_bwd(dmm, xh2, rs2, p[q_ + "ln2.g"])
        dx = dx + dx2
        wo = _r(p[q_ + "proj.w"], bf16)
        dxb = _r(dx, bf16)
        g[q_ + "proj.w"] = dxb.T @ yf
        g[q_ + "proj.b"] = dxb.sum(axis=0)
        dy = _r(dxb @ wo, bf16).reshape(B, T, H, dh).transpose(0, 2, 1, 3)
        dp = dy @ v.transpose(0, 1, 3, 2)                               # [B,H,T,T]
        dv = _r(pb.transpose(0, 1, 3, 2) @ dy, bf16)
        # D = rowsum(P o dP) = rowsum(dY o Y) (the FlashAttention identity,
        # exact in real arithmetic); formed from the stored bf16 dY and Y, a
        # 64-wide dot product instead of a T-wide one (csrc/gpt.cu
        # attn_rowdot_kernel)
        yb = yf.reshape(B, T, H, dh).transpose(0, 2, 1, 3)
        rowdot = (dy * yb).sum(axis=-1, keepdims=True)
        ds = _r(pb * (dp - rowdot) * scale, bf16)
        dq = _r(ds @ k, bf16)
        dk = _r(ds.transpose(0, 1, 3, 2) @ q, bf16)
        dqkv = np.stack([dq, dk, dv], axis=2).transpose(0, 3, 2, 1, 4).reshape(N, 3 * d)
        wqkv = _r(p[q_ + "attn.w"], bf16)
        g[q_ + "attn.w"] = dqkv.T @ a
        g[q_ + "attn.b"] = dqkv.sum(axis=0)
        da = dqkv @ wqkv
        dx1, g[q_ + "ln1.g"], g[q_ + "ln1.b"] = ln_bwd(da, xh1, rs1, p[q_ + "ln1.g"])
        dx = dx + dx1
    dx = dx.reshape(B, T, d)
    g["wpe"] = np.zeros_like(p["wpe"])
    g["wpe"][:T] = dx.sum(axis=0)
    gwte = np.zeros_like(p["wte"])
    np.add.at(gwte, inp.reshape(-1), dx.reshape(N, d))
    g["wte"] = gwte
    return loss, g
