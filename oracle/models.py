"""numpy restatement of the packed training tasks (oracle; test infrastructure).

Parameter layout restates ``paper_2410_22254_b200/csrc/models.cuh``
(``tlk_model_tensor``): each tensor starts at a multiple of 64 floats inside a
lane's fp32 arena.  Model definitions restate SURVEY.md Appendix B:

* MLP  784-512-512-10, ReLU (``TLK_MODEL_MLP``)
* CNN  pytorch/examples MNIST ``Net`` without dropout (``TLK_MODEL_CNN``):
  conv3x3(1->32)+ReLU, conv3x3(32->64)+ReLU, maxpool2, flatten (NHWC order
  (h, w, c)), fc(9216->128)+ReLU, fc(128->10); mean cross-entropy.

Weights use the (out, kh, kw, in) = "taps-major, channels-minor" layout the
NHWC kernels consume.  ``tests/golden/gen_torch_golden.py`` maps them onto
torch's (out, in, kh, kw) / NCHW-flatten layout to pin this file against
PyTorch CPU.

``bf16=True`` rounds exactly where the CUDA path rounds:
GEMM weight operands (bf16 shadow of fp32 masters), stored activations
(h1, p2, h3 / MLP h1, h2) and stored gradient operands (dz*).  The classifier
head (last Linear + CE + its backward) runs in fp32 on fp32 master weights,
as does conv1 (CUDA-core kernels in the GPU path).  Bias gradients are fp32
sums of the stored gradient operand.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import rng
from .bf16 import round_bf16

ALIGN = 64
MODEL_MLP = 1
MODEL_CNN = 2


@dataclass(frozen=True)
class Tensor:
    name: str
    shape: tuple
    fan_in: int

    @property
    def count(self) -> int:
        return int(np.prod(self.shape))


TENSORS = {
    MODEL_MLP: (
        Tensor("fc1.w", (512, 784), 784), Tensor("fc1.b", (512,), 784),
        Tensor("fc2.w", (512, 512), 512), Tensor("fc2.b", (512,), 512),
        Tensor("fc3.w", (10, 512), 512), Tensor("fc3.b", (10,), 512),
    ),
    MODEL_CNN: (
        Tensor("conv1.w", (32, 9), 9), Tensor("conv1.b", (32,), 9),
        Tensor("conv2.w", (64, 288), 288), Tensor("conv2.b", (64,), 288),
        Tensor("fc1.w", (128, 9216), 9216), Tensor("fc1.b", (128,), 9216),
        Tensor("fc2.w", (10, 128), 128), Tensor("fc2.b", (10,), 128),
    ),
}

MODEL_NAMES = {"mlp": MODEL_MLP, "cnn": MODEL_CNN}


def _round_up(x: int, a: int = ALIGN) -> int:
    return (x + a - 1) // a * a


def layout(model: int):
    """[(Tensor, offset)], param_count, param_stride -- restates tlk_model_tensor."""
    out, off = [], 0
    for t in TENSORS[model]:
        out.append((t, off))
        off = _round_up(off + t.count)
    return out, sum(t.count for t in TENSORS[model]), off


def init_params(model: int, seed: int) -> dict:
    return {
        t.name: rng.init_uniform(seed, i, t.count, t.fan_in).reshape(t.shape)
        for i, t in enumerate(TENSORS[model])
    }


def flatten_params(model: int, params: dict) -> np.ndarray:
    lay, _, stride = layout(model)
    flat = np.zeros(stride, np.float32)
    for t, off in lay:
        flat[off:off + t.count] = params[t.name].reshape(-1)
    return flat


def unflatten(model: int, flat: np.ndarray) -> dict:
    lay, _, _ = layout(model)
    return {t.name: flat[off:off + t.count].reshape(t.shape).copy() for t, off in lay}


# ------------------------------------------------------------------ pieces --
def _r(x, on):
    return round_bf16(x) if on else x.astype(np.float32, copy=False)


def head(h: np.ndarray, w: np.ndarray, b: np.ndarray, y: np.ndarray):
    """Last Linear + mean CE + its backward, fp32 (GPU: fused head kernel).

    Returns loss, dW, db, dh (pre-mask).
    """
    n = h.shape[0]
    logits = h @ w.T + b
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(s))[:, 0]
    loss = np.float32((lse - logits[np.arange(n), y]).sum() / np.float32(n))
    d = e / s
    d[np.arange(n), y] -= np.float32(1.0)
    d = (d / np.float32(n)).astype(np.float32)
    return loss, d.T @ h, d.sum(axis=0), d @ w


def mlp_step(p: dict, px: np.ndarray, y: np.ndarray, bf16: bool = True):
    """One forward+backward of the MLP; returns (loss, grads dict)."""
    x = px.astype(np.float32) / np.float32(256.0)
    w1, w2 = _r(p["fc1.w"], bf16), _r(p["fc2.w"], bf16)
    h1 = _r(np.maximum(x @ w1.T + p["fc1.b"], 0), bf16)
    h2 = _r(np.maximum(h1 @ w2.T + p["fc2.b"], 0), bf16)
    loss, g3w, g3b, dh2 = head(h2, p["fc3.w"], p["fc3.b"], y)
    dz2 = _r(dh2 * (h2 > 0), bf16)
    dh1 = dz2 @ w2
    dz1 = _r(dh1 * (h1 > 0), bf16)
    g = {
        "fc3.w": g3w, "fc3.b": g3b,
        "fc2.w": dz2.T @ h1, "fc2.b": dz2.sum(axis=0),
        "fc1.w": dz1.T @ x, "fc1.b": dz1.sum(axis=0),
    }
    return loss, g


def _taps(img: np.ndarray, out_hw: int) -> np.ndarray:
    """NHWC valid 3x3 im2col: [..., out, out, 9*C] with K index = tap*C + c."""
    cols = [img[:, kh:kh + out_hw, kw:kw + out_hw, :] for kh in range(3) for kw in range(3)]
    return np.concatenate(cols, axis=-1)


def cnn_step(p: dict, px: np.ndarray, y: np.ndarray, bf16: bool = True):
    """One forward+backward of the MNIST CNN (NHWC); returns (loss, grads)."""
    n = px.shape[0]
    x = (px.astype(np.float32) / np.float32(256.0)).reshape(n, 28, 28, 1)
    cols1 = _taps(x, 26)                                         # [n,26,26,9]
    h1 = _r(np.maximum(cols1 @ p["conv1.w"].T + p["conv1.b"], 0), bf16)   # [n,26,26,32]
    w2 = _r(p["conv2.w"], bf16)
    cols2 = _taps(h1, 24)                                        # [n,24,24,288]
    a2 = np.maximum(cols2 @ w2.T + p["conv2.b"], 0)              # [n,24,24,64]
    win = a2.reshape(n, 12, 2, 12, 2, 64).transpose(0, 1, 3, 2, 4, 5).reshape(n, 12, 12, 4, 64)
    idx = np.argmax(win, axis=3)                                 # first max in (dy,dx) order
    p2 = _r(np.take_along_axis(win, idx[:, :, :, None, :], axis=3)[:, :, :, 0, :], bf16)
    flat = p2.reshape(n, 9216)
    w3 = _r(p["fc1.w"], bf16)
    h3 = _r(np.maximum(flat @ w3.T + p["fc1.b"], 0), bf16)       # [n,128]
    loss, g4w, g4b, dh3 = head(h3, p["fc2.w"], p["fc2.b"], y)
    dz3 = _r(dh3 * (h3 > 0), bf16)
    dp2 = (dz3 @ w3).reshape(n, 12, 12, 64)
    onehot = (np.arange(4)[None, None, None, :, None] == idx[:, :, :, None, :])
    dwin = np.where(onehot & (p2[:, :, :, None, :] > 0), dp2[:, :, :, None, :], np.float32(0))
    dz2 = _r(dwin.reshape(n, 12, 12, 2, 2, 64).transpose(0, 1, 3, 2, 4, 5).reshape(n, 24, 24, 64), bf16)
    g2w = dz2.reshape(-1, 64).T @ cols2.reshape(-1, 288)
    dpad = np.pad(dz2, ((0, 0), (2, 2), (2, 2), (0, 0)))
    w2t = w2.reshape(64, 9, 32)
    dh1 = np.zeros((n, 26, 26, 32), np.float32)
    for kh in range(3):
        for kw in range(3):
            dh1 += dpad[:, 2 - kh:2 - kh + 26, 2 - kw:2 - kw + 26, :] @ w2t[:, kh * 3 + kw, :]
    dz1 = _r(dh1 * (h1 > 0), bf16)
    g = {
        "fc2.w": g4w, "fc2.b": g4b,
        "fc1.w": dz3.T @ flat, "fc1.b": dz3.sum(axis=0),
        "conv2.w": g2w, "conv2.b": dz2.reshape(-1, 64).sum(axis=0),
        "conv1.w": dz1.reshape(-1, 32).T @ cols1.reshape(-1, 9), "conv1.b": dz1.reshape(-1, 32).sum(axis=0),
    }
    return loss, g


STEP_FNS = {MODEL_MLP: mlp_step, MODEL_CNN: cnn_step}
