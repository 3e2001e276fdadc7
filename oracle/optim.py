"""Optimizers, restated op-for-op with the CUDA kernel (csrc/optim.cu).

Every fp32 operation below is a single IEEE-rounded numpy float32 op in the
same order as the kernel's __f*_rn intrinsics, so given identical gradients
the update is bit-exact (tests/test_gpu_parity.py::test_adam_bit_exact).

Semantics follow torch.optim (PyTorch 2.x, single-tensor path):
Adam   m = m + (1-b1)(g - m);  v = v*b2 + (g*g)(1-b2)
       p = p - step_size * (m / (sqrt(v)/bc2s + eps)),
       step_size = lr / (1 - b1^t), bc2s = sqrt(1 - b2^t) (both in float64,
       b^t by repeated multiplication), L2 weight decay g = g + wd*p.
AdamW  p = p * (1 - lr*wd) before the Adam update (decoupled decay).
SGD    g = g + wd*p; buf = buf*mu + g (buf = g at t=1); p = p - lr*buf.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ADAM, ADAMW, SGD = 1, 2, 3
OPT_NAMES = {"adam": ADAM, "adamw": ADAMW, "sgd": SGD}

f32 = np.float32


@dataclass
class OptState:
    kind: int
    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    momentum: float = 0.0
    t: int = 0
    b1t: float = 1.0
    b2t: float = 1.0
    m: np.ndarray | None = field(default=None, repr=False)
    v: np.ndarray | None = field(default=None, repr=False)

    def scalars(self):
        """Per-step fp32 scalars, as the device computes them (csrc/optim.cu)."""
        lr = float(f32(self.lr))
        b1 = float(f32(self.beta1))
        b2 = float(f32(self.beta2))
        b1t, b2t = self.b1t * b1, self.b2t * b2
        return dict(
            b1t=b1t, b2t=b2t,
            step_size=f32(lr / (1.0 - b1t)),
            bc2s=f32(math.sqrt(1.0 - b2t)),
            w1=f32(1.0 - b1), w2=f32(1.0 - b2), b2=f32(b2),
            eps=f32(self.eps), wd=f32(self.weight_decay), lr=f32(lr),
            decay=f32(1.0 - lr * float(f32(self.weight_decay))),
            mu=f32(self.momentum),
        )


def step(st: OptState, p: np.ndarray, g: np.ndarray) -> np.ndarray:
    """In-place-style update on flat fp32 arrays; returns the new params."""
    if st.m is None:
        st.m = np.zeros_like(p)
        st.v = np.zeros_like(p)
    s = st.scalars()
    p = p.astype(f32, copy=True)
    g = g.astype(f32, copy=False)
    if st.kind in (ADAM, ADAMW):
        if st.kind == ADAMW:
            p = p * s["decay"]
        elif st.weight_decay != 0.0:
            g = g + p * s["wd"]
        st.m = st.m + s["w1"] * (g - st.m)
        st.v = st.v * s["b2"] + (g * g) * s["w2"]
        denom = np.sqrt(st.v) / s["bc2s"] + s["eps"]
        p = p - s["step_size"] * (st.m / denom)
    elif st.kind == SGD:
        if st.weight_decay != 0.0:
            g = g + p * s["wd"]
        if st.momentum != 0.0:
            st.m = g.copy() if st.t == 0 else st.m * s["mu"] + g
            g = st.m
        p = p - s["lr"] * g
    else:
        raise ValueError(f"unknown optimizer {st.kind}")
    st.t += 1
    st.b1t, st.b2t = s["b1t"], s["b2t"]
    return p.astype(f32)
