"""Generate PyTorch-CPU golden vectors that pin the numpy oracle (oracle/models.py).

The reference (trilaunch) contains no training arithmetic -- its tasks are
opaque argv (executor.py:199) and SPEC.md:10 puts "actual ML training
(LeNet-4, ResNet-18, PyTorch)" out of its scope -- while PAPER.md:96-101 says
the paper's jobs are PyTorch MNIST/ResNet trainings.  So PyTorch CPU, fp32,
is the authority the oracle is pinned to: same init (loaded from the oracle's
counter RNG), same synthetic batches, torch's own layers / F.cross_entropy /
torch.optim.  Outputs go to tests/golden/torch_golden.npz (small: loss curves,
per-tensor norms and 4096 sampled weights per run).

Run:  python tests/golden/gen_torch_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import models, rng  # noqa: E402

RUNS = [
    # name, model, batch, steps, optim, kwargs
    ("mlp_adam", models.MODEL_MLP, 16, 6, "adam", dict(lr=1e-3)),
    ("mlp_adamw", models.MODEL_MLP, 16, 4, "adamw", dict(lr=2e-3, weight_decay=0.1)),
    ("mlp_sgd", models.MODEL_MLP, 16, 4, "sgd", dict(lr=0.05, momentum=0.9, weight_decay=1e-4)),
    ("cnn_adam", models.MODEL_CNN, 4, 3, "adam", dict(lr=1e-3)),
]
SEED = 11
SAMPLES = 4096


def to_torch_layout(model, name, a):
    if model == models.MODEL_CNN:
        if name == "conv1.w":
            return a.reshape(32, 1, 3, 3)
        if name == "conv2.w":
            return a.reshape(64, 3, 3, 32).transpose(0, 3, 1, 2)
        if name == "fc1.w":
            return a.reshape(128, 12, 12, 64).transpose(0, 3, 1, 2).reshape(128, 9216)
    return a


def from_torch_layout(model, name, a):
    if model == models.MODEL_CNN:
        if name == "conv1.w":
            return a.reshape(32, 9)
        if name == "conv2.w":
            return a.transpose(0, 2, 3, 1).reshape(64, 288)
        if name == "fc1.w":
            return a.reshape(128, 64, 12, 12).transpose(0, 2, 3, 1).reshape(128, 9216)
    return a


def forward(model, P, x):
    if model == models.MODEL_MLP:
        h = F.relu(F.linear(x, P["fc1.w"], P["fc1.b"]))
        h = F.relu(F.linear(h, P["fc2.w"], P["fc2.b"]))
        return F.linear(h, P["fc3.w"], P["fc3.b"])
    n = x.shape[0]
    h = F.relu(F.conv2d(x.reshape(n, 1, 28, 28), P["conv1.w"], P["conv1.b"]))
    h = F.relu(F.conv2d(h, P["conv2.w"], P["conv2.b"]))
    h = F.max_pool2d(h, 2).flatten(1)
    h = F.relu(F.linear(h, P["fc1.w"], P["fc1.b"]))
    return F.linear(h, P["fc2.w"], P["fc2.b"])


def run(name, model, batch, steps, opt, kw):
    init = models.init_params(model, SEED)
    P = {k: torch.tensor(np.ascontiguousarray(to_torch_layout(model, k, v)), requires_grad=True)
         for k, v in init.items()}
    params = list(P.values())
    if opt == "adam":
        o = torch.optim.Adam(params, foreach=False, **kw)
    elif opt == "adamw":
        o = torch.optim.AdamW(params, foreach=False, **kw)
    else:
        o = torch.optim.SGD(params, foreach=False, **kw)
    losses = []
    for t in range(steps):
        px, y = rng.batch(SEED, t, batch)
        x = torch.tensor(px.astype(np.float32) / 256.0)
        loss = F.cross_entropy(forward(model, P, x), torch.tensor(y, dtype=torch.long))
        o.zero_grad()
        loss.backward()
        o.step()
        losses.append(loss.item())
    final = {k: from_torch_layout(model, k, v.detach().numpy()) for k, v in P.items()}
    flat = models.flatten_params(model, final)
    _, count, stride = models.layout(model)
    idx = np.linspace(0, stride - 1, SAMPLES).astype(np.int64)
    norms = np.array([np.linalg.norm(final[t.name]) for t in models.TENSORS[model]], np.float64)
    return {f"{name}/losses": np.array(losses, np.float64), f"{name}/idx": idx,
            f"{name}/sample": flat[idx], f"{name}/norms": norms}


def main():
    torch.manual_seed(0)
    torch.set_num_threads(1)
    out = {}
    for r in RUNS:
        out.update(run(*r))
    path = os.path.join(HERE, "torch_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
