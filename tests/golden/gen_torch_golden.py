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

from oracle import gpt, models, resnet, rng  # noqa: E402

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


GPT_RUNS = [
    # name, cfg, steps, optim, kwargs
    ("gpt_small_adamw", gpt.GptCfg(2, 64, 2, 16, 17, 4), 3, "adamw", dict(lr=3e-3, weight_decay=0.1)),
    ("xformer_small_adam", gpt.GptCfg(1, 32, 2, 8, 256, 2), 3, "adam", dict(lr=1e-3)),
]


def gpt_forward(cfg, P, toks):
    """Independent torch implementation of oracle/gpt.py's model."""
    B, T, d, H = toks.shape[0], cfg.T, cfg.d, cfg.heads
    dh = d // H
    inp = toks[:, :-1]
    x = P["wte"][inp] + P["wpe"][:T][None]
    mask = torch.tril(torch.ones(T, T, dtype=torch.bool))
    for l in range(cfg.layers):
        q_ = f"h{l}."
        a = F.layer_norm(x, (d,), P[q_ + "ln1.g"], P[q_ + "ln1.b"], eps=1e-5)
        qkv = F.linear(a, P[q_ + "attn.w"], P[q_ + "attn.b"]).view(B, T, 3, H, dh)
        q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        s = (q @ k.transpose(-1, -2)) / (dh ** 0.5)
        s = s.masked_fill(~mask, float("-inf"))
        y = torch.softmax(s, dim=-1) @ v
        x = x + F.linear(y.transpose(1, 2).reshape(B, T, d), P[q_ + "proj.w"], P[q_ + "proj.b"])
        m = F.layer_norm(x, (d,), P[q_ + "ln2.g"], P[q_ + "ln2.b"], eps=1e-5)
        f = F.gelu(F.linear(m, P[q_ + "fc.w"], P[q_ + "fc.b"]), approximate="tanh")
        x = x + F.linear(f, P[q_ + "fc2.w"], P[q_ + "fc2.b"])
    x = F.layer_norm(x, (d,), P["lnf.g"], P["lnf.b"], eps=1e-5)
    return F.linear(x, P["head.w"])


def run_gpt(name, cfg, steps, opt, kw):
    init = gpt.init_params(cfg, SEED)
    P = {k: torch.tensor(v, requires_grad=True) for k, v in init.items()}
    params = list(P.values())
    o = (torch.optim.AdamW if opt == "adamw" else torch.optim.Adam)(params, foreach=False, **kw)
    losses = []
    for t in range(steps):
        toks = torch.tensor(gpt.tokens(cfg, SEED, t), dtype=torch.long)
        logits = gpt_forward(cfg, P, toks)
        loss = F.cross_entropy(logits.reshape(-1, cfg.V), toks[:, 1:].reshape(-1))
        o.zero_grad()
        loss.backward()
        o.step()
        losses.append(loss.item())
    final = {k: v.detach().numpy() for k, v in P.items()}
    flat = gpt.flatten(cfg, final)
    idx = np.linspace(0, flat.size - 1, SAMPLES).astype(np.int64)
    norms = np.array([np.linalg.norm(final[n]) for n, *_ in gpt.tensors(cfg)], np.float64)
    return {f"{name}/losses": np.array(losses, np.float64), f"{name}/idx": idx,
            f"{name}/sample": flat[idx], f"{name}/norms": norms}


RESNET_RUNS = [
    # name, batch, steps, optim, kwargs
    ("resnet18_sgd", 16, 2, "sgd", dict(lr=0.01, momentum=0.0)),
]


def resnet_forward(P, x):
    """Independent torch implementation of oracle/resnet.py's model (NCHW)."""
    def conv(h, w, stride):
        w = w.permute(0, 3, 1, 2)  # (co, kh, kw, ci) -> (co, ci, kh, kw)
        return F.conv2d(h, w, stride=stride, padding=(w.shape[-1] - 1) // 2)

    def bn(h, g, b):
        return F.batch_norm(h, None, None, g, b, training=True, eps=1e-5)

    h = x.permute(0, 3, 1, 2)
    h = F.relu(bn(conv(h, P["stem.w"], 1), P["bn0.g"], P["bn0.b"]))
    for s, (C, stride) in enumerate(resnet.STAGES):
        for b in range(2):
            q = f"l{s + 1}.{b}."
            st = stride if b == 0 else 1
            o = F.relu(bn(conv(h, P[q + "conv1.w"], st), P[q + "bn1.g"], P[q + "bn1.b"]))
            o = bn(conv(o, P[q + "conv2.w"], 1), P[q + "bn2.g"], P[q + "bn2.b"])
            short = bn(conv(h, P[q + "ds.w"], st), P[q + "dsbn.g"], P[q + "dsbn.b"]) if q + "ds.w" in P else h
            h = F.relu(o + short)
    return F.linear(h.mean(dim=(2, 3)), P["fc.w"], P["fc.b"])


def run_resnet(name, batch, steps, opt, kw):
    """float64: batch-statistics BN at batch 8 is ill-conditioned enough that
    torch's own fp32 CPU path differs from fp64 by up to ~35% on some
    gradients; the oracle (fp32, centred variance) is pinned to fp64."""
    init = resnet.init_params(SEED)
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in init.items()}
    o = torch.optim.SGD(list(P.values()), foreach=False, **kw)
    losses = []
    for t in range(steps):
        x, y = resnet.batch(SEED, t, batch)
        loss = F.cross_entropy(resnet_forward(P, torch.tensor(x, dtype=torch.float64)),
                               torch.tensor(y, dtype=torch.long))
        o.zero_grad()
        loss.backward()
        o.step()
        losses.append(loss.item())
    final = {k: v.detach().numpy().astype(np.float32) for k, v in P.items()}
    flat = resnet.flatten(final)
    idx = np.linspace(0, flat.size - 1, SAMPLES).astype(np.int64)
    norms = np.array([np.linalg.norm(final[n]) for n, *_ in resnet.tensors()], np.float64)
    return {f"{name}/losses": np.array(losses, np.float64), f"{name}/idx": idx,
            f"{name}/sample": flat[idx], f"{name}/norms": norms}


def main():
    torch.manual_seed(0)
    torch.set_num_threads(1)
    out = {}
    for r in RUNS:
        out.update(run(*r))
    for r in GPT_RUNS:
        out.update(run_gpt(*r))
    for r in RESNET_RUNS:
        out.update(run_resnet(*r))
    path = os.path.join(HERE, "torch_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
