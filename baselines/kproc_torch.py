"""K-process time-sliced PyTorch baseline job (the paper's sharing mechanism).

One ordinary PyTorch training process per task; K of them pinned to the same
GPU through the slot env (CUDA_VISIBLE_DEVICES from the triples mapping) and
time-sliced by the driver -- exactly what the reference's run_plan does with
the paper's LeNet/ResNet jobs (executor.py:105-141).  This is
a BASELINE, not product code: bench.py launches K copies through
paper_2410_22254_b200.run_plan (subprocess backend == reference mechanism).

Timing: every process warms up (imports, CUDA context, cuDNN autotune, at
least 3 steps), then announces itself in ``--sync-dir`` and keeps stepping
until all ``--procs`` processes are ready; the common window starts 1 s after
the last announcement (or at wall-clock ``--t0`` without a sync dir).  Each
process counts completed steps (``loss.item()`` per step, as a logging
training loop does) during [start, start + duration].  The aggregate is
sum(steps * batch) / duration over the K processes.
"""

from __future__ import annotations

import argparse
import json
import time

import torch
import torch.nn as nn
import torch.nn.functional as F


class Net(nn.Module):
    """pytorch/examples MNIST Net without dropout (same shapes as TLK_MODEL_CNN)."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(1, 32, 3, 1)
        self.conv2 = nn.Conv2d(32, 64, 3, 1)
        self.fc1 = nn.Linear(9216, 128)
        self.fc2 = nn.Linear(128, 10)

    def forward(self, x):
        x = F.relu(self.conv1(x))
        x = F.max_pool2d(F.relu(self.conv2(x)), 2)
        x = F.relu(self.fc1(torch.flatten(x, 1)))
        return self.fc2(x)


class MLP(nn.Module):
    def __init__(self):
        super().__init__()
        self.fc1, self.fc2, self.fc3 = nn.Linear(784, 512), nn.Linear(512, 512), nn.Linear(512, 10)

    def forward(self, x):
        x = torch.flatten(x, 1)
        return self.fc3(F.relu(self.fc2(F.relu(self.fc1(x)))))


class GPT(nn.Module):
    """Pre-LN decoder (same shapes as TLK_MODEL_XFORMER / TLK_MODEL_GPT):
    learned positions, fused qkv, tanh-GELU MLP, untied head without bias."""

    def __init__(self, layers, d, heads, T, V):
        super().__init__()
        self.T, self.heads = T, heads
        self.wte, self.wpe = nn.Embedding(V, d), nn.Embedding(T, d)
        self.blocks = nn.ModuleList(nn.ModuleDict(dict(
            ln1=nn.LayerNorm(d), attn=nn.Linear(d, 3 * d), proj=nn.Linear(d, d),
            ln2=nn.LayerNorm(d), fc=nn.Linear(d, 4 * d), fc2=nn.Linear(4 * d, d)))
            for _ in range(layers))
        self.lnf, self.head = nn.LayerNorm(d), nn.Linear(d, V, bias=False)

    def forward(self, idx):
        B, T = idx.shape
        x = self.wte(idx) + self.wpe.weight[:T][None]
        for b in self.blocks:
            q, k, v = b.attn(b.ln1(x)).view(B, T, 3, self.heads, -1).unbind(2)
            y = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                               v.transpose(1, 2), is_causal=True)
            x = x + b.proj(y.transpose(1, 2).reshape(B, T, -1))
            x = x + b.fc2(F.gelu(b.fc(b.ln2(x)), approximate="tanh"))
        return self.head(self.lnf(x))


GPT_CFGS = {"xformer": (2, 256, 4, 128, 256), "gpt": (6, 384, 6, 256, 65)}


class BasicBlock(nn.Module):
    def __init__(self, cin, c, stride):
        super().__init__()
        self.conv1 = nn.Conv2d(cin, c, 3, stride, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(c)
        self.conv2 = nn.Conv2d(c, c, 3, 1, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(c)
        self.ds = None
        if stride != 1 or cin != c:
            self.ds = nn.Sequential(nn.Conv2d(cin, c, 1, stride, bias=False), nn.BatchNorm2d(c))

    def forward(self, x):
        o = F.relu(self.bn1(self.conv1(x)))
        o = self.bn2(self.conv2(o))
        return F.relu(o + (self.ds(x) if self.ds is not None else x))


class ResNet18(nn.Module):
    """CIFAR ResNet-18 (3x3 stem, no max-pool) -- same shapes as TLK_MODEL_RESNET18."""

    def __init__(self):
        super().__init__()
        self.stem = nn.Sequential(nn.Conv2d(3, 64, 3, 1, 1, bias=False), nn.BatchNorm2d(64), nn.ReLU())
        layers, cin = [], 64
        for c, s in ((64, 1), (128, 2), (256, 2), (512, 2)):
            layers += [BasicBlock(cin, c, s), BasicBlock(c, c, 1)]
            cin = c
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(512, 10)

    def forward(self, x):
        return self.fc(self.layers(self.stem(x)).mean(dim=(2, 3)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="cnn", choices=("cnn", "mlp", "xformer", "gpt", "resnet18"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--t0", type=float, default=0.0, help="wall-clock start of the timed window")
    ap.add_argument("--sync-dir", default="", help="rendezvous directory (start when all are warm)")
    ap.add_argument("--procs", type=int, default=1)
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--bf16", type=int, default=None,
                    help="1: torch.autocast(bfloat16); default 1 for the transformer / ResNet models")
    ap.add_argument("--steps", type=int, default=0,
                    help="run exactly this many steps and exit (a fixed-size training task, as in a "
                         "parametric job list); 0 = the timed-window mode above")
    ap.add_argument("--fast", type=int, default=0,
                    help="1: the strongest plain-PyTorch job: bf16 autocast, fused Adam, no per-step "
                         "host sync (loss read every 50 steps)")
    a = ap.parse_args()
    torch.manual_seed(a.seed)
    dev = torch.device("cuda")
    if a.bf16 is None:
        a.bf16 = int(a.model in GPT_CFGS or a.model == "resnet18" or bool(a.fast))
    if a.model in GPT_CFGS:
        cfg = GPT_CFGS[a.model]
        model = GPT(*cfg).to(dev)
    elif a.model == "resnet18":
        model = ResNet18().to(dev).to(memory_format=torch.channels_last)
    else:
        model = (Net() if a.model == "cnn" else MLP()).to(dev)
    if a.model == "resnet18":
        opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9)
    else:
        opt = torch.optim.Adam(model.parameters(), lr=a.lr, fused=bool(a.fast))
    torch.backends.cudnn.benchmark = True
    nstep = [0]

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=bool(a.bf16)):
            if a.model in GPT_CFGS:
                T, V = GPT_CFGS[a.model][3:]
                toks = torch.randint(0, V, (a.batch, T + 1), device=dev)
                logits = model(toks[:, :-1])
                loss = F.cross_entropy(logits.reshape(-1, V).float(), toks[:, 1:].reshape(-1))
            elif a.model == "resnet18":
                x = torch.randn(a.batch, 3, 32, 32, device=dev).to(memory_format=torch.channels_last)
                y = torch.randint(0, 10, (a.batch,), device=dev)
                loss = F.cross_entropy(model(x).float(), y)
            else:
                x = torch.rand(a.batch, 1, 28, 28, device=dev)
                y = torch.randint(0, 10, (a.batch,), device=dev)
                loss = F.cross_entropy(model(x), y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        nstep[0] += 1
        if a.fast and nstep[0] % 50:
            return None
        return loss.item()

    if a.steps:
        t_start = time.time()
        last = None
        for _ in range(a.steps):
            v = step()
            last = v if v is not None else last
        torch.cuda.synchronize()
        el = time.time() - t_start
        print(json.dumps({"steps": a.steps, "elapsed_s": el, "batch": a.batch, "last_loss": last,
                          "samples_per_s": a.steps * a.batch / el}))
        return 0

    warm = 0
    while warm < 3 or (not a.sync_dir and time.time() < a.t0):
        step()
        warm += 1
    if a.sync_dir:
        import glob
        import os
        open(os.path.join(a.sync_dir, f"ready_{a.seed}"), "w").close()
        deadline = time.time() + 900
        while True:
            ready = glob.glob(os.path.join(a.sync_dir, "ready_*"))
            if len(ready) >= a.procs:
                t0 = max(os.path.getmtime(p) for p in ready) + 1.0
                break
            if time.time() > deadline:
                print(json.dumps({"error": "rendezvous timed out", "ready": len(ready)}))
                return 3
            step()
            warm += 1
        while time.time() < t0:
            step()
            warm += 1
        a.t0 = t0
    elif time.time() > a.t0 + 0.5 * a.duration:
        print(json.dumps({"error": "warm-up overran the timed window", "warm": warm}))
        return 3
    start = time.time()
    steps = 0
    while time.time() < a.t0 + a.duration:
        step()
        steps += 1
    elapsed = time.time() - start
    print(json.dumps({"steps": steps, "elapsed_s": elapsed, "batch": a.batch, "warm_steps": warm,
                      "samples_per_s": steps * a.batch / elapsed}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
