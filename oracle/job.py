"""CPU oracle job: train one task in numpy (test infrastructure / CPU baseline).

``python -m oracle.job --model cnn --seed 3 --steps 20 [--bf16 0|1] [--json]``
accepts the same flags as the product's job entry point
(``python -m paper_2410_22254_b200.job``), so one parametric task list drives
the packed runtime, the K-process PyTorch baseline and this CPU path.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import gpt, models, optim, resnet, rng

GPT_MODELS = {"xformer": gpt.MODEL_XFORMER, "gpt": gpt.MODEL_GPT}
RESNET_MODELS = {"resnet18": resnet.MODEL_RESNET18}


def add_job_args(ap: argparse.ArgumentParser) -> None:
    ap.add_argument("--model", choices=sorted(models.MODEL_NAMES) + sorted(GPT_MODELS) + sorted(RESNET_MODELS),
                    default="mlp")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--optim", choices=sorted(optim.OPT_NAMES), default="adam")
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--beta1", type=float, default=0.9)
    ap.add_argument("--beta2", type=float, default=0.999)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--wd", type=float, default=0.0)
    ap.add_argument("--momentum", type=float, default=0.0)


def train(model: int, seed: int, steps: int, batch: int, opt: optim.OptState,
          bf16: bool = True, warmup: int = 1):
    """Run ``steps`` steps; returns (losses [steps], final flat params, seconds/step).

    seconds/step is measured over the steps after the first ``warmup`` ones
    (all steps if there are not more than ``warmup``).
    """
    params = models.init_params(model, seed)
    flat = models.flatten_params(model, params)
    step_fn = models.STEP_FNS[model]
    losses = np.zeros(steps, np.float32)
    warmup = warmup if steps > warmup else 0
    t0 = time.perf_counter()
    for t in range(steps):
        if t == warmup:
            t0 = time.perf_counter()
        px, y = rng.batch(seed, t, batch)
        loss, g = step_fn(models.unflatten(model, flat), px, y, bf16=bf16)
        gflat = models.flatten_params(model, g)
        flat = optim.step(opt, flat, gflat)
        losses[t] = loss
    per_step = (time.perf_counter() - t0) / max(1, steps - warmup)
    return losses, flat, per_step


def train_gpt(cfg, seed: int, steps: int, opt: optim.OptState, bf16: bool = True, warmup: int = 1,
              batch: int | None = None):
    """Transformer job (oracle/gpt.py); returns (losses, final flat params, s/step)."""
    flat = gpt.flatten(cfg, gpt.init_params(cfg, seed))
    losses = np.zeros(steps, np.float32)
    warmup = warmup if steps > warmup else 0
    t0 = time.perf_counter()
    for t in range(steps):
        if t == warmup:
            t0 = time.perf_counter()
        toks = gpt.tokens(cfg, seed, t, batch)
        loss, g = gpt.gpt_step(cfg, gpt.unflatten(cfg, flat), toks, bf16=bf16)
        flat = optim.step(opt, flat, gpt.flatten(cfg, g))
        losses[t] = loss
    per_step = (time.perf_counter() - t0) / max(1, steps - warmup)
    return losses, flat, per_step


def train_resnet(seed: int, steps: int, batch: int, opt: optim.OptState, bf16: bool = True,
                 warmup: int = 1):
    """ResNet-18 job (oracle/resnet.py); returns (losses, final flat params, s/step)."""
    flat = resnet.flatten(resnet.init_params(seed))
    losses = np.zeros(steps, np.float32)
    warmup = warmup if steps > warmup else 0
    t0 = time.perf_counter()
    for t in range(steps):
        if t == warmup:
            t0 = time.perf_counter()
        x, y = resnet.batch(seed, t, batch)
        loss, g = resnet.resnet_step(resnet.unflatten(flat), x, y, bf16=bf16)
        flat = optim.step(opt, flat, resnet.flatten(g))
        losses[t] = loss
    per_step = (time.perf_counter() - t0) / max(1, steps - warmup)
    return losses, flat, per_step


def opt_from_args(a) -> optim.OptState:
    return optim.OptState(kind=optim.OPT_NAMES[a.optim], lr=a.lr, beta1=a.beta1, beta2=a.beta2,
                          eps=a.eps, weight_decay=a.wd, momentum=a.momentum)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="oracle.job")
    add_job_args(ap)
    ap.add_argument("--bf16", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1, help="steps excluded from the timing")
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args(argv)
    if a.model in RESNET_MODELS:
        losses, _, per_step = train_resnet(a.seed, a.steps, a.batch, opt_from_args(a), bool(a.bf16),
                                           warmup=a.warmup)
    elif a.model in GPT_MODELS:
        cfg = gpt.CFGS[GPT_MODELS[a.model]]
        losses, _, per_step = train_gpt(cfg, a.seed, a.steps, opt_from_args(a), bool(a.bf16),
                                        warmup=a.warmup, batch=a.batch)
    else:
        model = models.MODEL_NAMES[a.model]
        losses, _, per_step = train(model, a.seed, a.steps, a.batch, opt_from_args(a),
                                    bool(a.bf16), warmup=a.warmup)
    out = {
        "model": a.model, "seed": a.seed, "steps": a.steps, "batch": a.batch,
        "timed_steps": a.steps - (a.warmup if a.steps > a.warmup else 0),
        "seconds_per_step": per_step,
        "samples_per_s": a.batch / per_step if per_step > 0 else None,
        "first_loss": float(losses[0]), "last_loss": float(losses[-1]),
    }
    print(json.dumps(out) if a.json else out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
