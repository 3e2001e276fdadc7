"""Training-task argv <-> job description.

A task in a parametric task list (reference plan.py:191-233) is an argv.  The
packed backend recognises the tasks it can run as lanes of a packed runtime
by their argv -- the job entry point of this package:

    python -m paper_2410_22254_b200.job --model cnn --seed 3 --lr 1e-3 --steps 200

(any python executable; ``tlk-job`` as argv[0] is accepted too).  Every other
argv is opaque, exactly as in the reference, and is run as a process.
"""

from __future__ import annotations

import argparse
import os
from dataclasses import asdict, dataclass

JOB_MODULE = "paper_2410_22254_b200.job"
MODELS = ("mlp", "cnn", "xformer", "gpt", "resnet18")
SEQ_MODELS = ("xformer", "gpt")  # batch = sequences
OPTIMIZERS = ("adam", "adamw", "sgd")


@dataclass(frozen=True)
class JobSpec:
    model: str = "mlp"
    seed: int = 0
    steps: int = 100
    batch: int = 64
    optim: str = "adam"
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    wd: float = 0.0
    momentum: float = 0.0

    def to_dict(self) -> dict:
        return asdict(self)

    def argv(self, python: str = "python3") -> list[str]:
        out = [python, "-m", JOB_MODULE]
        for k, v in asdict(self).items():
            out += [f"--{k}", str(v)]
        return out


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # raise instead of exiting
        raise ValueError(message)


def job_parser(prog: str = JOB_MODULE) -> argparse.ArgumentParser:
    ap = _Parser(prog=prog, add_help=False)
    d = JobSpec()
    ap.add_argument("--model", choices=MODELS, default=d.model)
    ap.add_argument("--seed", type=int, default=d.seed)
    ap.add_argument("--steps", type=int, default=d.steps)
    ap.add_argument("--batch", type=int, default=d.batch)
    ap.add_argument("--optim", choices=OPTIMIZERS, default=d.optim)
    ap.add_argument("--lr", type=float, default=d.lr)
    ap.add_argument("--beta1", type=float, default=d.beta1)
    ap.add_argument("--beta2", type=float, default=d.beta2)
    ap.add_argument("--eps", type=float, default=d.eps)
    ap.add_argument("--wd", type=float, default=d.wd)
    ap.add_argument("--momentum", type=float, default=d.momentum)
    return ap


def parse_job_flags(flags) -> JobSpec:
    ns = job_parser().parse_args(list(flags))
    spec = JobSpec(**vars(ns))
    if spec.steps < 1:
        raise ValueError("--steps must be >= 1")
    if spec.model in SEQ_MODELS:
        if spec.batch < 1 or spec.batch > 4096:
            raise ValueError("--batch (sequences) must be in [1, 4096]")
    elif spec.model == "resnet18":
        if spec.batch < 8 or spec.batch > 512 or spec.batch % 8:
            raise ValueError("--batch must be a multiple of 8 in [8, 512] for resnet18")
    elif spec.batch < 8 or spec.batch > 64 or spec.batch % 8:
        raise ValueError("--batch must be a multiple of 8 in [8, 64]")
    if spec.lr <= 0 or spec.eps <= 0:
        raise ValueError("--lr and --eps must be positive")
    return spec


def job_flags_of(argv) -> list[str] | None:
    """The flag list if ``argv`` invokes the job entry point, else None."""
    argv = list(argv)
    if not argv:
        return None
    if os.path.basename(argv[0]) == "tlk-job":
        return argv[1:]
    if "python" in os.path.basename(argv[0]) and len(argv) >= 3 and argv[1] == "-m" \
            and argv[2] == JOB_MODULE:
        return argv[3:]
    return None


def parse_task(argv) -> JobSpec | None:
    """JobSpec for a packable task argv, None for an opaque command.

    A job argv with invalid flags raises ValueError (reported as a task
    failure, like a child process exiting with a usage error).
    """
    flags = job_flags_of(argv)
    if flags is None:
        return None
    return parse_job_flags(flags)
