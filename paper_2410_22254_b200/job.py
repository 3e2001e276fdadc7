"""Job entry point: ``python -m paper_2410_22254_b200.job --model cnn --seed 3 ...``.

Run as an ordinary process (e.g. by the reference-style subprocess executor,
or by hand) it trains its one task on the GPU it was pinned to through
CUDA_VISIBLE_DEVICES, as a one-lane pack of libtlk -- the same kernels the
packed backend uses for K lanes.  Under ``run_plan(..., backend="packed")``
this argv is not spawned at all: the per-GPU worker loads it into a lane.

stdout: one JSON line {task summary}.  Exit 0 on success; 1 on failure with
the reason on stderr ("out of memory" for allocation failures, so the
reference's classify_failure sets oom_flag); 2 on a usage error.
"""

from __future__ import annotations

import json
import sys
import time

from .jobspec import parse_job_flags


def run_job(spec, device: int = 0) -> dict:
    from . import runtime as rt

    with rt.Context(device) as ctx:
        pack = ctx.pack(rt.MODELS[spec.model], spec.batch, 1, spec.steps)
        pack.load(0, seed=spec.seed, steps=spec.steps, optimizer=rt.OPTIMIZERS[spec.optim],
                  lr=spec.lr, beta1=spec.beta1, beta2=spec.beta2, eps=spec.eps,
                  weight_decay=spec.wd, momentum=spec.momentum)
        t0 = time.perf_counter()
        pack.run(spec.steps)
        ctx.sync()
        dt = time.perf_counter() - t0
        losses = pack.losses(0, spec.steps)
    return {"model": spec.model, "seed": spec.seed, "steps": spec.steps, "batch": spec.batch,
            "first_loss": float(losses[0]), "last_loss": float(losses[-1]),
            "samples_per_s": spec.steps * spec.batch / dt if dt > 0 else None}


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        spec = parse_job_flags(argv)
    except ValueError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 2
    try:
        out = run_job(spec)
    except Exception as exc:  # TlkError carries "out of memory" on OOM
        print(f"{type(exc).__name__}: {exc}", file=sys.stderr)
        return 1
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
