"""Command line: the reference's hot-path modes with a packed backend switch.

    python -m paper_2410_22254_b200 --mode plan --triple 1,8,1 --tasks jobs.jsonl --gpus 1
    python -m paper_2410_22254_b200 --mode exec --triple 1,8,1 --tasks jobs.jsonl --gpus 1 --backend packed

Mirrors the reference CLI's ``plan`` and ``exec`` modes (cli.py:99-142,
264-337): same flags, same settings precedence (flag > --config JSON >
default), same artefacts (node_###.sh + plan_summary.json; run_report.json
in a runs/<ts>-<mode> directory), same exit codes (ConfigError/TripleError
-> 2; exec -> min(failures, 125)), and the exec-mode telemetry sampler
(``--provider {none,host,command,const,nvml} --interval --query-cmd`` ->
telemetry.csv in the reference's schema, cli.py:227-249,298-329; ``nvml`` is
new: the packed workers' GPUs through NVML).  New: ``--backend
{subprocess,packed}`` and ``--chunk``.  The reference's sim/sweep/report modes model or tabulate
runs without touching a GPU; they are outside the packed hot path
 and are rejected here with exit status 2.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

from .core import NodeSpec, TripleError, TripleSpec, validate_triple
from .executor import BACKENDS, run_plan
from .plan import TaskDef, build_plan, emit_script, load_workload, plan_summary
from .telemetry import (DEFAULT_QUERY_COMMAND, CommandProvider, ConstantProvider, GpuReading, HostProvider,
                        NvmlProvider, run_sampler, write_series_csv)

QUERY_CMD_ENV = "TRILAUNCH_QUERY_CMD"  # reference cli.py:53

DEFAULTS = {
    "cores": os.cpu_count() or 1,
    "gpus": 0,
    "gpu_mem": 32768,
    "strict": False,
    "outdir": "runs",
    "node_index": 0,
    "backend": "subprocess",
    "chunk": 64,
    "admit_mem": False,
    "provider": "none",
    "interval": 1.0,
    "query_cmd": os.environ.get(QUERY_CMD_ENV, DEFAULT_QUERY_COMMAND),
}
OUT_OF_SCOPE = ("sim", "sweep", "report")


class ConfigError(ValueError):
    """Bad or missing user input (exit status 2)."""


class _Settings:
    def __init__(self, args, config):
        self._a, self._c = args, config

    def get(self, name, default=None):
        v = getattr(self._a, name, None)
        if v is not None:
            return v
        if name in self._c:
            return self._c[name]
        return DEFAULTS.get(name, default)


def _parser():
    p = argparse.ArgumentParser(prog="paper_2410_22254_b200",
                                description="Triples-mode launcher with a packed B200 backend.")
    p.add_argument("--mode", required=True, choices=("plan", "exec") + OUT_OF_SCOPE)
    p.add_argument("--config")
    p.add_argument("--triple")
    p.add_argument("--tasks")
    p.add_argument("--num-tasks", type=int)
    p.add_argument("--cores", type=int)
    p.add_argument("--gpus", type=int)
    p.add_argument("--gpu-mem", type=int)
    p.add_argument("--strict", action="store_true", default=None)
    p.add_argument("--outdir")
    p.add_argument("--run-name")
    p.add_argument("--node-index", type=int)
    p.add_argument("--timeout", type=float)
    p.add_argument("--backend", choices=BACKENDS)
    p.add_argument("--chunk", type=int, help="packed backend: steps per graph-replay chunk")
    p.add_argument("--admit-mem", action="store_true", default=None,
                   help="packed backend: admit tasks against --gpu-mem MiB per GPU (per-task OOM)")
    p.add_argument("--provider", choices=("none", "host", "command", "const", "nvml"),
                   help="telemetry source while executing (telemetry.csv)")
    p.add_argument("--query-cmd", help=f"device query command for --provider command (or {QUERY_CMD_ENV})")
    p.add_argument("--interval", type=float, help="sampling interval in seconds")
    return p


def _triple(s):
    raw = s.get("triple")
    if raw is None:
        raise ConfigError("--triple NNODE,NPPN,NTPP is required for this mode")
    try:
        return TripleSpec(*map(int, raw)) if isinstance(raw, (list, tuple)) else TripleSpec.parse(str(raw))
    except (TypeError, ValueError) as exc:
        raise ConfigError(f"bad triple {raw!r}: {exc}") from exc


def _node(s):
    gpus = int(s.get("gpus"))
    try:
        return NodeSpec(cores=int(s.get("cores")), gpus=gpus,
                        gpu_mem_mib=int(s.get("gpu_mem")) if gpus > 0 else 0)
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc


def _tasks(s):
    path, num = s.get("tasks"), s.get("num_tasks")
    if path and num:
        raise ConfigError("give either --tasks or --num-tasks, not both")
    if path:
        try:
            tasks = load_workload(path)
        except (OSError, ValueError, KeyError) as exc:
            raise ConfigError(f"cannot load workload {path}: {exc}") from exc
        if not tasks:
            raise ConfigError(f"workload {path} holds no tasks")
        return tasks
    if num is not None:
        if int(num) < 1:
            raise ConfigError(f"--num-tasks must be >= 1, got {num}")
        return [TaskDef(i, ("true",)) for i in range(int(num))]
    raise ConfigError("a workload is required: --tasks FILE or --num-tasks N")


def _plan_inputs(s):
    triple, node, tasks = _triple(s), _node(s), _tasks(s)
    strict = bool(s.get("strict"))
    validate_triple(triple, node, strict=strict).raise_for_error()
    for w in validate_triple(triple, node).warnings:
        print(f"warning: {w}", file=sys.stderr)
    try:
        return triple, node, build_plan(tasks, triple, node, strict=strict)
    except TripleError:
        raise
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc


def _run_dir(s, mode):
    base = Path(s.get("outdir"))
    name = s.get("run_name") or time.strftime("%Y%m%d-%H%M%S") + "-" + mode
    d, n = base / name, 2
    while d.exists():
        d, n = base / f"{name}-{n}", n + 1
    d.mkdir(parents=True)
    return d


def _write_json(path, obj):
    Path(path).write_text(json.dumps(obj, indent=2) + "\n")


def _mode_plan(s):
    triple, _, plan = _plan_inputs(s)
    d = _run_dir(s, "plan")
    _write_json(d / "plan_summary.json", plan_summary(plan).to_json_dict())
    for i in range(triple.nnode):
        p = d / f"node_{i:03d}.sh"
        p.write_text(emit_script(plan, i))
        p.chmod(0o755)
        print(p)
    print(d / "plan_summary.json")
    return 0


def _provider(s, node):
    """Telemetry provider of an exec run (reference cli.py:227-249, + nvml)."""
    kind = s.get("provider")
    if kind == "none":
        return None
    if not float(s.get("interval")) > 0:
        raise ConfigError("--interval must be positive")
    if kind == "host":
        if node.gpus > 0:
            raise ConfigError("host provider reports no devices; use --provider command when --gpus > 0")
        return HostProvider()
    if kind in ("command", "nvml") and node.gpus < 1:
        raise ConfigError(f"{kind} provider needs --gpus >= 1")
    if kind == "command":
        return CommandProvider(ngpus=node.gpus, command=str(s.get("query_cmd")))
    if kind == "nvml":
        try:
            return NvmlProvider(node.gpus)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
    if kind == "const":
        return ConstantProvider(gpu_readings=tuple(GpuReading(0.0, 0) for _ in range(node.gpus)))
    raise ConfigError(f"unknown provider {kind!r}")


def _mode_exec(s):
    triple, node, plan = _plan_inputs(s)
    ni = int(s.get("node_index"))
    if not 0 <= ni < triple.nnode:
        raise ConfigError(f"--node-index {ni} outside 0..{triple.nnode - 1}")
    provider = _provider(s, node)
    d = _run_dir(s, "exec")
    stop, box, sampler = threading.Event(), {}, None
    if provider is not None:
        interval = float(s.get("interval"))
        sampler = threading.Thread(target=lambda: box.setdefault("series", run_sampler(provider, interval, stop)),
                                   name="sampler", daemon=True)
        sampler.start()
    t = s.get("timeout")
    backend = s.get("backend")
    opts = None
    if backend == "packed":
        opts = {"chunk": int(s.get("chunk"))}
        if s.get("admit_mem"):
            opts["mem_limit_mib"] = node.gpu_mem_mib
    try:
        report = run_plan(plan, ni, timeout_s=float(t) if t is not None else None, log_dir=d / "logs",
                          backend=backend, packed_options=opts)
    finally:
        if sampler is not None:
            stop.set()
            sampler.join()
            if "series" in box:
                write_series_csv(box["series"], d / "telemetry.csv")
    report.write_json(d / "run_report.json")
    print(f"elapsed_ms={report.elapsed_ms} failures={report.failures} "
          f"peak_concurrency={report.max_observed_concurrency}")
    print(d / "run_report.json")
    return report.exit_code


def run_cli(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    config = {}
    if args.config:
        try:
            config = json.loads(Path(args.config).read_text())
        except (OSError, json.JSONDecodeError) as exc:
            print(f"error: cannot read config {args.config}: {exc}", file=sys.stderr)
            return 2
        if not isinstance(config, dict):
            print(f"error: config {args.config} must hold a JSON object", file=sys.stderr)
            return 2
    s = _Settings(args, config)
    try:
        if args.mode in OUT_OF_SCOPE:
            raise ConfigError(f"--mode {args.mode} is not part of the packed hot path "
                              "(use the reference trilaunch for simulation/reporting)")
        return {"plan": _mode_plan, "exec": _mode_exec}[args.mode](s)
    except (ConfigError, TripleError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


def main() -> None:
    sys.exit(run_cli())


if __name__ == "__main__":
    main()
