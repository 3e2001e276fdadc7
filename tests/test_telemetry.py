"""Exec-mode telemetry of this package (the reference's own telemetry tests
run against our module in test_reference_suite.py)."""
import csv
import json
import sys

import pytest

from paper_2410_22254_b200 import cli, telemetry as tm


def test_exec_writes_reference_schema_telemetry(tmp_path):
    (tmp_path / "w.txt").write_text("sleep 0.2\nsleep 0.2\nsleep 0.2\n")
    rc = cli.run_cli(["--mode", "exec", "--triple", "1,2,1", "--tasks", str(tmp_path / "w.txt"), "--gpus", "2",
                      "--provider", "const", "--interval", "0.01", "--outdir", str(tmp_path),
                      "--run-name", "r"])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "r" / "telemetry.csv")))
    assert rows[0] == ["t_s", "cpu_load", "sys_mem_mib", "gpu0_util", "gpu0_mem_mib", "gpu1_util", "gpu1_mem_mib"]
    series = tm.read_series_csv(tmp_path / "r" / "telemetry.csv")
    assert all(len(s.gpu) == 2 for s in series.samples)
    assert json.loads((tmp_path / "r" / "run_report.json").read_text())["exit_code"] == 0


def test_provider_validation(tmp_path):
    base = ["--mode", "exec", "--triple", "1,1,1", "--num-tasks", "1", "--outdir", str(tmp_path)]
    assert cli.run_cli(base + ["--gpus", "1", "--provider", "host"]) == 2
    assert cli.run_cli(base + ["--gpus", "0", "--provider", "nvml"]) == 2
    assert cli.run_cli(base + ["--gpus", "1", "--provider", "const", "--interval", "0"]) == 2


def test_nvml_failures_are_gaps():
    """Without a usable NVML (this container) every read is a SampleError,
    which the sampler records as a gap -- never a crash or a fake reading."""
    prov = tm.NvmlProvider(1)
    try:
        prov.read()
    except tm.SampleError:
        pass  # no driver here
    ticks = iter([False, False, True])
    series = tm.run_sampler(prov, 0.5, None, waiter=lambda _: next(ticks))
    assert len(series.samples) + len(series.gaps) == 2


def test_virtual_clock_series_is_byte_identical():
    prov = tm.TraceProvider([(1.0, 10, (tm.GpuReading(0.5, 7),)), (2.0, 11, (tm.GpuReading(1.0, 8),))])
    ticks = iter([False, False, False, True])
    s = tm.run_sampler(prov, 0.25, None, waiter=lambda _: next(ticks))
    assert [x.t for x in s.samples] == [0.25, 0.5] and s.gaps == [0.75]
    text = tm.format_series_csv(s)
    assert text == tm.format_series_csv(s)
    assert text.splitlines()[-1] == "0.75,,,,"
    st = tm.series_stats(s, "gpu0_util")
    assert (st.min, st.avg, st.max, st.n_samples) == (0.5, 0.75, 1.0, 2)
