"""Our CLI's plan/exec modes keep the reference's artefacts and exit codes."""

import json

from paper_2410_22254_b200 import NodeSpec, TripleSpec, build_plan, emit_script, load_workload
from paper_2410_22254_b200.cli import run_cli


def test_plan_mode_artifacts_match_library(tmp_path):
    w = tmp_path / "jobs.jsonl"
    w.write_text("".join(json.dumps({"argv": ["python3", "-m", "paper_2410_22254_b200.job", "--model",
                                              "cnn", "--seed", str(i)]}) + "\n" for i in range(10)))
    code = run_cli(["--mode", "plan", "--triple", "1,8,1", "--tasks", str(w), "--gpus", "1", "--cores", "8",
                    "--outdir", str(tmp_path / "runs"), "--run-name", "p"])
    assert code == 0
    plan = build_plan(load_workload(w), TripleSpec(1, 8, 1), NodeSpec(cores=8, gpus=1, gpu_mem_mib=32768))
    assert (tmp_path / "runs/p/node_000.sh").read_text() == emit_script(plan, 0)
    summary = json.loads((tmp_path / "runs/p/plan_summary.json").read_text())
    assert summary["queue_lengths"] == [2, 2, 1, 1, 1, 1, 1, 1] and summary["gpu_slot_counts"] == {"0": 8}


def test_exec_subprocess_backend_and_exit_codes(tmp_path, capsys):
    w = tmp_path / "t.txt"
    w.write_text("echo a\nsh -c 'exit 3'\necho c\n")
    code = run_cli(["--mode", "exec", "--triple", "1,2,1", "--tasks", str(w), "--cores", "4",
                    "--outdir", str(tmp_path), "--run-name", "e"])
    assert code == 1
    rep = json.loads((tmp_path / "e/run_report.json").read_text())
    assert rep["failures"] == 1 and [r["exit_status"] for r in rep["results"]] == [0, 3, 0]


def test_config_errors_exit_2(tmp_path, capsys):
    assert run_cli(["--mode", "exec", "--num-tasks", "2", "--outdir", str(tmp_path)]) == 2
    assert "triple" in capsys.readouterr().err
    assert run_cli(["--mode", "sweep", "--triple", "1,1,1", "--num-tasks", "1"]) == 2
    assert run_cli(["--mode", "plan", "--triple", "1,4,4", "--num-tasks", "2", "--cores", "8",
                    "--strict", "--outdir", str(tmp_path)]) == 2
