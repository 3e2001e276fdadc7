"""Generate tests/golden/mapping.json from the REFERENCE trilaunch (read-only import).

Pins the drop-in surface bit-exactly: for every BASELINE config triple plus
the paper's Table I and the edge cases SURVEY.md Appendix A
lists, record what the reference's own code produces -- validation verdicts,
slot bindings + env lists, queues (task ids per slot), plan_summary JSON text,
emit_script text sha256 + length, and _max_overlap / classify_failure
answers.  tests/test_mapping_golden.py replays the same inputs through
paper_2410_22254_b200 and requires identical outputs.

Run (needs /root/reference):  python tests/golden/gen_mapping_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def cases():
    """(name, triple, node kwargs, tasks spec) -- shared with the replay test."""
    out = []
    # BASELINE.json configs (tasks = parametric job argv), cores=8 like the survey
    out.append(("c1_mlp_1_4_1", (1, 4, 1), dict(cores=8, gpus=1, gpu_mem_mib=183359), ("job", 4, "mlp")))
    out.append(("c1_cpu_1_4_1", (1, 4, 1), dict(cores=8), ("job", 4, "mlp")))
    out.append(("c2_cnn_1_8_1", (1, 8, 1), dict(cores=8, gpus=1, gpu_mem_mib=183359), ("job", 8, "cnn")))
    out.append(("c3_resnet_1_64_2", (1, 64, 2), dict(cores=8, gpus=8, gpu_mem_mib=183359), ("job", 64, "resnet18")))
    out.append(("c5_gpt_1_128_1", (1, 128, 1), dict(cores=8, gpus=8, gpu_mem_mib=183359), ("job", 128, "gpt")))
    for nppn in (1, 2, 4, 8, 16, 32):
        out.append((f"c4_mix_1_{nppn}_1", (1, nppn, 1), dict(cores=64, gpus=1, gpu_mem_mib=183359), ("mix", 40, None)))
    # Table I (2x V100, 40 cores) with the paper's 24 jobs
    for t in [(1, 1, 40), (1, 2, 20), (1, 4, 10), (1, 6, 6), (1, 8, 5), (1, 12, 3), (1, 24, 1)]:
        out.append((f"table1_{t[0]}_{t[1]}_{t[2]}", t, dict(cores=40, gpus=2, gpu_mem_mib=32768), ("job", 24, "cnn")))
    # edge cases: multi-node slot count, ragged queues, oversubscription, custom ids
    out.append(("multinode_2_3_1", (2, 3, 1), dict(cores=8, gpus=2, gpu_mem_mib=1024), ("job", 7, "mlp")))
    out.append(("ragged_1_24_1", (1, 24, 1), dict(cores=40, gpus=2, gpu_mem_mib=32768), ("job", 48, "mlp")))
    out.append(("oversub_1_16_4", (1, 16, 4), dict(cores=8, gpus=4, gpu_mem_mib=1024), ("job", 37, "cnn")))
    out.append(("idle_slots_1_5_1", (1, 5, 1), dict(cores=8, gpus=3, gpu_mem_mib=1024), ("job", 2, "mlp")))
    out.append(("jsonl_ids_1_2_1", (1, 2, 1), dict(cores=8, gpus=2, gpu_mem_mib=1), ("jsonl", 0, None)))
    rnd = random.Random(20251017)
    for i in range(12):
        nn, np_, nt = rnd.randint(1, 3), rnd.randint(1, 20), rnd.randint(1, 4)
        g = rnd.choice([0, 1, 2, 3, 8])
        node = dict(cores=rnd.choice([4, 16, 64]), gpus=g, gpu_mem_mib=1024 if g else 0)
        out.append((f"random_{i}", (nn, np_, nt), node, ("job", rnd.randint(1, 90), rnd.choice(["mlp", "cnn"]))))
    return out


JSONL_TEXT = (
    '{"task_id": 7, "argv": ["python3", "-m", "paper_2410_22254_b200.job", "--model", "mlp", "--seed", "7"]}\n'
    '\n'
    '{"task_id": 3, "argv": ["a b", "c\'d"], "env": {"CUDA_VISIBLE_DEVICES": "5", "LR": "0.1"}}\n'
    '{"task_id": 5, "argv": ["echo", "$HOME"], "env": [["SEED", 42]]}\n'
)

MIX_MODELS = ("mlp", "cnn", "xformer")


def make_tasks(TaskDef, spec):
    kind, n, model = spec
    if kind == "job":
        return [TaskDef(i, ("python3", "-m", "paper_2410_22254_b200.job", "--model", model,
                            "--seed", str(i), "--lr", f"{1e-3 * (1 + i % 4):g}", "--steps", "200"))
                for i in range(n)]
    if kind == "mix":
        return [TaskDef(i, ("python3", "-m", "paper_2410_22254_b200.job", "--model",
                            MIX_MODELS[i % 3], "--seed", str(i)))
                for i in range(n)]
    raise ValueError(kind)


def describe(mod, name, triple, node_kw, spec):
    """Everything observable about planning this case, as JSON-able data."""
    core, plan_m, ex = mod
    T = core.TripleSpec(*triple)
    node = core.NodeSpec(**node_kw)
    if spec[0] == "jsonl":
        tasks = plan_m.parse_workload_jsonl(JSONL_TEXT)
    else:
        tasks = make_tasks(plan_m.TaskDef, spec)
    v = core.validate_triple(T, node)
    vs = core.validate_triple(T, node, strict=True)
    rec = {
        "verdict": [v.status, list(v.warnings), type(v.error).__name__ if v.error else None],
        "verdict_strict": [vs.status, list(vs.warnings), type(vs.error).__name__ if vs.error else None],
        "str": str(T), "total_processes": T.total_processes,
    }
    if not v.passed:
        return rec
    plan = plan_m.build_plan(tasks, T, node)
    rec["bindings"] = [[b.node_index, b.slot_index, b.gpu_index, b.thread_count,
                        [list(p) for p in core.render_env(b)]] for b in plan.bindings]
    rec["queues"] = [[b.node_index, b.slot_index, [t.task_id for t in plan.queue_for(b.node_index, b.slot_index)]]
                     for b in plan.bindings]
    rec["summary_json"] = json.dumps(plan_m.plan_summary(plan).to_json_dict(), sort_keys=False)
    scripts = []
    for i in range(T.nnode):
        s = plan_m.emit_script(plan, i)
        scripts.append([hashlib.sha256(s.encode()).hexdigest(), len(s)])
    rec["scripts"] = scripts
    return rec


def executor_facts(ex):
    rnd = random.Random(1420)
    overlaps = []
    for _ in range(40):
        iv = []
        for _ in range(rnd.randint(0, 12)):
            s = rnd.randint(0, 50)
            iv.append([s, s + rnd.randint(0, 20)])
        overlaps.append([iv, ex._max_overlap([tuple(x) for x in iv])])
    tails = ["", "CUDA out of memory", "Cannot Allocate Memory", "killed: OOM", "segfault",
             "zoom in", "tlk: out of memory allocating 3 GiB", "boomerang", "oom"]
    classify = [[st, t, ex.classify_failure(st, t)] for st in (1, 124, 137) for t in tails]
    return {"overlaps": overlaps, "classify": classify,
            "consts": [ex.TIMEOUT_EXIT_STATUS, ex.SPAWN_FAILURE_EXIT_STATUS, ex.MAX_FAILURE_EXIT,
                       ex.STDERR_TAIL_BYTES, list(ex.DEFAULT_OOM_PATTERNS)]}


def main():
    sys.path.insert(0, REF_SRC)
    from trilaunch import core, executor, plan  # the reference, read-only

    mod = (core, plan, executor)
    out = {"cases": {name: describe(mod, name, t, n, s) for name, t, n, s in cases()},
           "executor": executor_facts(executor)}
    path = os.path.join(HERE, "mapping.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", path, len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
