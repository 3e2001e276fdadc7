"""Bit-exact mapping parity: our drop-in surface vs outputs of the reference.

tests/golden/mapping.json was produced by the reference trilaunch itself
(tests/golden/gen_mapping_golden.py).  The same inputs replayed through
paper_2410_22254_b200 must give identical verdicts, slot bindings, env lists,
queues, plan_summary JSON and emit_script bytes (sha256), plus identical
_max_overlap / classify_failure answers.  No /root/reference needed.
"""

import json
import os

import pytest

from paper_2410_22254_b200 import core, executor, plan
from tests.golden import gen_mapping_golden as gen

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mapping.json")))
CASES = {name: (t, n, s) for name, t, n, s in gen.cases()}


@pytest.mark.parametrize("name", sorted(CASES))
def test_case_matches_reference(name):
    t, n, s = CASES[name]
    ours = json.loads(json.dumps(gen.describe((core, plan, executor), name, t, n, s)))
    assert ours == GOLDEN["cases"][name]


def test_golden_covers_baseline_configs():
    for name in ("c1_mlp_1_4_1", "c2_cnn_1_8_1", "c3_resnet_1_64_2", "c5_gpt_1_128_1"):
        assert "bindings" in GOLDEN["cases"][name]


def test_executor_facts_match_reference():
    ours = json.loads(json.dumps(gen.executor_facts(executor)))
    assert ours == GOLDEN["executor"]
