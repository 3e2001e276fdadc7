"""The committed packed-runtime calibration feeds the reference simulator's
``table`` slowdown model (skipped without the reference)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
CAL = os.path.join(ROOT, "profiles", "r1h_sim_calibration_cnn.json")


def test_calibration_is_monotone_and_sublinear():
    cal = json.load(open(CAL))
    pts = {int(k): v for k, v in cal["slowdown_points"].items()}
    ks = sorted(pts)
    assert pts[1] == 1.0
    assert all(pts[a] <= pts[b] for a, b in zip(ks, ks[1:]))
    assert all(pts[k] < k for k in ks if k > 1)  # packing beats time slicing at every k


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_reference_sim_accepts_the_table(tmp_path):
    cal = json.load(open(CAL))
    table = cal["reference_cli"][cal["reference_cli"].index("--slowdown-table") + 1]
    code = ("import sys; from trilaunch.sim import make_slowdown;"
            "f = make_slowdown('table', table=dict(p.split(':') for p in sys.argv[1].split(',')));"
            "print(f(1), f(8), f(12))")
    out = subprocess.run([sys.executable, "-c", code, table], env=dict(os.environ, PYTHONPATH=REF),
                         capture_output=True, text=True, cwd=tmp_path)
    assert out.returncode == 0, out.stderr
    f1, f8, f12 = map(float, out.stdout.split())
    assert f1 == 1.0 and abs(f8 - cal["slowdown_points"]["8"]) < 1e-9 and f8 < f12
