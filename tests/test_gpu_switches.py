"""Every performance switch of libtlk leaves the numbers alone.

Each run is a fresh process (the switches are read once per process):
programmatic dependent launch off, the serial CNN graph (no forked conv2 wgrad
branch), fc1 wgrad+Adam on the main stream / on the graph's side branch / before
the conv2 wgrad on an odd CTA count instead of deferred past the step graph
(the default) -> bit-identical loss curves; the ResNet conv variants (no halo
tiles, no three-tap wgrad, 128-wide N tiles) only reorder fp32 sums -> loss
curves within the oracle's own bf16 spread of the default."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2410_22254_b200 import runtime as rt
model, lanes, batch, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
opt = dict(optimizer=rt.OPT_SGD, lr=0.02, momentum=0.9) if model == "resnet18" else {}
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODELS[model], batch, lanes, steps)
    for j in range(lanes):
        p.load(j, seed=70 + j, steps=steps, **opt)
    p.run(steps)
    ctx.sync()
    print(json.dumps([p.losses(j, steps).tolist() for j in range(lanes)]))
""" % ROOT


def _curves(env, *args):
    out = subprocess.run([sys.executable, "-c", CODE, *map(str, args)], capture_output=True, text=True,
                         env=dict(os.environ, **env), timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return np.array(json.loads(out.stdout.strip().splitlines()[-1]), np.float32)


@pytest.mark.parametrize("env", [{"TLK_PDL": "0"}, {"TLK_CNN_NOFORK": "1"}, {"TLK_CNN_FWA_SIDE": "0"},
                                 {"TLK_CNN_FWA_SIDE": "1"}, {"TLK_CNN_FWA_SIDE": "2", "TLK_FWA_CTAS": "37"},
                                 {"TLK_FWA_CTAS": "23"}, {"TLK_CNN_SPLIT_OPT": "1"}, {"TLK_FWA_DEFER_AT": "0"}, {"TLK_FWA_DEFER_AT": "2", "TLK_FWA_CTAS": "120"},
                                 {"TLK_CNN_FWA_SIDE": "4"}, {"TLK_CNN_JOIN_EARLY": "1"}, {"TLK_CNN_FLAG_JOIN": "1"}, {"TLK_CNN_FORK_LATE": "1"}])
def test_launch_switches_are_bit_identical(env):
    base = _curves({}, "cnn", 3, 64, 6)
    assert np.array_equal(_curves(env, "cnn", 3, 64, 6), base)


def test_pdl_off_bit_identical_transformer():
    assert np.array_equal(_curves({"TLK_PDL": "0"}, "xformer", 2, 8, 3), _curves({}, "xformer", 2, 8, 3))


@pytest.mark.parametrize("env", [{"TLK_NO_HALO": "1"}, {"TLK_NO_TAPGROUP": "1"}, {"TLK_CONV_BN256": "0"}])
def test_resnet_conv_variants_agree(env):
    base = _curves({}, "resnet18", 2, 16, 3)
    other = _curves(env, "resnet18", 2, 16, 3)
    assert np.allclose(base[:, 0], other[:, 0], rtol=5e-3)  # step 1: forward rounding only
    assert np.allclose(base, other, atol=0.1)
