"""In-graph kernel timeline of the CNN step (needs libtlk built with -DTLK_KTRACE).

    TLK_NVCC_FLAGS=-DTLK_KTRACE python -m paper_2410_22254_b200.build --force
    python tools/cnn_timeline.py [LANES] [STEPS]
Runs STEPS steps of an 8-lane (default) CNN pack after a warm-up and prints,
for the last few steps, every kernel's first CTA entry, end of its PDL wait
and last warp exit relative to the step's first kernel entry (µs)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_22254_b200 import runtime as rt  # noqa: E402

NAMES = ["conv1_fwd", "conv2_fwd", "fc1_fwd", "head", "fc1_dgrad", "conv2_wgrad", "conv2_dgrad",
         "conv1_wgrad", "fc1_wgrad_adam", "opt", "conv1_opt", "-"]
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
lib = rt.lib()
buf = (ctypes.c_uint64 * 288)()
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_CNN, 64, lanes, 40 + steps)
    for j in range(lanes):
        p.load(j, seed=j, steps=40 + steps)
    p.run(20)
    ctx.sync()
    assert lib.tlk_cnn_ktrace(1, None, 0) == 0, lib.tlk_last_error()
    p.run(steps)
    ctx.sync()
    assert lib.tlk_cnn_ktrace(0, buf, 288) == 0
t = np.frombuffer(buf, np.uint64).reshape(8, 12, 3).astype(np.float64)
rows = []
for k in range(20 + 1, 20 + steps):  # skip the first timed step (no overlap from before)
    s = t[k % 8]
    valid = s[:, 2] > 0
    t0 = s[valid, 0].min()
    nxt = t[(k + 1) % 8]
    print(f"step {k}: next step's conv1_fwd entry at {(nxt[0, 0] - t0) / 1e3:7.1f} us")
    for i in np.argsort(np.where(valid, s[:, 0], np.inf)):
        if not valid[i]:
            continue
        e, w, x = (s[i] - t0) / 1e3
        print(f"  {NAMES[i]:16s} entry {e:7.1f}  waited {w:7.1f}  exit {x:7.1f}  run {x - w:6.1f}")
