"""Timeline of the fused attention kernels (CTA 0, first 64 tiles): python tools/attn_trace.py [lanes batch]

Runs one tiny-GPT step with TLK_ATTN_TRACE=1 and prints, per tile, the clock64
offsets (cycles, relative to the first event of the launch) of each role's events."""
import os
import sys

os.environ["TLK_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2410_22254_b200 import runtime as rt  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 16
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_GPT, batch, lanes, 3)
    for j in range(lanes):
        p.load(j, seed=j, steps=3)
    p.run(2)
    ctx.sync()
    tr = p.named("attn.trace", "f4").cpu().numpy().view(np.uint64).astype(np.int64).reshape(2, 64, 32)
NAMES = {
    "fwd": {0: "sfull", 1: "Sld", 2: "max", 4: "pfull", 5: "drain", 8: "M:sfree", 10: "M:Scom", 11: "M:Owait",
            12: "M:Ocom", 16: "P:Q", 17: "P:K", 18: "P:V"},
    "bwd": {0: "sdpfull", 2: "math", 3: "mmadone", 4: "pds", 5: "drains", 8: "M:sdpfree", 9: "M:loads",
            10: "M:SdPcom", 11: "M:pds", 12: "M:empt", 13: "M:VKQcom", 16: "P:Q0", 17: "P:dY0", 18: "P:K0",
            19: "P:V0", 20: "P:Q1", 21: "P:dY1", 22: "P:K1", 23: "P:V1"},
}
for k, name in enumerate(("fwd", "bwd")):
    t = tr[k]
    nz = t[t > 0]
    if nz.size == 0:
        print(name, "no trace")
        continue
    t0 = nz.min()
    cols = sorted(NAMES[name])
    print(f"== {name} (cycles from launch start)")
    print("tile " + " ".join(f"{NAMES[name][c]:>9s}" for c in cols))
    for i in range(40):
        row = t[i]
        if not row.any():
            continue
        print(f"{i:4d} " + " ".join(f"{(row[c] - t0) if row[c] else -1:9d}" for c in cols))
