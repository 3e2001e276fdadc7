"""Hash of a CNN pack's losses and parameters after N steps (bit-exactness across libtlk builds):
    TLK_LIB=... python tools/scratch/state_hash.py [model] [lanes] [steps]"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_22254_b200 import runtime as rt
model = sys.argv[1] if len(sys.argv) > 1 else "cnn"
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODELS[model], 64, lanes, steps)
    for j in range(lanes):
        p.load(j, seed=100 + j, steps=steps)
    p.run(steps)
    ctx.sync()
    h = hashlib.sha256()
    for j in range(lanes):
        h.update(p.losses(j, steps).tobytes())
        h.update(p.params(j).tobytes())
    print(model, lanes, steps, h.hexdigest()[:16], p.losses(0, steps)[-1])
