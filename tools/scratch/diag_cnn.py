import numpy as np, sys
sys.path.insert(0, '.')
from paper_2410_22254_b200 import runtime as rt
from tests.test_gpu_pack import _bf
B, L = 64, 2
with rt.Context(0) as ctx:
    p = ctx.pack(rt.MODEL_CNN, B, L, 2)
    for l in range(L): p.load(l, seed=31 + l, steps=2)
    p.run(1); ctx.sync()
    npos = 32 + B * 784 + 64
    raw = p.tensor(rt.BUF_ACTS).cpu().numpy().view(np.uint8)
    sizes = [("h1", 4 * npos * 16), ("p2", B * 9216 * 2), ("idx", B * 9216), ("h3", B * 128 * 2),
             ("dz3", B * 128 * 2), ("dz2", 8 * npos * 16), ("dz1", 4 * npos * 16)]
    off = 0
    for name, per in sizes:
        blob = raw[off: off + per]
        if name in ("h1", "dz2", "dz1") and blob.size == per:
            C = per // (npos * 16)
            pl = blob.view(np.uint16).reshape(C, npos, 8)
            front = np.abs(_bf(pl[:, :32])).sum(); back = np.abs(_bf(pl[:, 32 + B * 784:])).sum()
            img = _bf(pl[:, 32:32 + B * 784]).reshape(C, B, 28, 28, 8)
            rows = [np.abs(img[:, :, r]).sum() for r in range(28)]
            cols = [np.abs(img[:, :, :, c]).sum() for c in range(28)]
            print(name, 'front', front, 'back', back, 'rows', np.nonzero(rows)[0], 'cols', np.nonzero(cols)[0])
        off += (L * per + 15) // 16 * 16
    print("acts bytes", raw.size, "computed", off)
