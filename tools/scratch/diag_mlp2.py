import numpy as np, sys, torch
sys.path.insert(0, '.')
from oracle import models as om, rng
from oracle.bf16 import round_bf16
import oracle.models as M
from paper_2410_22254_b200 import runtime as rt
def rel(a, b): return float(np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30))
def bf(u16): return (u16.astype(np.uint32) << 16).view(np.float32)
for seed in (21, 1, 23):
  with rt.Context(0) as ctx:
    p = ctx.pack(1, 64, 1, 1); p.load(0, seed=seed, steps=1); p.run(1); ctx.sync()
    acts = p.tensor(rt.BUF_ACTS).cpu().numpy().astype(np.uint16)
    n = 64*512
    h1, h2, dz1, dz2 = [bf(acts[i*n:(i+1)*n]).reshape(64,512) for i in range(4)]
    g = p.tensor(rt.BUF_GRADS).cpu().numpy()
    prm = om.init_params(1, seed); px, y = rng.batch(seed, 0, 64)
    r = M._r; x = px.astype(np.float32)/256
    w1, w2 = r(prm["fc1.w"], True), r(prm["fc2.w"], True)
    z1 = x @ w1.T + prm["fc1.b"]; rh1 = r(np.maximum(z1, 0), True)
    z2 = rh1 @ w2.T + prm["fc2.b"]; rh2 = r(np.maximum(z2, 0), True)
    print(seed, 'h1 mismatch', (h1 != rh1).sum(), 'h2 mismatch', (h2 != rh2).sum())
    bad = np.argwhere(h1 != rh1)[:5]
    for b, o in bad: print('   h1', b, o, h1[b,o], rh1[b,o], z1[b,o])
    bad = np.argwhere(h2 != rh2)[:5]
    for b, o in bad: print('   h2', b, o, h2[b,o], rh2[b,o], z2[b,o])
    loss, g3w, g3b, dh2 = M.head(h2, prm["fc3.w"], prm["fc3.b"], y)  # teacher-forced on GPU h2
    rdz2 = r(dh2 * (h2 > 0), True)
    print('  dz2 mismatch (forced)', (dz2 != rdz2).sum(), 'max', np.abs(dz2-rdz2).max())
    rdz1 = r((dz2 @ w2) * (h1 > 0), True)
    print('  dz1 mismatch (forced)', (dz1 != rdz1).sum(), 'max', np.abs(dz1-rdz1).max(), np.abs(rdz1).max())
    off = 0
    print('  fc1.w forced rel', rel(g[:512*784], (dz1.T @ x).reshape(-1)))
