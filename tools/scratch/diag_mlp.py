import numpy as np, sys, torch
sys.path.insert(0, '.')
from oracle import job as ojob, models as om, optim as oo, rng
from paper_2410_22254_b200 import runtime as rt
M = om.MODEL_MLP
def rel(a, b): return float(np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30))
with rt.Context(0) as ctx:
    # first-step grads
    p = ctx.pack(M, 64, 1, 1); p.load(0, seed=1, steps=1); p.run(1); ctx.sync()
    g = p.tensor(rt.BUF_GRADS).cpu().numpy()
    params = om.init_params(M, 1); px, y = rng.batch(1, 0, 64)
    loss, gref = om.mlp_step(params, px, y, bf16=True)
    gflat = om.flatten_params(M, gref)
    for t, off in om.layout(M)[0]:
        print('grad', t.name, rel(g[off:off+t.count], gflat[off:off+t.count]))
    print('loss', p.losses(0,1), loss)
    for lr, b1, opt in [(1e-3,.9,1),(3e-3,.8,1),(3e-3,.9,3)]:
        steps=12
        q = ctx.pack(M, 64, 1, steps); q.load(0, seed=1, steps=steps, lr=lr, beta1=b1, optimizer=opt, momentum=0.9 if opt==3 else 0); q.run(steps); ctx.sync()
        init = om.flatten_params(M, om.init_params(M, 1))
        st = oo.OptState(kind=opt, lr=lr, beta1=b1, momentum=0.9 if opt==3 else 0)
        l, f, _ = ojob.train(M, 1, steps, 64, st, bf16=True)
        gp = q.params(0)
        print('lr', lr, b1, opt, 'loss maxdiff', np.abs(q.losses(0,steps)-l).max())
        for t, off in om.layout(M)[0]:
            s = slice(off, off+t.count)
            print('  ', t.name, 'w', rel(gp[s], f[s]), 'delta', rel(gp[s]-init[s], f[s]-init[s]))
