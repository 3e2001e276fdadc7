"""Where the packed worker's start-up time goes (imports, context, pack, graph)."""
import sys, time
t0 = time.perf_counter()
sys.path.insert(0, ".")
import paper_2410_22254_b200  # noqa: F401
t1 = time.perf_counter()
from paper_2410_22254_b200 import runtime as rt
from paper_2410_22254_b200.scheduler import TlkBackend  # noqa: F401
t2 = time.perf_counter()
ctx = rt.Context(0)
t3 = time.perf_counter()
p = ctx.pack(rt.MODEL_CNN, 64, 8, 100, flags=rt.PACK_OWN_STREAM)
t4 = time.perf_counter()
for j in range(8):
    p.load(j, seed=j, steps=100)
ctx.sync()
t5 = time.perf_counter()
p.run(1)
ctx.sync()
t6 = time.perf_counter()
p.run(10)
ctx.sync()
t7 = time.perf_counter()
print(f"import pkg {t1-t0:.3f}  import runtime {t2-t1:.3f}  tlk_open {t3-t2:.3f}  pack_create {t4-t3:.3f}  "
      f"lane loads {t5-t4:.3f}  first step (graph capture) {t6-t5:.3f}  10 steps {t7-t6:.4f}")
