"""e2e breakdown of the c2 public-API step (ctor + 100 host applies)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
o = igb.H2Options(m=4)
x = np.random.default_rng(0).uniform(-1, 1, d.dof_count())
h = igb.H2Matrix(d, o); h @ x; del h
for it in range(3):
    t0 = time.perf_counter(); h = igb.H2Matrix(d, o); t1 = time.perf_counter()
    print(f"[py] ctor returned {1e3*(t1-t0):.1f} ms", file=sys.stderr, flush=True)
    y = h @ x; t2 = time.perf_counter()
    for _ in range(99): y = h @ x
    t3 = time.perf_counter(); del h; t4 = time.perf_counter()
    print(f"ctor {1e3*(t1-t0):.1f} ms  first apply {1e3*(t2-t1):.2f} ms  99 applies {1e3*(t3-t2):.1f} ms  dtor {1e3*(t4-t3):.1f} ms",
          file=sys.stderr, flush=True)
h = igb.H2Matrix(d, o)
print({k: round(v, 2) for k, v in h.assembly_times().items()})
