"""Host-buffer apply vs device graph time (c2)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
h = igb.H2Matrix(d, igb.H2Options(m=4))
x = np.random.default_rng(0).uniform(-1, 1, d.dof_count())
for _ in range(20): y = h @ x
t = time.perf_counter()
for _ in range(200): y = h @ x
th = (time.perf_counter() - t) / 200
ms, _ = h.bench_apply(200)
print(f"host apply {th * 1e3:.4f} ms, device graph {ms / 200:.4f} ms, overhead {th * 1e3 - ms / 200:.4f} ms")
