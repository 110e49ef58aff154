"""One step (device assembly + a few matvecs) of c1 / c2 / c5 after the first
assembly, for ncu launch lists / captures.  Not a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_00785_b200 as igb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
P, L, m = {"c1": (2, 3, 8), "c2": (3, 6, 4), "c5": (4, 8, 5)}[cfg]
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), P, 1, L)
h = igb.H2Matrix(d, igb.H2Options(m=m, eta=1.6))
h.bench_steps(1, 100 if cfg != "c5" else 20)
print("ok", h.assembly_times())
