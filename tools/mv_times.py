"""c2 matvec: graph time per apply and serialised phase times."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
h = igb.H2Matrix(d, igb.H2Options(m=4))
ms, n = h.bench_apply(200)
ms, n = h.bench_apply(200)
p = h.profile_apply(50)
print("graph ms/apply", round(ms / 200, 4), "launches", n, {k: round(v / 50, 4) for k, v in p.items()})
