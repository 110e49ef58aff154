"""A/B probe: far-field phase time at c2 and matvec parity vs the oracle (L=3)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyoracle as po
name = sys.argv[1] if len(sys.argv) > 1 else "?"
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
h = igb.H2Matrix(d, igb.H2Options(m=4))
h.profile_apply(20)
p = h.profile_apply(50)
ms, _ = h.bench_apply(200); ms, _ = h.bench_apply(200)
res = {"far_ms": round(p["far"] / 50, 4), "apply_ms": round(ms / 200, 4)}
for (P, L, m) in ((3, 3, 4), (2, 4, 8), (4, 3, 5)):
    dd = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), P, 1, L); hh = igb.H2Matrix(dd, igb.H2Options(m=m))
    x = np.random.default_rng(0).uniform(-1, 1, dd.dof_count())
    cache = f"/tmp/ab_oracle_{P}_{L}_{m}.npy"
    try:
        y = np.load(cache)
    except OSError:
        y = po.H2Matrix(po.Discretization("laplace", P, 1, L), m=m).apply(x)
        np.save(cache, y)
    res[f"rel_P{P}L{L}m{m}"] = float(np.linalg.norm(hh @ x - y) / np.linalg.norm(y))
print(name, res)
