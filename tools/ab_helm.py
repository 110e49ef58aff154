"""A/B probe: complex-kind far-field phase times (Helmholtz c3 space at L=6, Maxwell c4) and
matvec parity vs the oracle at small L."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyoracle as po
name = sys.argv[1] if len(sys.argv) > 1 else "?"
out = {}
for tag, pde, P, L, m in (("helm", igb.Pde.helmholtz(4 * np.pi), 3, 6, 8), ("maxw", igb.Pde.maxwell(2 * np.pi), 2, 5, 8)):
    d = igb.Discretization(igb.make_sphere(), pde, P, 1, L)
    h = igb.H2Matrix(d, igb.H2Options(m=m))
    h.profile_apply(3)
    p = h.profile_apply(10)
    out[tag + "_far_ms"] = round(p["far"] / 10, 3)
for tag, kind, k, P, L in (("helm", "helmholtz", 4 * np.pi, 3, 3), ("maxw", "maxwell", 2 * np.pi, 2, 2)):
    pde = igb.Pde.helmholtz(k) if kind == "helmholtz" else igb.Pde.maxwell(k)
    d = igb.Discretization(igb.make_sphere(), pde, P, 1, L)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, d.dof_count()) + 1j * rng.uniform(-1, 1, d.dof_count())
    cache = f"/tmp/ab_oracle_{kind}_{P}_{L}.npy"
    try:
        y = np.load(cache)
    except OSError:
        y = po.H2Matrix(po.Discretization(kind, P, 1, L, kappa=k), m=8).apply(x)
        np.save(cache, y)
    out["rel_" + tag] = float(np.linalg.norm(h @ x - y) / np.linalg.norm(y))
print(name, out)
