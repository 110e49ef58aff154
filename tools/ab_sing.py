"""A/B probe: singular-class assembly times (c2, c5-space at L=6, Helmholtz c3-space at L=5) and near-block parity."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyoracle as po
name = sys.argv[1] if len(sys.argv) > 1 else "?"
out = {}
for tag, pde, P, L, m in (("c2", igb.Pde.laplace(), 3, 6, 4), ("p4", igb.Pde.laplace(), 4, 6, 5),
                          ("helm", igb.Pde.helmholtz(4 * np.pi), 3, 5, 4)):
    d = igb.Discretization(igb.make_sphere(), pde, P, 1, L)
    h = igb.H2Matrix(d, igb.H2Options(m=m))
    for _ in range(3):
        h.reassemble()
    t = h.assembly_times()
    out[tag] = {k[:-3]: round(t[k], 3) for k in ("coincident_ms", "edge_ms", "vertex_ms")}
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 3)
h = igb.H2Matrix(d, igb.H2Options(m=4))
x = np.random.default_rng(0).uniform(-1, 1, d.dof_count())
try:
    y = np.load("/tmp/ab_oracle_3_3_4.npy")
except OSError:
    y = po.H2Matrix(po.Discretization("laplace", 3, 1, 3), m=4).apply(x)
    np.save("/tmp/ab_oracle_3_3_4.npy", y)
out["rel"] = float(np.linalg.norm(h @ x - y) / np.linalg.norm(y))
print(name, out)
