"""c1 solve parity vs the reference at two tolerances (GMRES restart 200, CG)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyref
X0 = np.array([0.0, 0.1, 1.5])
ps = lambda p: 1.0 / (4 * np.pi * np.linalg.norm(p - X0, axis=1))
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 2, 1, 3)
h = igb.H2Matrix(d, igb.H2Options(m=8))
rd = pyref.Discretization("laplace", 2, 1, 3)
rh = pyref.H2Matrix(rd, m=8)
b = igb.compute_rhs(d, ps)
rb = rd.rhs(0, X0)
xr = np.random.default_rng(1).uniform(-1, 1, d.dof_count())
print("matvec rel", np.linalg.norm(h @ xr - rh.apply(xr)) / np.linalg.norm(rh.apply(xr)))
for tol in (1e-8, 1e-10, 1e-12):
    for method in ("gmres", "cg"):
        opts = igb.SolverOptions(tol=tol, max_iter=5000, restart=200)
        x, st = (igb.gmres if method == "gmres" else igb.cg)(h, b, opts)
        rx, rst = rh.solve(rb, method, tol=tol, max_iter=5000, restart=200)
        print(method, tol, "its", st.iterations, rst["iterations"], "rel", np.linalg.norm(x - rx) / np.linalg.norm(rx))
