import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyref
from test_gpu_solve import _rel
k = 2 * np.pi
d = igb.Discretization(igb.make_sphere(), igb.Pde.maxwell(k), 2, 1, 2)
h = igb.H2Matrix(d, igb.H2Options(m=6))
rd = pyref.Discretization("maxwell", 2, 1, 2, kappa=k); rh = pyref.H2Matrix(rd, m=6)
pol = np.array([1.0, 0.0, 0.0])
bw = igb.compute_rhs(d, lambda p: -pol[None, :] * np.exp(-1j * k * p[:, 2:3]))
rbw = rd.rhs(3, [0, 0, 1, 1, 0, 0])
print('rhs', _rel(bw, rbw), 'dofs', d.dof_count())
x0 = np.random.default_rng(1).standard_normal(d.dof_count()) + 0j
print('matvec', _rel(h @ x0, rh.apply(x0)))
for tol, rs in ((1e-8, 50), (1e-8, 200), (1e-10, 200)):
    o = igb.SolverOptions(tol=tol, max_iter=3000, restart=rs)
    x, st = igb.gmres(h, bw, o); rx, rst = rh.solve(rbw, "gmres", tol=tol, max_iter=3000, restart=rs)
    print(tol, rs, st, rst, 'x rel %.3e' % _rel(x, rx))
