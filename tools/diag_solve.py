import sys; sys.path.insert(0, '.')
import numpy as np
import paper_1906_00785_b200 as igb
from oracle import pyref
sys.path.insert(0, 'tests')
from test_gpu_solve import laplace_ps, X0, _rel
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 2, 1, 3)
h = igb.H2Matrix(d, igb.H2Options(m=8))
rd = pyref.Discretization("laplace", 2, 1, 3); rh = pyref.H2Matrix(rd, m=8)
b = igb.compute_rhs(d, laplace_ps); rb = rd.rhs(0, X0)
print('rhs rel', _rel(b, rb))
grid = igb.make_sphere_grid(0.5, 10); exact = laplace_ps(grid)
for tol in (1e-8, 1e-10, 1e-12):
  for method, fn in (("cg", igb.cg), ("gmres", igb.gmres)):
    o = igb.SolverOptions(tol=tol, max_iter=5000, restart=200)
    x, st = fn(h, b, o); rx, rst = rh.solve(rb, method, tol=tol, max_iter=5000, restart=200)
    u = igb.eval_potential(d, x, grid); ru = rd.potential(rx, grid)
    print(method, tol, st.iterations, rst['iterations'], 'x rel %.3e' % _rel(x, rx), 'err %.6e %.6e' % (np.abs(u-exact).max(), np.abs(ru-exact).max()), 't %.3f %.3f' % (st.seconds, rst['seconds']))
