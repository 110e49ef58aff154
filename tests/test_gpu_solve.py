"""SURVEY 8(f) on the B200 against the reference itself (oracle/_ref): load
vectors, device-resident GMRES / CG (solver.hpp, same algorithm), potentials
and the point-charge / dipole errors against analytic fields.  North star:
solutions within 1e-8 relative, the same error against the analytic field."""
import numpy as np
import pytest

from oracle import pyref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")]

X0 = np.array([0.0, 0.1, 1.5])


def laplace_ps(p, x0=X0):
    return 1.0 / (4 * np.pi * np.linalg.norm(p - x0, axis=1))


def helmholtz_ps(p, k, x0=X0):
    r = np.linalg.norm(p - x0, axis=1)
    return np.exp(-1j * k * r) / (4 * np.pi * r)


def maxwell_dipole(x, y0, pol, k):  # operators.cpp:7-20
    d = x - y0
    r = np.linalg.norm(d, axis=1)[:, None]
    rhat = d / r
    g = np.exp(-1j * k * r) / (4 * np.pi * r)
    a = -1j * k - 1.0 / r
    gp = g * a
    gpp = g * (a * a + 1.0 / (r * r))
    rp = (rhat @ pol)[:, None]
    return k * k * g * pol + (gpp - gp / r) * rp * rhat + (gp / r) * pol


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_laplace_c1_pipeline(igb):
    """c1: point charge, CG and GMRES on the H2 operator, interior potential error"""
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 2, 1, 3)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    rd = pyref.Discretization("laplace", 2, 1, 3)
    rh = pyref.H2Matrix(rd, m=8)
    b = igb.compute_rhs(d, laplace_ps)
    rb = rd.rhs(0, X0)
    assert _rel(b, rb) < 1e-13
    grid = igb.make_sphere_grid(0.5, 10)  # tools/main.cpp:218-220 interior default
    exact = laplace_ps(grid)
    # Solution parity needs a tolerance that pins the discrete solution to 1e-8:
    # at the config's tol 1e-8 two valid runs whose matvecs differ only in
    # rounding (6e-16 here) stop a few iterations apart and differ by ~cond * tol
    # (measured: GMRES(200) 60 vs 61 its / 4.2e-7, CG 72 vs 75 / 5.6e-7).  At
    # tol 1e-10 GMRES gives 82 = 82 its / 2.0e-9; CG is rounding-sensitive (loss
    # of orthogonality) and is compared at 1e-12: 130 = 130 its / 4.7e-12.  At
    # tol 1e-8 the iteration counts (GMRES +-1, CG +-3) and the point-charge
    # error must agree.
    for method, tol in (("gmres", 1e-8), ("cg", 1e-8)):
        fn = igb.cg if method == "cg" else igb.gmres
        opts = igb.SolverOptions(tol=tol, max_iter=5000, restart=200)
        x, st = fn(h, b, opts)
        rx, rst = rh.solve(rb, method, tol=tol, max_iter=opts.max_iter, restart=opts.restart)
        assert st.converged and rst["converged"]
        assert abs(st.iterations - rst["iterations"]) <= (1 if method == "gmres" else 3)
        u, ru = igb.eval_potential(d, x, grid), rd.potential(rx, grid)
        err, rerr = np.abs(u - exact).max(), np.abs(ru - exact).max()
        assert abs(err - rerr) <= 1e-3 * rerr and err < 1e-5  # same point-charge error
    for method, opts, its in (("gmres", igb.SolverOptions(tol=1e-10, max_iter=5000, restart=200), 1),
                              ("cg", igb.SolverOptions(tol=1e-12, max_iter=5000), 3)):
        fn = igb.cg if method == "cg" else igb.gmres
        x, st = fn(h, b, opts)
        rx, rst = rh.solve(rb, method, tol=opts.tol, max_iter=opts.max_iter, restart=opts.restart)
        assert st.converged and rst["converged"]
        assert abs(st.iterations - rst["iterations"]) <= its
        assert _rel(x, rx) < 1e-8  # north star: GMRES/CG solution within 1e-8
        u = igb.eval_potential(d, x, grid)
        ru = rd.potential(rx, grid)
        assert _rel(u, ru) < 1e-10
        err, rerr = np.abs(u - exact).max(), np.abs(ru - exact).max()
        assert abs(err - rerr) <= 1e-3 * rerr  # same point-charge error
        assert err < 1e-5


def test_helmholtz_pipeline(igb):
    k = 3.0
    d = igb.Discretization(igb.make_sphere(), igb.Pde.helmholtz(k), 2, 1, 2)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    rd = pyref.Discretization("helmholtz", 2, 1, 2, kappa=k)
    rh = pyref.H2Matrix(rd, m=8)
    b = igb.compute_rhs(d, lambda p: helmholtz_ps(p, k))
    rb = rd.rhs(1, X0)
    assert _rel(b, rb) < 1e-13
    opts = igb.SolverOptions(tol=1e-10, max_iter=2000, restart=50)
    x, st = igb.gmres(h, b, opts)
    rx, rst = rh.solve(rb, "gmres", tol=opts.tol, max_iter=opts.max_iter, restart=opts.restart)
    assert st.converged and abs(st.iterations - rst["iterations"]) <= 1
    assert _rel(x, rx) < 1e-8
    grid = igb.make_sphere_grid(0.5, 6)
    assert _rel(igb.eval_potential(d, x, grid), rd.potential(rx, grid)) < 1e-10


def test_maxwell_dipole_and_plane_wave(igb):
    k = 2 * np.pi
    d = igb.Discretization(igb.make_sphere(), igb.Pde.maxwell(k), 2, 1, 2)
    h = igb.H2Matrix(d, igb.H2Options(m=6))
    rd = pyref.Discretization("maxwell", 2, 1, 2, kappa=k)
    rh = pyref.H2Matrix(rd, m=6)
    y0, pol = np.array([0.0, 0.0, 0.3]), np.array([1.0, 0.0, 0.0])
    b = igb.compute_rhs(d, lambda p: maxwell_dipole(p, y0, pol, k))
    assert _rel(b, rd.rhs(2, np.r_[y0, pol])) < 1e-13
    # c4 excitation: plane wave along z, polarisation x (E = -pol e^{-i k z})
    bw = igb.compute_rhs(d, lambda p: -pol[None, :] * np.exp(-1j * k * p[:, 2:3]))
    rbw = rd.rhs(3, [0, 0, 1, 1, 0, 0])
    assert _rel(bw, rbw) < 1e-13
    # the EFIE is ill-conditioned: at tol 1e-8 two valid GMRES(50) runs differ
    # by ~5e-8 (632 vs 636 its); at tol 1e-10, restart 200 (the CLI's) the
    # iterations match (143 = 143) and the solutions agree to ~5e-11
    opts = igb.SolverOptions(tol=1e-10, max_iter=3000, restart=200)
    x, st = igb.gmres(h, bw, opts)
    rx, rst = rh.solve(rbw, "gmres", tol=opts.tol, max_iter=opts.max_iter, restart=opts.restart)
    assert st.converged and abs(st.iterations - rst["iterations"]) <= 2
    assert _rel(x, rx) < 1e-8
    g = np.random.default_rng(20261019).standard_normal((100, 3))
    pts = 3.0 * g / np.linalg.norm(g, axis=1)[:, None]  # c4: 100 seeded points on radius 3
    e, re = igb.eval_maxwell_potential(d, x, pts), rd.potential(rx, pts)
    assert _rel(e, re) < 1e-10


def _gold(name):
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated (tools/make_golden.py solve)")
    z = np.load(p)
    return {k: z[k] for k in z.files}


def test_c2_cg_point_charge(igb):
    """c2 at full size (26,136 DOFs, m = 4): point-charge RHS, device CG against
    the reference's own CG (tests/golden/solve_c2_*.npz).  At tol 1e-12 the
    solutions agree to 1e-8 (north star); at the config's tol 1e-8 the iteration
    counts and the point-charge error on the interior grid agree."""
    g = _gold("solve_c2_laplace_P3_L6_m4.npz")
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
    h = igb.H2Matrix(d, igb.H2Options(m=4))
    b = igb.compute_rhs(d, laplace_ps)
    assert _rel(b, g["b"]) < 1e-13
    grid = g["grid"]
    exact = laplace_ps(grid)
    # CG is rounding-sensitive (loss of orthogonality over ~950 iterations):
    # measured 935 vs the reference's 959 at tol 1e-12, both converged
    x, st = igb.cg(h, b, igb.SolverOptions(tol=1e-12, max_iter=5000))
    assert st.converged and abs(st.iterations - int(g["its_t12"])) <= 0.05 * int(g["its_t12"])
    assert _rel(x, g["x_t12"]) < 1e-8
    u = igb.eval_potential(d, x, grid)
    assert _rel(u, g["u_t12"]) < 1e-10
    x8, st8 = igb.cg(h, b, igb.SolverOptions(tol=1e-8, max_iter=5000))
    assert st8.converged and abs(st8.iterations - int(g["its_t8"])) <= 0.05 * int(g["its_t8"])
    err, rerr = np.abs(igb.eval_potential(d, x8, grid) - exact).max(), np.abs(g["u_t8"] - exact).max()
    assert abs(err - rerr) <= 1e-2 * rerr
    print(f"c2 CG: {st8.iterations} its (reference {int(g['its_t8'])}), point-charge error {err:.4e} "
          f"(reference {rerr:.4e}); tol 1e-12: {st.iterations} its, |x - x_ref| / |x_ref| {_rel(x, g['x_t12']):.2e}")


def test_c4_gmres_scattered_field(igb):
    """c4 at full size (13,068 DOFs, Maxwell, m = 8): plane-wave excitation,
    device GMRES(200) at tol 1e-10 against the reference's (tests/golden/
    solve_c4_*.npz): solution within 1e-8 and the scattered field at the 100
    seeded radius-3 points within 1e-10."""
    g = _gold("solve_c4_maxwell_P2_L5_m8_k2pi.npz")
    k = 2 * np.pi
    d = igb.Discretization(igb.make_sphere(), igb.Pde.maxwell(k), 2, 1, 5)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    pol = np.array([1.0, 0.0, 0.0])
    b = igb.compute_rhs(d, lambda p: -pol[None, :] * np.exp(-1j * k * p[:, 2:3]))
    assert _rel(b, g["b"]) < 1e-13
    x, st = igb.gmres(h, b, igb.SolverOptions(tol=1e-10, max_iter=5000, restart=200))
    e = igb.eval_maxwell_potential(d, x, g["pts"])
    print(f"c4 GMRES(200): {st.iterations} its (reference {int(g['its'])}), |x - x_ref| / |x_ref| {_rel(x, g['x']):.2e}, "
          f"|E - E_ref| / |E_ref| {_rel(e, g['e']):.2e}")
    # ~3100 iterations over 16 restart cycles: the count moves by a few per cent with rounding
    assert st.converged and abs(st.iterations - int(g["its"])) <= 0.03 * int(g["its"])
    assert _rel(x, g["x"]) < 1e-8
    assert _rel(e, g["e"]) < 1e-10


def test_c3_gmres_report(igb):
    """c3 at full size (101,400 DOFs, Helmholtz kappa = 4 pi, m = 8): GMRES(50)
    at tol 1e-8 on the B200 operator.  kappa = 4 pi is an interior Dirichlet
    eigenvalue of the unit sphere (j_0(4 pi) = 0): the operator is singular, so
    this is a report (iterations, residual; capped at 400 iterations here),
    not a pass/fail solution check."""
    k = 4 * np.pi
    d = igb.Discretization(igb.make_sphere(), igb.Pde.helmholtz(k), 3, 1, 7)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    b = igb.compute_rhs(d, lambda p: helmholtz_ps(p, k))
    x, st = igb.gmres(h, b, igb.SolverOptions(tol=1e-8, max_iter=400, restart=50))
    r = np.linalg.norm(h @ x - b) / np.linalg.norm(b)
    assert np.isfinite(x).all() and r < 1.0
    print(f"c3 GMRES(50): {st.iterations} its, converged {st.converged}, relative residual {r:.3e}, "
          f"{st.seconds:.1f} s")
