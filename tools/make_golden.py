"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
igabem core compiled against the Eigen-subset shim).  Run in this container
(needs /root/reference at build time only):

    python tools/make_golden.py            # small cases
    python tools/make_golden.py c2         # full-size c2 matvec (minutes)
    python tools/make_golden.py c4         # full-size c4 (Maxwell, 34 GB of couplings in host RAM)
    python tools/make_golden.py solve c2   # config-level solve fixtures (c2 CG, c4 GMRES)

Each fixture stores the configuration, the seeded input x
(uniform[-1,1], numpy default_rng(20261019)), y = H x, partition counts,
storage report, and near-field blocks of a deterministic sample of pairs."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SMALL = {
    # name: kind, P, rep, L, m, kappa
    "c1_laplace_P2_L3_m8": ("laplace", 2, 1, 3, 8, 0.0),
    "laplace_P3_L3_m4": ("laplace", 3, 1, 3, 4, 0.0),
    "laplace_P4_L2_m5": ("laplace", 4, 1, 2, 5, 0.0),
    "laplace_P0_L3_m4": ("laplace", 0, 1, 3, 4, 0.0),
    "helmholtz_P3_L2_m8_k4pi": ("helmholtz", 3, 1, 2, 8, 4 * np.pi),
    "maxwell_P2_L2_m8_k2pi": ("maxwell", 2, 1, 2, 8, 2 * np.pi),
}
BIG = {"c2_laplace_P3_L6_m4": ("laplace", 3, 1, 6, 4, 0.0)}
BIG_C4 = {"c4_maxwell_P2_L5_m8_k2pi": ("maxwell", 2, 1, 5, 8, 2 * np.pi)}


def make(name, cfg, nblocks=400):
    kind, P, rep, L, m, kappa = cfg
    t0 = time.time()
    d = pyref.Discretization(kind, P, rep, L, kappa=kappa)
    h = pyref.H2Matrix(d, m=m, eta=1.6)
    rng = np.random.default_rng(20261019)
    x = rng.uniform(-1, 1, d.dof_count)
    if d.is_complex:
        x = x + 1j * rng.uniform(-1, 1, d.dof_count)
    y = h.apply(x)
    near = h.nearfield_pairs()
    idx = np.linspace(0, len(near) - 1, min(nblocks, len(near))).astype(np.int64)
    blocks = d.pair_blocks(near[idx])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), kind=kind, P=P, rep=rep, L=L, m=m, eta=1.6,
                        kappa=kappa, x=x, y=y, near_count=h.near_count, far_count=h.far_count,
                        nearfield_entries=h.nearfield_entries, farfield_entries=h.farfield_entries,
                        total_bytes=h.total_bytes, block_pairs=near[idx], blocks=blocks,
                        generator="oracle/_ref (reference igabem core + Eigen-subset shim)")
    print(f"{name}: dofs={d.dof_count} near={h.near_count} far={h.far_count} {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "solve"):
    os.makedirs(OUT, exist_ok=True)
    arg = sys.argv[1] if len(sys.argv) > 1 else ""
    which = {"c2": BIG, "c4": BIG_C4}.get(arg, SMALL)
    for name, cfg in which.items():
        make(name, cfg)


def make_solve(which):
    """Config-level solve fixtures from the reference (tests/test_gpu_solve.py):
    c2: point-charge RHS, CG at tol 1e-8 and 1e-12, interior potential;
    c4: plane-wave RHS, GMRES(200) at tol 1e-10, E at 100 seeded radius-3 points."""
    x0 = [0.0, 0.1, 1.5]
    t0 = time.time()
    if which == "c2":
        d = pyref.Discretization("laplace", 3, 1, 6)
        h = pyref.H2Matrix(d, m=4, eta=1.6)
        b = d.rhs(0, x0)
        out = dict(b=b)
        k = np.arange(10)
        grid = make_grid(0.5, 10)
        for tag, tol in (("t8", 1e-8), ("t12", 1e-12)):
            x, st = h.solve(b, "cg", tol=tol, max_iter=5000, restart=30)
            out[f"x_{tag}"] = x
            out[f"its_{tag}"] = st["iterations"]
            out[f"u_{tag}"] = d.potential(x, grid)
            print(which, tag, st, flush=True)
        np.savez_compressed(os.path.join(OUT, "solve_c2_laplace_P3_L6_m4.npz"), grid=grid, **out,
                            generator="oracle/_ref (reference igabem core + Eigen-subset shim)")
    else:
        k = 2 * np.pi
        d = pyref.Discretization("maxwell", 2, 1, 5, kappa=k)
        h = pyref.H2Matrix(d, m=8, eta=1.6)
        b = d.rhs(3, [0, 0, 1, 1, 0, 0])
        x, st = h.solve(b, "gmres", tol=1e-10, max_iter=5000, restart=200)
        print(which, st, flush=True)
        g = np.random.default_rng(20261019).standard_normal((100, 3))
        pts = 3.0 * g / np.linalg.norm(g, axis=1)[:, None]
        e = d.potential(x, pts)
        np.savez_compressed(os.path.join(OUT, "solve_c4_maxwell_P2_L5_m8_k2pi.npz"), b=b, x=x,
                            its=st["iterations"], pts=pts, e=e,
                            generator="oracle/_ref (reference igabem core + Eigen-subset shim)")
    print(which, f"{time.time() - t0:.0f}s", flush=True)


def make_grid(radius, n):  # util.cpp:9-24 (theta-major), as igabem.make_sphere_grid
    k = np.arange(n)
    theta = np.pi * (k + 0.5) / n
    phi = 2.0 * np.pi * k / n
    th, ph = np.meshgrid(theta, phi, indexing="ij")
    return radius * np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], axis=-1).reshape(-1, 3)


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[1] == "solve":
    make_solve(sys.argv[2])
