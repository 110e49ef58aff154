"""the dense Galerkin matrix assembled on the B200
(assemble_dense / assemble_dense_complex, assembly.cpp:16-53) against the
reference itself (oracle/_ref) and the oracle restatement; the reference's own
dense pins (symmetry, kappa=0 Helmholtz == Laplace, H2 vs dense)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from oracle import pyref

pytestmark = pytest.mark.gpu

CASES = [("laplace", 0, 1, 1, 0.0), ("laplace", 2, 1, 2, 0.0), ("laplace", 3, 1, 2, 0.0), ("laplace", 1, 1, 3, 0.0),
         ("helmholtz", 2, 1, 2, 3.0), ("maxwell", 2, 1, 1, 3.0), ("maxwell", 1, 1, 2, 2 * np.pi)]


def _pde(igb, kind, k):
    if kind == "laplace":
        return igb.Pde.laplace()
    return igb.Pde.helmholtz(k) if kind == "helmholtz" else igb.Pde.maxwell(k)


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c[:4])))
def test_dense_matches_reference(igb, case):
    kind, P, rep, L, k = case
    d = igb.Discretization(igb.make_sphere(), _pde(igb, kind, k), P, rep, L)
    A = igb.assemble_dense(d)
    assert A.shape == (d.dof_count(),) * 2 and np.isfinite(A).all()
    ref = (pyref.Discretization(kind, P, rep, L, kappa=k) if pyref.available() else
           po.Discretization(kind, P, rep, L, kappa=k)).assemble_dense()
    assert _rel(A, ref) < 1e-12  # north star 1e-10
    # Galerkin symmetry (test_assembly.cpp:20-29): the bilinear forms are symmetric
    assert _rel(A, A.T) < 1e-13


def test_dense_orders_and_kappa0(igb):
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 1, 1, 1)
    A = igb.assemble_dense(d, igb.AssemblyOptions(far_order=7, sing_order=8))
    B = po.Discretization("laplace", 1, 1, 1).assemble_dense(far_order=7, sing_order=8)
    assert _rel(A, B) < 1e-12
    h = igb.assemble_dense(igb.Discretization(igb.make_sphere(), igb.Pde.helmholtz(0.0), 1, 1, 1))
    assert np.abs(h.imag).max() == 0 and _rel(h.real, igb.assemble_dense(d)) < 1e-13  # acceptance.cpp:216-229


def test_h2_against_device_dense(igb):
    # test_h2.cpp:94-106: H2 vs dense < 1e-6 at m = 8, now both on the device
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 2, 1, 3)
    A = igb.assemble_dense(d)
    h = igb.H2Matrix(d, igb.H2Options(m=8))
    x = np.random.default_rng(3).uniform(-1, 1, d.dof_count())
    assert np.linalg.norm(h @ x - A @ x) / np.linalg.norm(A @ x) < 1e-6


def test_dense_chunked_equals_whole(igb):
    # c4-sized rows force several chunks only at large N; check a mid-size case bitwise-deterministic
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 3)
    A, B = igb.assemble_dense(d), igb.assemble_dense(d)
    assert np.array_equal(A, B)
