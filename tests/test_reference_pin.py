"""Pins the oracle restatement to the reference itself: oracle/_ref is the
igabem core compiled unmodified against our Eigen-subset shim.  Skipped when
oracle/_ref was not built (no /root/reference at build time)."""
import numpy as np
import pytest

from oracle import pyref

pytestmark = pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")

CASES = [("laplace", 0, 1, 2, 4), ("laplace", 1, 1, 2, 8), ("laplace", 2, 1, 2, 8), ("laplace", 3, 2, 2, 4),
         ("helmholtz", 1, 1, 2, 6), ("maxwell", 1, 1, 1, 6), ("maxwell", 2, 1, 1, 4)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_oracle_equals_reference(po, case):
    kind, P, rep, L, m = case
    kap = 3.0 if kind != "laplace" else 0.0
    od, rd = po.Discretization(kind, P, rep, L, kappa=kap), pyref.Discretization(kind, P, rep, L, kappa=kap)
    assert np.array_equal(od.elements()[1], rd.elements()[1])  # boxes bit-identical
    for a, b in zip(od.l2g(), rd.l2g()):
        assert np.array_equal(a, b)
    oh, rh = po.H2Matrix(od, m=m), pyref.H2Matrix(rd, m=m)
    assert np.array_equal(oh.nearfield_pairs(), rh.nearfield_pairs())
    assert np.array_equal(oh.farfield_pairs(), rh.farfield_pairs())
    assert (oh.nearfield_entries, oh.farfield_entries, oh.total_bytes) == (
        rh.nearfield_entries, rh.farfield_entries, rh.total_bytes)
    pairs = oh.nearfield_pairs()
    assert np.array_equal(od.pair_blocks(pairs), rd.pair_blocks(pairs))  # identical arithmetic
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, od.dof_count) + (1j * rng.uniform(-1, 1, od.dof_count) if od.is_complex else 0)
    assert np.linalg.norm(oh.apply(x) - rh.apply(x)) <= 1e-14 * np.linalg.norm(rh.apply(x))


def test_rules_and_classification_identical(po):
    for cls in (1, 2, 3):
        for n in (3, 6):
            assert np.array_equal(po.pair_rule(cls, n), pyref.pair_rule(cls, n))
    od, rd = po.Discretization("laplace", 1, 1, 1), pyref.Discretization("laplace", 1, 1, 1)
    for ea in range(od.element_count):
        for eb in range(od.element_count):
            c1, m1 = od.classify_pair(ea, eb)
            c2, m2 = rd.classify_pair(ea, eb)
            assert c1 == c2 and np.array_equal(m1, m2)
