"""CPU tests of the oracle (oracle/igb_oracle.cpp) against the reference's own
pins: frozen constants and identities from /root/reference/proj/tests
(restated; the reference is not read at run time)."""
import numpy as np
import pytest

# test_quadrature.cpp:16-18 / test_assembly.cpp:53-55 (frozen adaptive-oracle values)
K_COINCIDENT = 2.366005020877e-01
K_EDGE = 8.850038917189e-02
K_VERTEX = 5.959972386089e-02


def quad_flat(po, cls, n):
    """flat canonical configurations (test_quadrature.cpp:24-47)"""
    r = po.pair_rule(cls, n)
    ub, vb = r[:, 2], r[:, 3]
    if cls == po.EDGE:
        vb = -vb
    if cls == po.VERTEX:
        ub, vb = -ub, -vb
    return float(np.sum(r[:, 4] / (4 * np.pi * np.hypot(r[:, 0] - ub, r[:, 1] - vb))))


def test_gauss_exactness(po):  # test_quadrature.cpp:49-66
    for n in (1, 2, 5, 12, 30, 64):
        x, w = po.gauss(n)
        assert abs(w.sum() - 1) < 1e-14
        assert x.min() > 0 and x.max() < 1
        for k in range(2 * n):
            assert abs(np.sum(w * x ** k) - 1 / (k + 1)) <= 1e-13 * (1 / (k + 1)) + 1e-15
    for bad in (0, 65):
        with pytest.raises(ValueError):
            po.gauss(bad)


def test_pair_rules_volume(po):  # test_quadrature.cpp:68-82
    for cls in (po.COINCIDENT, po.EDGE, po.VERTEX):
        for n in (2, 4, 8):
            r = po.pair_rule(cls, n)
            assert len(r) == {po.COINCIDENT: 8, po.EDGE: 6, po.VERTEX: 4}[cls] * n ** 4
            assert abs(r[:, 4].sum() - 1) < 1e-13
            assert (r[:, 0] >= 0).all() and (r[:, 0] <= 1).all()
            assert (r[:, 3] >= 0).all() and (r[:, 3] <= 1).all()


def test_frozen_singular_constants(po):  # test_quadrature.cpp:84-96
    assert abs(quad_flat(po, po.COINCIDENT, 8) - K_COINCIDENT) < 1e-8
    assert abs(quad_flat(po, po.EDGE, 8) - K_EDGE) < 1e-8
    assert abs(quad_flat(po, po.VERTEX, 8) - K_VERTEX) < 1e-8


def test_rules_converge(po):  # test_quadrature.cpp:98-109
    for cls, ref in ((po.COINCIDENT, K_COINCIDENT), (po.EDGE, K_EDGE), (po.VERTEX, K_VERTEX)):
        e3, e6, e10 = (abs(quad_flat(po, cls, n) - ref) for n in (3, 6, 10))
        assert e6 < e3 and e10 < e6 and e10 < 1e-9


def test_naive_gauss_canary(po):  # test_quadrature.cpp:111-125
    x, w = po.gauss(16)
    X = np.meshgrid(x, x, x, x, indexing="ij")
    W = np.einsum("i,j,k,l->ijkl", w, w, w, w)
    r = np.maximum(np.hypot(X[0] - X[2], X[1] - X[3]), 1e-300)
    assert abs(np.sum(W / (4 * np.pi * r)) - K_COINCIDENT) > 1e-3


@pytest.mark.parametrize("P,L", [(p, l) for p in (0, 1, 2, 3) for l in (0, 1, 2)])
def test_scalar_dof_counts(po, P, L):  # test_spaces.cpp:20-37
    d = po.Discretization("laplace", P, 1, L)
    r = min(1, P)
    k = (1 << L) if P == 0 else ((1 << L) * r + P - r)
    assert d.dof_count == 6 * k * k
    assert d.element_count == 6 << (2 * L)
    q = max(P - 1, 0)
    assert d.local_count == (q + 1) ** 2


def test_maxwell_dof_counts(po):  # test_spaces.cpp:39-53
    d = po.Discretization("maxwell", 1, 1, 0, kappa=3.0)
    assert d.dof_count == 12 and d.local_count == 4
    for P in (1, 2):
        for L in (0, 1):
            d = po.Discretization("maxwell", P, 1, L, kappa=3.0)
            kp, kq = (1 << L) + P, (1 << L) + P - 1
            assert d.dof_count == 6 * 2 * kp * kq - 12 * kq


def test_invalid_configurations(po):  # test_spaces.cpp:55-60
    for args in (("maxwell", 0, 1, 1), ("maxwell", 1, 2, 1), ("laplace", 1, 5, 1), ("laplace", -1, 1, 1)):
        with pytest.raises(ValueError):
            po.Discretization(*args, kappa=3.0 if args[0] == "maxwell" else 0)


def test_partition_of_unity(po):  # test_spaces.cpp:62-71
    d = po.Discretization("laplace", 2, 1, 2)
    for e in (0, 17, 55, 95):
        for u in (0.0, 0.4, 1.0):
            for v in (0.2, 0.9):
                assert abs(d.sample_shapes(e, u, v)["value"].sum() - 1) < 1e-13


def test_classification_maps(po):  # test_spaces.cpp:100-137
    d = po.Discretization("laplace", 1, 1, 1)
    ints, dbl = d.elements()

    def phys(e, u, v):
        return d.frame(int(ints[e, 0]), dbl[e, 1] + dbl[e, 0] * u, dbl[e, 2] + dbl[e, 0] * v)["x"]

    def apply(m, u, v):
        if m[0]:
            u, v = v, u
        if m[1]:
            u = 1 - u
        if m[2]:
            v = 1 - v
        return u, v
    n = {po.COINCIDENT: 0, po.EDGE: 0, po.VERTEX: 0}
    for ea in range(d.element_count):
        for eb in range(d.element_count):
            cls, maps = d.classify_pair(ea, eb)
            assert d.classify_pair(eb, ea)[0] == cls
            if cls == po.FAR:
                continue
            n[cls] += 1
            if cls == po.EDGE:
                for t in (0.0, 0.5, 1.0):
                    xa = phys(ea, *apply(maps[:3], t, 0.0))
                    xb = phys(eb, *apply(maps[3:], t, 0.0))
                    assert np.linalg.norm(xa - xb) < 1e-12
            elif cls == po.VERTEX:
                assert np.linalg.norm(phys(ea, *apply(maps[:3], 0, 0)) - phys(eb, *apply(maps[3:], 0, 0))) < 1e-12
    assert n[po.COINCIDENT] == 24 and n[po.EDGE] == 96 and n[po.VERTEX] > 0


def test_laplace_dense_spd_equal_diagonals(po):  # test_assembly.cpp:20-29
    a = po.Discretization("laplace", 1, 1, 1).assemble_dense()
    assert np.abs(a - a.T).max() < 1e-14
    assert np.allclose(np.diag(a), a[0, 0], rtol=1e-10, atol=0)
    np.linalg.cholesky(a)


def test_shell_theorem(po):  # test_assembly.cpp:31-42
    a = po.Discretization("laplace", 0, 1, 0).assemble_dense(far_order=8, sing_order=8)
    s = a.sum(axis=1)
    assert np.all(np.abs(s - 4 * np.pi / 6) <= 2e-4 * 4 * np.pi / 6)


def test_flat_square_frozen_entries(po):  # test_assembly.cpp:44-67
    d = po.Discretization("laplace", 0, 1, 1, geometry="square")
    assert d.dof_count == 4
    a = d.assemble_dense(far_order=10, sing_order=10)
    ints, _ = d.elements()
    g, _ = d.l2g()
    for ea in range(4):
        for eb in range(4):
            dx, dy = abs(ints[ea, 1] - ints[eb, 1]), abs(ints[ea, 2] - ints[eb, 2])
            exp = K_COINCIDENT if dx + dy == 0 else (K_EDGE if dx + dy == 1 else K_VERTEX)
            assert abs(a[g[ea, 0], g[eb, 0]] - 0.125 * exp) <= 1e-7 * 0.125 * exp


def test_flat_far_entries(po):  # test_assembly.cpp:69-83
    d = po.Discretization("laplace", 0, 1, 2, geometry="square")
    a = d.assemble_dense(far_order=14, sing_order=10)
    g, _ = d.l2g()
    h3 = 0.25 ** 3
    e00, e20, e21 = 0, 2, 2 + 4
    assert abs(a[g[e00, 0], g[e20, 0]] - h3 * 4.064234359104e-02) <= 1e-8 * h3 * 4.064234359104e-02
    assert abs(a[g[e00, 0], g[e21, 0]] - h3 * 3.623121915119e-02) <= 1e-8 * h3 * 3.623121915119e-02


def test_helmholtz_kappa0_is_laplace(po):  # test_assembly.cpp:85-93
    for L in (0, 1):
        a = po.Discretization("laplace", 1, 1, L).assemble_dense()
        b = po.Discretization("helmholtz", 1, 1, L, kappa=0).assemble_dense()
        assert np.abs(b - a).max() < 1e-13


def test_complex_symmetric(po):  # test_assembly.cpp:95-104
    b = po.Discretization("helmholtz", 1, 1, 1, kappa=3.0).assemble_dense()
    assert np.abs(b - b.T).max() < 1e-14
    m = po.Discretization("maxwell", 1, 1, 1, kappa=3.0).assemble_dense()
    assert np.abs(m - m.T).max() < 1e-14


def test_admissibility(po):  # test_h2.cpp:60-73
    a = [0, 0, 0, 1, 1, 1]
    assert not po.admissible(a, a, 1.6)
    assert po.admissible(a, [10, 0, 0, 11, 1, 1], 1.6)
    assert not po.admissible(a, [1.5, 0, 0, 2.5, 1, 1], 1.6)
    assert po.admissible(a, [1.5, 0, 0, 2.5, 1, 1], 4.0)


@pytest.mark.parametrize("L", [2, 3])
def test_block_partition_exact_cover(po, L):  # test_h2.cpp:75-92
    d = po.Discretization("laplace", 0, 1, L)
    h = po.H2Matrix(d, m=4)
    n = d.element_count
    npp = sum(4 ** l for l in range(L + 1))
    offs = [sum(4 ** j for j in range(l)) for l in range(L + 1)]

    def decode(node):
        p, r = divmod(int(node), npp)
        l = max(i for i in range(L + 1) if offs[i] <= r)
        s = r - offs[l]
        return p, l, s % (1 << l), s >> l

    def leaves(node):
        p, l, sx, sy = decode(node)
        k = 1 << (L - l)
        return [p * (1 << 2 * L) + (sx * k + i) + (1 << L) * (sy * k + j) for j in range(k) for i in range(k)]
    cover = np.zeros((n, n), dtype=np.int32)
    for ea, eb in h.nearfield_pairs():
        cover[ea, eb] += 1
    for ta, tb in h.farfield_pairs():
        la, lb = leaves(ta), leaves(tb)
        cover[np.ix_(la, lb)] += 1
    assert (cover == 1).all()


def test_h2_vs_dense(po):  # test_h2.cpp:94-106
    for P in (0, 1):
        d = po.Discretization("laplace", P, 1, 2)
        a = d.assemble_dense()
        h = po.H2Matrix(d, m=8)
        rng = np.random.default_rng(P)
        worst = 0
        for _ in range(3):
            x = rng.uniform(-1, 1, d.dof_count)
            worst = max(worst, np.linalg.norm(h.apply(x) - a @ x) / np.linalg.norm(a @ x))
        assert worst < 1e-6


def test_interpolation_error_decreases(po):  # test_h2.cpp:108-119
    d = po.Discretization("laplace", 0, 1, 3)
    a = d.assemble_dense()
    x = np.random.default_rng(3).uniform(-1, 1, d.dof_count)
    ref = a @ x
    e4 = np.linalg.norm(po.H2Matrix(d, m=4).apply(x) - ref) / np.linalg.norm(ref)
    e8 = np.linalg.norm(po.H2Matrix(d, m=8).apply(x) - ref) / np.linalg.norm(ref)
    assert e8 < 1e-6 and e4 > 100 * e8


def test_complex_kinds_compress(po):  # test_h2.cpp:121-133
    for kind in ("helmholtz", "maxwell"):
        d = po.Discretization(kind, 1, 1, 2, kappa=3.0)
        a = d.assemble_dense()
        h = po.H2Matrix(d, m=8)
        rng = np.random.default_rng(7)
        x = rng.uniform(-1, 1, d.dof_count) + 1j * rng.uniform(-1, 1, d.dof_count)
        assert np.linalg.norm(h.apply(x) - a @ x) / np.linalg.norm(a @ x) < 1e-6


def test_storage_growth(po):  # test_h2.cpp:145-159
    entries = []
    for L in (2, 3, 4):
        h = po.H2Matrix(po.Discretization("laplace", 0, 1, L), m=4)
        assert h.nearfield_entries > 0 and h.farfield_entries > 0
        assert h.total_bytes >= (h.nearfield_entries + h.farfield_entries) * 8
        entries.append(h.nearfield_entries + h.farfield_entries)
    assert entries[1] / entries[0] < 6.5 and entries[2] / entries[1] < 5.0


def test_survey_partition_counts(po):  # SURVEY Appendix A cross-check (c1)
    h = po.H2Matrix(po.Discretization("laplace", 2, 1, 3), m=4, flags=3)
    assert (h.near_count, h.far_count) == (8760, 27456)
