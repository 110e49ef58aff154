"""CPU tests of the product's host side and C ABI (no device): the library
loads, exports every symbol of include/igabem_b200.h, builds the same
discretization and block partition as the oracle bit for bit, maps errors
to the reference's exception types, and refuses to run without a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "igabem_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|void)\s+(igb_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol(igb):
    syms = header_symbols()
    assert len(syms) > 30
    lib = igb.lib()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(igb.SYMBOLS)
    assert lib.igb_version() == 1


def test_library_is_sm100a(igb):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", igb.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


CASES = [("laplace", 0, 1, 2), ("laplace", 2, 1, 3), ("laplace", 3, 1, 3), ("laplace", 3, 2, 2),
         ("laplace", 4, 1, 2), ("helmholtz", 3, 1, 2), ("maxwell", 1, 1, 2), ("maxwell", 2, 1, 2)]


def _pde(igb, kind):
    if kind == "laplace":
        return igb.Pde.laplace()
    return igb.Pde.helmholtz(3.0) if kind == "helmholtz" else igb.Pde.maxwell(3.0)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_discretization_matches_oracle(igb, po, case):
    kind, P, rep, L = case
    d = igb.Discretization(igb.make_sphere(), _pde(igb, kind), P, rep, L)
    od = po.Discretization(kind, P, rep, L, kappa=3.0 if kind != "laplace" else 0)
    assert (d.dof_count(), d.element_count(), d.local_count()) == (od.dof_count, od.element_count, od.local_count)
    g, s = d.local_to_global()
    og, os_ = od.l2g()
    assert np.array_equal(g, og) and np.array_equal(s, os_)
    ei, ed = d.elements()
    oi, oe = od.elements()
    assert np.array_equal(ei, oi)
    assert np.array_equal(ed, oe)  # element boxes bit-identical: the partition depends on them


@pytest.mark.parametrize("case", CASES[:6], ids=lambda c: "-".join(map(str, c)))
def test_block_partition_matches_oracle(igb, po, case):
    kind, P, rep, L = case
    m = 4
    d = igb.Discretization(igb.make_sphere(), _pde(igb, kind), P, rep, L)
    plan = igb.H2Plan(d, igb.H2Options(m=m))
    od = po.Discretization(kind, P, rep, L, kappa=3.0 if kind != "laplace" else 0)
    oh = po.H2Matrix(od, m=m, flags=3)
    assert np.array_equal(plan.nearfield_pairs(), oh.nearfield_pairs())
    assert np.array_equal(plan.farfield_pairs(), oh.farfield_pairs())


def test_classification_matches_oracle_all_pairs(igb, po):
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 1, 1, 2)
    od = po.Discretization("laplace", 1, 1, 2)
    for ea in range(d.element_count()):
        for eb in range(d.element_count()):
            c1, m1 = d.classify_pair(ea, eb)
            c2, m2 = od.classify_pair(ea, eb)
            assert c1 == c2 and np.array_equal(m1, m2)


def test_class_counts_c2_structure(igb):
    # L6, P3 -> coincident 24,576, edge 98,304 (ordered), vertex 98,280, regular 339,072
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
    plan = igb.H2Plan(d, igb.H2Options(m=4))
    assert (plan.near_count, plan.far_count) == (560232, 2057544)
    cc = plan.class_counts()
    assert cc == dict(regular=339072, vertex=98280 // 2, edge=98304 // 2, coincident=24576)


@pytest.mark.parametrize("geom,kind,P,L", [("sphere", "laplace", 3, 0), ("sphere", "laplace", 1, 1),
                                           ("sphere", "laplace", 3, 4), ("sphere", "maxwell", 2, 3),
                                           ("square", "laplace", 2, 3), ("square", "helmholtz", 1, 0)])
def test_singular_items_from_topology(igb, geom, kind, P, L):
    """The device integrates the singular pairs before the block partition
    exists, enumerating them from the mesh topology; they must be exactly the
    near list's singular pairs (same order, same maps) on every rank."""
    g = igb.make_sphere() if geom == "sphere" else igb.make_square()
    d = igb.Discretization(g, _pde(igb, kind), P, 1, L)
    plan = igb.H2Plan(d, igb.H2Options(m=4))
    cc = plan.class_counts()
    counts, equal = plan.singular_items()
    assert equal
    assert counts == [cc["regular"], cc["vertex"], cc["edge"], cc["coincident"]]
    for world in (2, 3, 5):
        tot = np.zeros(4, dtype=np.int64)
        for r in range(world):
            c, equal = plan.singular_items(world, r)
            assert equal, (world, r)
            tot += c
        assert tot[3] == cc["coincident"]  # coincident items belong to exactly one rank


def test_row_partition_covers_everything(igb):
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 2, 1, 3)
    plan = igb.H2Plan(d, igb.H2Options(m=8))
    for world in (1, 2, 3, 4, 8):
        parts = [plan.partition(world, r) for r in range(world)]
        assert sum(p["elements"] for p in parts) == d.element_count()
        assert sum(p["near"] for p in parts) == plan.near_count
        # level-0 far pairs would be replicated; the sphere has none
        assert sum(p["far"] for p in parts) == plan.far_count
        assert parts[0]["clusters"][0] == 0 and parts[-1]["clusters"][1] == 24


def test_errors_map_reference_exceptions(igb):
    g = igb.make_sphere()
    with pytest.raises(ValueError):
        igb.Discretization(g, igb.Pde.laplace(), -1, 1, 1)
    with pytest.raises(ValueError):
        igb.Discretization(g, igb.Pde.maxwell(3.0), 1, 2, 1)
    with pytest.raises(ValueError):
        igb.Pde.maxwell(0)
    with pytest.raises(ValueError):
        igb.make_sphere(-1.0)
    d = igb.Discretization(g, igb.Pde.laplace(), 1, 1, 1)
    with pytest.raises(ValueError):
        igb.H2Plan(d, igb.H2Options(m=1))
    with pytest.raises(ValueError):
        igb.H2Plan(d, igb.H2Options(eta=-1.0))
    with pytest.raises(ValueError):
        d.classify_pair(0, 10 ** 6)


def test_custom_geometry_roundtrip(igb, po):
    # Geometry(std::vector<PatchSurface>) from raw patch data == make_sphere
    od = po.Discretization("laplace", 1, 1, 1)
    patches = []
    for p in range(6):
        pd = od.patch(p)
        patches.append(dict(degree_u=pd["pu"], degree_v=pd["pv"], knots_u=pd["ku"], knots_v=pd["kv"],
                            ctrl_w=pd["cw"].ravel(), weight=pd["w"]))
    g = igb.Geometry(patches)
    assert (g.patch_count(), g.edge_count(), g.vertex_count()) == (6, 12, 24)
    d = igb.Discretization(g, igb.Pde.laplace(), 1, 1, 2)
    _, e1 = d.elements()
    _, e2 = po.Discretization("laplace", 1, 1, 2).elements()
    assert np.array_equal(e1, e2)


def test_no_cpu_fallback_without_gpu(igb):
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("device present")
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 1, 1, 1)
    with pytest.raises(igb.CudaError):
        igb.H2Matrix(d)
