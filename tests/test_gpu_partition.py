"""the setup on the device -- element boxes, tree boxes and
diagonals, the block partition (traversal, sort, row starts, transposes) and
the classes and maps of the near pairs -- must equal the host's, and thereby
the reference's, bit for bit; an operator built on it gives the same matvec."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [("laplace", 0, 0, 4), ("laplace", 2, 3, 8), ("laplace", 3, 6, 4),
                                  ("helmholtz", 2, 4, 8), ("maxwell", 2, 3, 8)],
                         ids=lambda c: "-".join(map(str, c)))
def test_device_partition_equals_host(igb, case):
    kind, P, L, m = case
    pde = igb.Pde.laplace() if kind == "laplace" else (igb.Pde.helmholtz(3.0) if kind == "helmholtz"
                                                      else igb.Pde.maxwell(3.0))
    d = igb.Discretization(igb.make_sphere(), pde, P, 1, L)
    o = igb.H2Options(m=m)
    ph, pd = igb.H2Plan(d, o), igb.H2Plan(d, o, device=0)
    assert (pd.near_count, pd.far_count) == (ph.near_count, ph.far_count)
    assert np.array_equal(pd.nearfield_pairs(), ph.nearfield_pairs())
    assert np.array_equal(pd.farfield_pairs(), ph.farfield_pairs())
    # element and tree boxes computed on the device (eval_patch + inflation, unions)
    assert np.array_equal(pd.node_boxes(), ph.node_boxes())
    # classes and maps of the near pairs, classified on the device: the per-class
    # work lists (ea, eb, map bits) equal the mesh-topology enumeration of the host
    assert pd.class_counts() == ph.class_counts()
    assert pd.singular_items()[1]


def test_operator_on_device_partition(igb):
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 4)
    o = igb.H2Options(m=4)
    h1, h2 = igb.H2Matrix(d, o, device_partition=False), igb.H2Matrix(d, o, device_partition=True)
    x = np.random.default_rng(5).uniform(-1, 1, d.dof_count())
    assert np.array_equal(h1 @ x, h2 @ x)  # identical partition -> identical operator
