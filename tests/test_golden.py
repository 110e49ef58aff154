"""Golden fixtures produced by the REFERENCE itself (tests/golden/*.npz, made by
tools/make_golden.py from oracle/_ref = igabem core + Eigen-subset shim):
the CPU oracle must reproduce them (CPU), and the B200 path must too (GPU)."""
import glob
import os

import numpy as np
import pytest

GOLD = sorted(g for g in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
              if not os.path.basename(g).startswith("solve_"))  # solver fixtures: tests/test_gpu_solve.py
# full-size fixtures (c2, c4): only the B200 side runs them (the oracle's own
# c4 operator stores 34 GB of couplings; tests/test_gpu_full_size.py probes it)
BIG = [g for g in GOLD if os.path.basename(g).startswith(("c2_", "c4_"))]
SMALL = [g for g in GOLD if g not in BIG]


def load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("path", SMALL, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_reproduces_reference_golden(po, path):
    g = load(path)
    d = po.Discretization(str(g["kind"]), int(g["P"]), int(g["rep"]), int(g["L"]), kappa=float(g["kappa"]))
    h = po.H2Matrix(d, m=int(g["m"]), eta=float(g["eta"]))
    assert (h.near_count, h.far_count) == (int(g["near_count"]), int(g["far_count"]))
    assert (h.nearfield_entries, h.farfield_entries, h.total_bytes) == (
        int(g["nearfield_entries"]), int(g["farfield_entries"]), int(g["total_bytes"]))
    assert _rel(h.apply(g["x"]), g["y"]) < 1e-13
    blocks = d.pair_blocks(g["block_pairs"])
    assert np.abs(blocks - g["blocks"]).max() <= 1e-14 * np.abs(g["blocks"]).max()


def _pde(igb, g):
    kind = str(g["kind"])
    if kind == "laplace":
        return igb.Pde.laplace()
    k = float(g["kappa"])
    return igb.Pde.helmholtz(k) if kind == "helmholtz" else igb.Pde.maxwell(k)


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=lambda p: os.path.basename(p)[:-4])
def test_b200_reproduces_reference_golden(igb, path):
    g = load(path)
    d = igb.Discretization(igb.make_sphere(), _pde(igb, g), int(g["P"]), int(g["rep"]), int(g["L"]))
    h = igb.H2Matrix(d, igb.H2Options(m=int(g["m"]), eta=float(g["eta"])))
    assert (h.near_count, h.far_count) == (int(g["near_count"]), int(g["far_count"]))
    s = h.storage_report()
    assert (s.nearfield_entries, s.farfield_entries, s.total_bytes) == (
        int(g["nearfield_entries"]), int(g["farfield_entries"]), int(g["total_bytes"]))
    # matvec: north-star tolerance 1e-10 relative
    assert _rel(h.apply(g["x"]), g["y"]) < 1e-10
    # assembled near-field entries: 1e-10 relative per block
    near = h.nearfield_pairs()
    key = near[:, 0].astype(np.int64) * (1 << 32) + near[:, 1]
    want = g["block_pairs"][:, 0].astype(np.int64) * (1 << 32) + g["block_pairs"][:, 1]
    idx = np.searchsorted(key, want)
    assert np.array_equal(key[idx], want)
    got = np.stack([h.near_blocks(int(i), 1)[0] for i in idx])
    err = np.abs(got - g["blocks"]).max(axis=(1, 2)) / np.abs(g["blocks"]).max(axis=(1, 2))
    assert err.max() < 1e-10
