"""Full-size configuration check on one B200: assembly + matvec timings and
sampled near-field parity against the reference's own pair_block (oracle/_ref).
  python tools/check_big.py c5|c3|c4"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb  # noqa: E402
from oracle import pyref  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = CONFIGS[name]
pde = {"laplace": igb.Pde.laplace(), "helmholtz": igb.Pde.helmholtz(c["kappa"])}.get(c["kind"]) \
    if c["kind"] != "maxwell" else igb.Pde.maxwell(c["kappa"])
t0 = time.time()
d = igb.Discretization(igb.make_sphere(), pde, c["P"], c["rep"], c["L"])
t1 = time.time()
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]))
t2 = time.time()
print(f"{name}: dofs={d.dof_count()} elements={d.element_count()} near={h.near_count} far={h.far_count}")
print(f"  discretization {t1 - t0:.2f}s, H2Matrix ctor (plan+upload+assembly) {t2 - t1:.2f}s")
print("  assembly times", {k: round(v, 2) for k, v in h.assembly_times().items()})
print("  device bytes", h.device_bytes(), "class counts", h.class_counts())
ms, launches = h.bench_apply(5)
print(f"  matvec {ms / 5:.3f} ms ({launches} launches), phases", {k: round(v / 3, 4) for k, v in h.profile_apply(3).items()})
asm = h.reassemble()
print(f"  device re-assembly {asm[0]:.1f} ms")
x = np.random.default_rng(20261019).uniform(-1, 1, d.dof_count())
if h.dtype == np.complex128:
    x = x + 0j
y = h @ x
print("  |y|", np.linalg.norm(y), "finite", np.isfinite(y).all(), "deterministic", np.array_equal(h @ x, y))
if pyref.available():
    rd = pyref.Discretization(c["kind"], c["P"], c["rep"], c["L"], kappa=c["kappa"])
    near = h.nearfield_pairs()
    idx = np.unique(np.linspace(0, len(near) - 1, 48).astype(np.int64))
    t = time.time()
    ref = rd.pair_blocks(near[idx])
    got = np.stack([h.near_blocks(int(i), 1)[0] for i in idx])
    err = (np.abs(got - ref).max(axis=(1, 2)) / np.abs(ref).max(axis=(1, 2))).max()
    print(f"  sampled near blocks vs reference pair_block: {len(idx)} pairs, max rel {err:.2e} ({time.time() - t:.1f}s)")
    fidx = np.unique(np.linspace(0, h.far_count - 1, 16).astype(np.int64))
    K = np.stack([h.couplings(int(i), 1)[0] for i in fidx])
    print("  couplings finite", np.isfinite(K).all())
