import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 4, 1, L)
h = igb.H2Matrix(d, igb.H2Options(m=5, eta=1.6))
x = np.random.default_rng(1).uniform(-1, 1, d.dof_count())
y = h.apply(x)
tag = os.environ.get("TAG", "x")
np.save(f"gpurun_out/wsdbg_{tag}.npy", y)
print(tag, "ok", np.linalg.norm(y), flush=True)
if os.path.exists("gpurun_out/wsdbg_ref.npy"):
    r = np.load("gpurun_out/wsdbg_ref.npy")
    print(tag, "rel diff vs ref", np.linalg.norm(y - r) / np.linalg.norm(r))
