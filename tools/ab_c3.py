"""c3 (Helmholtz, m = 8) matvec time and a y dump: python tools/ab_c3.py tag [level]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
tag = sys.argv[1]
c = dict(CONFIGS["c3"])
if len(sys.argv) > 2:
    c["L"] = int(sys.argv[2])
d = make_disc(igb, c)
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]), stored_couplings=False)
h.bench_apply(2)
ms, _ = h.bench_apply(5)
p = h.profile_apply(2)
x = np.random.default_rng(20261019).uniform(-1, 1, d.dof_count()) + 0j
y = h.apply(x)
np.save(f"gpurun_out/c3_{tag}.npy", y)
print(tag, f"c3 L={c['L']}: {ms / 5:.2f} ms/apply", {k: round(v / 2, 3) for k, v in p.items()}, flush=True)
