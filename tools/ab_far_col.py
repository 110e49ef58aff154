"""A/B of the far-field kernels (IGB_FAR_KERNEL / IGB_FAR_COL_MINB set by the
caller): graph time per apply, the graph's kernels serialised, and y for a
seeded x saved to gpurun_out/ab_<tag>_<cfg>.npy for cross-variant comparison."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc

tag = sys.argv[1]
for name in sys.argv[2:]:
    c = CONFIGS[name]
    d = make_disc(igb, c)
    h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]))
    n = 200 if name == "c2" else 40
    h.bench_apply(n)
    ms, _ = h.bench_apply(n)
    k = h.profile_kernels(10)
    x = np.random.default_rng(20261019).uniform(-1, 1, d.dof_count())
    y = h.apply(x)
    np.save(f"gpurun_out/ab_{tag}_{name}.npy", y)
    print(f"{tag} {name}: graph {ms / n:.4f} ms/apply;", {a: round(b / 10, 4) for a, b in k.items()}, flush=True)
