"""host-buffer apply vs graph-only time at a config: python tools/e2e_probe.py c5"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
d = make_disc(igb, c)
t = time.perf_counter(); h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"])); print("ctor", time.perf_counter() - t)
N = d.dof_count()
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, N)).pin_memory().numpy()
y = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
h.bench_apply(20)
ms, _ = h.bench_apply(100); print("graph ms/apply", ms / 100)
for rep in range(3):
    t = time.perf_counter()
    for _ in range(100):
        h.apply(x, out=y)
    print("host apply ms", (time.perf_counter() - t) * 10)
t = time.perf_counter(); del h; print("del", time.perf_counter() - t)
t = time.perf_counter(); h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"])); print("ctor warm", time.perf_counter() - t)
t = time.perf_counter()
for _ in range(100):
    h.apply(x, out=y)
print("host apply ms (fresh handle)", (time.perf_counter() - t) * 10)
for rep in range(2):
    t = time.perf_counter()
    for _ in range(100):
        h.apply(x, out=y)
    print("host apply ms (2nd handle, later)", (time.perf_counter() - t) * 10)
ms, _ = h.bench_apply(100); print("graph ms/apply (2nd handle)", ms / 100)
print({k: round(v / 10, 3) for k, v in h.profile_kernels(10).items()})
del h
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]))
t = time.perf_counter(); h.apply(x, out=y); print("first apply s", time.perf_counter() - t)
ms, _ = h.bench_apply(100); print("graph ms/apply (3rd handle)", ms / 100)
print({k: round(v / 10, 3) for k, v in h.profile_kernels(10).items()})
