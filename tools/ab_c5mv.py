"""A/B probe: c5 matvec graph time (Laplace P=4, L=8, m=5) + ab_far's c2 numbers and parity."""
import subprocess, sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
name = sys.argv[1] if len(sys.argv) > 1 else "?"
subprocess.run([sys.executable, "tools/ab_far.py", name], check=True)
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 4, 1, 8)
h = igb.H2Matrix(d, igb.H2Options(m=5))
h.bench_apply(5)
ms, _ = h.bench_apply(20)
print(name, "c5 apply ms", round(ms / 20, 3))
