"""c2 (or given case) device assembly timings per kernel (reassemble x3)."""
import sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
P, L, m = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (3, 6, 4)))
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), P, 1, L)
h = igb.H2Matrix(d, igb.H2Options(m=m))
for _ in range(3):
    h.reassemble()
t = h.assembly_times()
print({k: round(v, 3) for k, v in t.items() if k.endswith("_ms")})
