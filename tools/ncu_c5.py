"""c5 operator, a few graph matvecs (ncu target: the far-field kernels)."""
import sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
d = make_disc(igb, c)
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]))
h.bench_apply(3)
