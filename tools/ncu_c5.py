"""A config's operator + a few graph matvecs (ncu target).  `c5@L5` = c5 with
level 5 (same kernels, 1/64 of the work)."""
import sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
base, _, lv = name.partition("@L")
c = dict(CONFIGS[base])
if lv:
    c["L"] = int(lv)
d = make_disc(igb, c)
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]))
h.bench_apply(3)
