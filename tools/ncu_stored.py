import sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
c = CONFIGS[sys.argv[1]]
d = make_disc(igb, c)
h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]), stored_couplings=True)
h.bench_apply(2)
