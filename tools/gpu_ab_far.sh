#!/bin/bash
# A/B of compile-time variants of the far-field kernel: far ms + c3 parity vs oracle
cd paper_1906_00785_b200
for v in "$@"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  (cd .. && python - "$v" << 'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1906_00785_b200 as igb
from oracle import pyoracle as po
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
h = igb.H2Matrix(d, igb.H2Options(m=4))
p = h.profile_apply(20); p = h.profile_apply(50)
od = po.Discretization("laplace", 3, 1, 3); oh = po.H2Matrix(od, m=4)
d3 = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 3); h3 = igb.H2Matrix(d3, igb.H2Options(m=4))
x = np.random.default_rng(0).uniform(-1, 1, od.dof_count)
y = oh.apply(x)
print(sys.argv[1], "far ms", round(p["far"] / 50, 4), "rel", np.linalg.norm(h3 @ x - y) / np.linalg.norm(y))
PY
  )
done
