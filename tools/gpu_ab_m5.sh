#!/bin/bash
# A/B of the m = 5 lane grid of the symmetric far kernel on c5
cd paper_1906_00785_b200
for v in "-DIGB_M5_MINB=2" "-DIGB_M5_BR=2 -DIGB_M5_BC=16 -DIGB_M5_MINB=1"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  echo "variant: $v"
  (cd .. && python - << 'PY'
import sys; sys.path.insert(0, '.')
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 4, 1, 8)
h = igb.H2Matrix(d, igb.H2Options(m=5))
ms, n = h.bench_apply(20); ms, n = h.bench_apply(50)
p = h.profile_apply(10)
print("c5 graph ms/apply", round(ms / 50, 3), "far", round(p["far"] / 10, 3))
PY
  )
done
