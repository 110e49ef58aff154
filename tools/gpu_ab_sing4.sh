#!/bin/bash
# A/B of singular-kernel variants on the c4 space (Maxwell, P=2) assembly
cd paper_1906_00785_b200
for v in "$@"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  echo "variant: $v"
  (cd .. && python - << 'PY'
import sys; sys.path.insert(0, '.')
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.maxwell(2 * 3.141592653589793), 2, 1, 5)
h = igb.H2Matrix(d, igb.H2Options(m=8))
for _ in range(2): h.reassemble()
t = h.assembly_times()
print({k: round(v, 2) for k, v in t.items() if k in ("coincident_ms", "edge_ms", "vertex_ms", "regular_ms", "elements_ms")})
PY
  )
done
