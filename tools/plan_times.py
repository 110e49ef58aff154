"""Block-partition time, host (OpenMP) vs device traversal/sort/transposes (c2, c5)."""
import sys
import time
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
import os
for P, L, m in ((3, 6, 4), (4, 8, 5)):
    d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), P, 1, L)
    o = igb.H2Options(m=m)
    igb.H2Plan(d, o, device=0)  # context / module load
    for dev in (None, 0):
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            igb.H2Plan(d, o, device=dev)
            ts.append(time.perf_counter() - t)
        print(f"L={L} P={P}: {'host' if dev is None else 'device'} partition plan {1e3 * min(ts):.1f} ms "
              f"(cores {os.cpu_count()})", flush=True)
