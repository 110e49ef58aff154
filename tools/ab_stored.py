"""Stored couplings (streamed, HBM-bound) vs on-the-fly couplings (FP64-bound)
per config: graph ms per apply and phase times.  python tools/ab_stored.py c4 [c3 ...]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc

for name in sys.argv[1:]:
    c = CONFIGS[name]
    d = make_disc(igb, c)
    for stored in (False, True):
        try:
            h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]), stored_couplings=stored)
        except Exception as e:  # noqa: BLE001
            print(name, "stored" if stored else "fused", "failed:", e)
            continue
        h.bench_apply(5)
        ms, _ = h.bench_apply(20)
        p = h.profile_apply(5)
        print(f"{name} {'stored' if stored else 'fused'}: {ms / 20:.3f} ms/apply, asm {h.assembly_times()['device_total_ms']:.1f} ms,"
              f" phases", {k: round(v / 5, 3) for k, v in p.items()}, h.device_bytes(), flush=True)
        del h
