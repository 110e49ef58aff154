#!/usr/bin/env python
"""bench.py -- B200 H² boundary-element hot path (assembly + matvecs).

Workload (N=1): BASELINE.json configs[1] = "c2": Laplace single layer on the
six-patch exact sphere (make_sphere, see DESIGN.md for the x/|x| substitution),
level 6, reference degree P=3 (C^1 quadratic density, 26,136 DOFs), H² with
eta = 1.6 and m = 4 Chebyshev points per direction (interpolation degree 3).
One step = full H² assembly + 100 matvecs (the config's "full assembly plus 100
matvecs").  Metric: DOF-matvecs per second over the whole step, in GDOF/s
(= 100 * N_dofs / step time / 1e9).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

`--impl reference` times the CPU reference algorithm on this host (oracle/_ref
-- the reference compiled against our Eigen-subset shim -- when built, else the
oracle/ restatement) on a bounded sample of the same workload, all host cores.
"""
import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: kind, reference degree P, repetition, level, m, eta, kappa, matvecs per step
    "c1": dict(kind="laplace", P=2, rep=1, L=3, m=8, eta=1.6, kappa=0j, matvecs=100),
    "c2": dict(kind="laplace", P=3, rep=1, L=6, m=4, eta=1.6, kappa=0j, matvecs=100),
    "c3": dict(kind="helmholtz", P=3, rep=1, L=7, m=8, eta=1.6, kappa=4 * np.pi + 0j, matvecs=100),
    "c4": dict(kind="maxwell", P=2, rep=1, L=5, m=8, eta=1.6, kappa=2 * np.pi + 0j, matvecs=100),
    "c5": dict(kind="laplace", P=4, rep=1, L=8, m=5, eta=1.6, kappa=0j, matvecs=1000),
}
FP64_PEAK_TFLOPS = 36.85  # DFMA microbenchmark on this pool's B200 (profiles/r01_fp64_peak_probe.txt)


class _Traffic(dict):
    def get(self, prefix, default=None):  # kernel names carry template arguments: match by prefix
        for k, v in self.items():
            if k == prefix or k.startswith(prefix.rstrip(">") + ",") or k.startswith(prefix):
                return v
        return default


def load_traffic():
    """per-launch DRAM bytes of the dominant kernels from the committed ncu capture"""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic_c2.json")) as f:
            return _Traffic(json.load(f)["kernels"])
    except Exception:
        return _Traffic()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def workload_name(name, c):
    return (f"{name}: {c['kind']} single layer, make_sphere, L={c['L']}, ref P={c['P']}, rep={c['rep']}, "
            f"m={c['m']}, eta={c['eta']}; step = H2 assembly + {c['matvecs']} matvecs")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in csv.reader(io.StringIO(self.out or "")) if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        load = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- CPU sample
def cpu_sample(c, sample_every=100, matvecs=3):
    """Bounded CPU run of the same workload with the reference's own code path:
    the H2Matrix ctor with 1-point singular rules (everything else -- cluster
    tree, traversal, couplings, moments, regular near blocks -- at full cost),
    plus the full-order singular work measured on every `sample_every`-th near
    pair (full minus 1-point, extrapolated), plus `matvecs` timed applies
    (extrapolated to the step's count)."""
    impl, kind = cpu_impl()
    od = impl.Discretization(c["kind"], c["P"], c["rep"], c["L"], kappa=c["kappa"])
    t0 = time.perf_counter()
    oh = impl.H2Matrix(od, m=c["m"], eta=c["eta"], sing_order=1)
    t_ctor1 = time.perf_counter() - t0
    pairs = oh.nearfield_pairs()
    samp = pairs[::sample_every]
    t0 = time.perf_counter()
    od.pair_blocks(samp)
    t_full = time.perf_counter() - t0
    t0 = time.perf_counter()
    od.pair_blocks(samp, sing_order=1)
    t_cheap = time.perf_counter() - t0
    t_near = max(t_full - t_cheap, 0.0) * len(pairs) / len(samp)
    x = np.random.default_rng(20261019).uniform(-1, 1, od.dof_count)
    if od.is_complex:
        x = x + 0j
    t0 = time.perf_counter()
    for _ in range(matvecs):
        oh.apply(x)
    t_mv = (time.perf_counter() - t0) / matvecs
    step = t_ctor1 + t_near + c["matvecs"] * t_mv
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    return dict(step_s=step, build_s=t_ctor1, near_s_extrap=t_near, matvec_s=t_mv, dofs=od.dof_count, cores=cores,
                kind=kind, sample=(f"{'reference igabem core (Eigen-subset shim)' if kind == 'reference' else 'oracle port'}"
                                   f": H2Matrix ctor with 1-point singular rules in full ({t_ctor1:.2f}s); full-order "
                                   f"singular quadrature on {len(samp)}/{len(pairs)} near pairs extrapolated "
                                   f"({t_near:.1f}s); {matvecs} applies extrapolated to {c['matvecs']} "
                                   f"({t_mv * 1e3:.1f} ms each); {cores} OpenMP threads"))


def cpu_impl():
    from oracle import pyoracle
    ref = os.path.join(ROOT, "oracle", "_ref", "libigabem_ref.so")
    if os.path.exists(ref):
        try:
            from oracle import pyref
            pyref.lib()
            return pyref, "reference"
        except Exception:
            pass
    return pyoracle, "port"


def run_reference(args, c, name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    for _ in range(min(args.warmup, 1)):
        cpu_sample(c, sample_every=1000, matvecs=1)
    vals = []
    info = None
    for _ in range(args.steps):
        info = cpu_sample(c)
        vals.append(info["step_s"])
    step = statistics.mean(vals)
    value = c["matvecs"] * info["dofs"] / step / 1e9
    line = {"metric": f"{name} H2 assembly + {c['matvecs']} matvecs throughput", "value": value, "unit": "GDOF/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (built-in make_sphere geometry, seeded uniform[-1,1] x)",
            "config": {"workload": workload_name(name, c), "dofs": info["dofs"]},
            "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": info["cores"], "kind": info["kind"],
                             "sample": info["sample"]},
            "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ B200 arm
def far_kernel_bytes(h, c):
    sw = 16 if h.dtype == np.complex128 else 8
    mm = c["m"] ** 2
    return h.far_count * mm * mm * sw


def run_b200(args, c, name):
    import torch
    import paper_1906_00785_b200 as igb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))
    else:
        dist = None
    dev = local
    if c["kind"] == "laplace":
        pde = igb.Pde.laplace()
    elif c["kind"] == "helmholtz":
        pde = igb.Pde.helmholtz(c["kappa"])
    else:
        pde = igb.Pde.maxwell(c["kappa"])
    geom = igb.make_sphere()
    disc = igb.Discretization(geom, pde, c["P"], c["rep"], c["L"])
    opts = igb.H2Options(m=c["m"], eta=c["eta"])
    N = disc.dof_count()
    mv = c["matvecs"]
    if world > 1 or args.force_dist:
        return run_dist(args, c, name, igb, torch, dist, disc, opts, world, rank, dev), None
    # -- setup: first assembly (plan + upload + kernels)
    h = igb.H2Matrix(disc, opts, device=dev)
    t_first = h.assembly_times()
    # -- warm-up
    for _ in range(args.warmup):
        h.bench_steps(1, mv)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev) as clk:
        total_ms, asm_ms = h.bench_steps(args.steps, mv)
    torch.cuda.synchronize(dev)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    asm_step = asm_ms / args.steps
    mv_ms = (ms_step - asm_step) / mv
    value = world * mv * N / (ms_step * 1e-3) / 1e9
    clocks = clk.summary()
    # -- per-kernel shares and rooflines
    times = h.assembly_times()
    # serialised phase times (shares / rooflines only; the step value above is
    # the timed region): warm the profiling path, best of three repetitions
    h.profile_apply(5)
    runs = [h.profile_apply(20) for _ in range(3)]
    prof = {k: min(r[k] for r in runs) / 20 for k in runs[0]}
    peaks, src = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    kernels = {
        "singular_edge": times["edge_ms"], "singular_vertex": times["vertex_ms"],
        "singular_coincident": times["coincident_ms"], "regular_near": times["regular_ms"],
        "couplings": times["couplings_ms"], "element_moments": times["elements_ms"], "images": times["images_ms"],
    }
    for k, v in prof.items():
        kernels["matvec_" + k] = v * mv
    dominant = max(kernels, key=kernels.get)
    sing_pts = singular_points(h, c)
    n_asm_k, n_mv_k = h.launch_counts()
    launches = args.steps * (n_asm_k + mv * n_mv_k)
    traffic = load_traffic()
    mm = c["m"] ** 2
    fp64 = FP64_PEAK_TFLOPS
    rooflines = {}
    far_ms = prof["far"]
    if h.stored_couplings:
        fb = far_kernel_bytes(h, c)
        rooflines["matvec_far"] = {"bound": "hbm", "achieved": fb / (far_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                   "peak_source": src, "bytes_per_launch": fb, "ms": far_ms}
    else:
        sym = c["kind"] == "laplace" and 2 <= c["m"] <= 6
        evals = (h.far_count // 2 if sym else h.far_count) * mm * mm
        # Laplace kernel 12 flop per evaluation, + 2 flop per product it
        # feeds (symmetric: K up[s] and K^T up[t]); complex kinds ~4x
        fl = evals * (16 if sym else 14) * (1 if h.dtype == np.float64 else 4)
        rooflines["matvec_far"] = {"bound": "fp64", "achieved": fl / (far_ms * 1e-3) / 1e12, "peak": fp64,
                                   "unit": "TFLOP/s", "peak_source": "measured DFMA probe (profiles/r01_fp64_peak_probe.txt)",
                                   "flops_per_launch": fl, "kernel_evals": evals, "ms": far_ms,
                                   "note": "couplings evaluated on the fly (symmetric: each unordered pair once)"
                                   if sym else "couplings evaluated on the fly"}
        # the profile path times the unfused far kernels (leaf + coarse launches)
        kt = traffic.get(f"k_far_sym_standalone<{c['m']}>") or traffic.get(f"k_far_sym<{c['m']}>")
        if kt:
            rooflines["matvec_far"]["traffic"] = kt["dram_read_bytes"] + kt["dram_write_bytes"]
    nb = h.device_bytes()["near"]
    rooflines["matvec_near"] = {"bound": "hbm", "achieved": nb / (prof["near_rows"] * 1e-3) / 1e9, "peak": hbm,
                                "unit": "GB/s", "peak_source": src, "bytes_per_launch": nb, "ms": prof["near_rows"],
                                "note": "near-field rows, timed serialised (overlapped with the far field in the graph)"}
    kt = traffic.get(f"k_near_rows<double, {disc.local_count()}>")
    if kt:
        rooflines["matvec_near"]["traffic"] = kt["dram_read_bytes"] + kt["dram_write_bytes"]
    for cls, key in (("edge", "edge_ms"), ("vertex", "vertex_ms"), ("coincident", "coincident_ms")):
        fl = sing_pts[cls] * flops_per_point(c, disc)
        ms = times[key]
        if ms > 0:
            rooflines["singular_" + cls] = {"bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": fp64,
                                           "unit": "TFLOP/s", "peak_source": "measured DFMA probe",
                                           "flops_per_launch": fl, "ms": ms, "points": sing_pts[cls]}
    for r in rooflines.values():
        r["frac"] = r["achieved"] / r["peak"]
        r.setdefault("traffic", None)
    dom_key = {"matvec_far": "matvec_far", "matvec_near_rows": "matvec_near", "singular_edge": "singular_edge",
               "singular_vertex": "singular_vertex", "singular_coincident": "singular_coincident"}.get(dominant, "matvec_far")
    roof = {k: rooflines[dom_key][k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
    roof["kernel"] = dom_key
    # -- e2e through the public API with host buffers
    e2e_times = []
    x_host = np.random.default_rng(20261019).uniform(-1, 1, N)
    if h.dtype == np.complex128:
        x_host = x_host + 0j
    upload = h.upload_bytes()
    del h
    for it in range(max(1, min(args.steps, 3)) + 1):
        t0 = time.perf_counter()
        he = igb.H2Matrix(disc, opts, device=dev)
        for _ in range(mv):
            y = he.apply(x_host)
        _ = float(y[0].real)
        dt = time.perf_counter() - t0
        if it > 0:
            e2e_times.append(dt)
        del he
    e2e_step = statistics.mean(e2e_times)
    if dist:
        t = torch.tensor([e2e_step], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())
    sw = 16 if np.iscomplexobj(x_host) else 8
    e2e = {"value": world * mv * N / e2e_step / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_step * 1e3,
           "h2d_bytes_per_step": int(upload + mv * N * sw), "d2h_bytes_per_step": int(mv * N * sw)}
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu and name in ("c1", "c2", "c4"):  # c3 / c5: CPU operator does not fit host RAM
            os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
            info = cpu_sample(c)
            cpu = {"value": mv * info["dofs"] / info["step_s"] / 1e9, "unit": "GDOF/s", "cores": info["cores"],
                   "kind": info["kind"], "sample": info["sample"], "step_s": info["step_s"]}
        out = {"metric": f"{name} H2 assembly + {mv} matvecs throughput", "value": value, "unit": "GDOF/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (built-in make_sphere geometry, seeded uniform[-1,1] x)",
               "config": {"workload": workload_name(name, c), "dofs": N,
                          "l2": "operator (couplings+near blocks) >> 126 MB L2: every matvec streams from HBM"},
               "assembly_ms": asm_step, "matvec_ms": mv_ms, "matvec_gdofs": N / (mv_ms * 1e-3) / 1e9,
               "first_assembly": t_first, "matvec_phase_ms": prof,
               "kernel_ms_per_step": kernels, "dominant_kernel": dominant,
               "roofline": roof, "rooflines": rooflines, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": clocks}
    return out, locals()


def run_dist(args, c, name, igb, torch, dist, disc, opts, world, rank, dev):
    """N > 1: the row-cluster partition (DistH2Matrix): each rank assembles the
    block rows of 24/N level-1 clusters; a matvec all-gathers the up moments
    and all-reduces y over NCCL.  Strong scaling: the c2 operator is fixed."""
    N = disc.dof_count()
    mv = c["matvecs"]
    D = igb.DistH2Matrix(disc, opts, device=dev)
    dt = D.dtype
    x = torch.empty(N, dtype=dt, device=f"cuda:{dev}").uniform_(-1, 1) if dt == torch.float64 else \
        torch.complex(torch.empty(N, dtype=torch.float64, device=f"cuda:{dev}").uniform_(-1, 1),
                      torch.zeros(N, dtype=torch.float64, device=f"cuda:{dev}"))
    y = torch.empty_like(x)

    def step():
        D.h.reassemble()
        for _ in range(mv):
            D.apply(x, y)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record()
        asm = 0.0
        for _ in range(args.steps):
            asm += D.h.reassemble()[0]
            for _ in range(mv):
                D.apply(x, y)
        e1.record()
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, asm], device=f"cuda:{dev}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, asm_step = float(t[0]) / args.steps, float(t[1]) / args.steps
    # e2e: public API with host buffers (plan + assembly + 100 x (H2D x, matvec, D2H y))
    x_host = np.random.default_rng(20261019).uniform(-1, 1, N)
    e2e_t = []
    for it in range(2):
        dist.barrier()
        t0 = time.perf_counter()
        De = igb.DistH2Matrix(disc, opts, device=dev)
        xs = torch.empty(N, dtype=De.dtype, device=f"cuda:{dev}")
        for _ in range(mv):
            xs.copy_(torch.from_numpy(x_host).to(De.dtype).pin_memory(), non_blocking=True)
            yh = De.apply(xs).cpu()
        float(yh[0].real)
        if it:
            e2e_t.append(time.perf_counter() - t0)
        del De
    tt = torch.tensor([max(e2e_t)], device=f"cuda:{dev}", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_step = float(tt)
    n_asm, n_mv = D.h.launch_counts()
    if rank != 0:
        return None
    sw = 16 if dt == torch.complex128 else 8
    return {"metric": f"{name} H2 assembly + {mv} matvecs throughput", "value": mv * N / (ms_step * 1e-3) / 1e9,
            "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (built-in make_sphere geometry, seeded uniform[-1,1] x)",
            "config": {"workload": workload_name(name, c), "dofs": N, "parallelism": f"row clusters x{world}",
                       "l2": "operator >> L2 per rank; matvec = phase-1 graph, NCCL all-gather, phase-2 graph, NCCL all-reduce"},
            "assembly_ms": asm_step, "matvec_ms": (ms_step - asm_step) / mv,
            "e2e": {"value": mv * N / e2e_step / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_step * 1e3,
                    "h2d_bytes_per_step": int(mv * N * sw), "d2h_bytes_per_step": int(mv * N * sw)},
            "gpu_launches": args.steps * (n_asm + mv * n_mv), "clocks": clk.summary(), "cpu_baseline": None,
            "roofline": None}


def singular_points(h, c):
    """quadrature points executed per singular class (unique pairs x rule size;
    coincident items run half the 8 n^4 rule and add the transpose)"""
    n4 = (c["P"] + 3) ** 4
    cc = h.class_counts()
    return {"coincident": cc["coincident"] * 4 * n4, "edge": cc["edge"] * 6 * n4, "vertex": cc["vertex"] * 4 * n4}


def flops_per_point(c, disc):
    """FP64 flops of one singular quadrature point in this implementation
    (FMA = 2): 2 rational degree-4 jets (4 homogeneous components x 55 FMA +
    rational/normal ~30 flops), kernel ~12, weights 6, shapes 2*(2*(q+1)*q +
    (q+1)^2) FMA-ish, staging nl multiplies, and the nl^2 FMA outer product."""
    nl = disc.local_count()
    q = int(round(nl ** 0.5)) - 1
    jet = 4 * 55 * 2 + 30
    shapes = 2 * (2 * (q + 1) * q * 2 + (q + 1) ** 2)
    return 2 * jet + 12 + 6 + shapes + nl + 2 * nl * nl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--force-dist", action="store_true",
                    help="test aid: run the multi-GPU (NCCL) path even at one rank (under torchrun)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, c, args.config)
    out, ctx = run_b200(args, c, args.config)
    if isinstance(out, tuple):
        out = out[0]
    if out is not None:
        print(json.dumps(out), flush=True)
    try:
        import torch.distributed as tdist
        if tdist.is_available() and tdist.is_initialized():
            tdist.barrier()
            tdist.destroy_process_group()
    except Exception:  # noqa: BLE001 -- teardown only
        pass
    return 0


if __name__ == "__main__":
    sys.exit(main())
