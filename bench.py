#!/usr/bin/env python
"""bench.py -- B200 H² boundary-element hot path (assembly + matvecs).

Workload (N=1): BASELINE.json configs[4] = "c5", the configuration the
metric ("H2 assembly time & matvec GDOF/s at 1/2/4/8 B200") is quoted on:
Laplace single layer on the six-patch exact sphere (make_sphere, see DESIGN.md
for the x/|x| substitution), level 8, reference degree P=4 (C^2 cubic density,
402,486 DOFs), H² with eta = 1.6 and m = 5 Chebyshev points per direction
(interpolation degree 4).  One step = full H² assembly + 1000 matvecs of
seeded uniform[-1,1] vectors.  Metric: DOF-matvecs per second over the whole
step, in GDOF/s (= 1000 * N_dofs / step time / 1e9).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl b200|reference]

`--impl reference` times the reference's own CPU implementation of the path
(oracle/_ref: the reference's core sources compiled against our Eigen-subset
shim; the oracle/ restatement if that is missing) on this host's cores, on a
bounded, declared sample of the same workload (RefSample below).
`--gpus N` without torchrun re-launches itself under torch.distributed.run.
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

# kind, reference degree P, repetition, level, m, eta, kappa, matvecs per step;
# near / far: ordered pair counts of the reference's block partition (SURVEY
# 8(a5); the B200 plan reproduces them bit for bit and run_b200 asserts them)
CONFIGS = {
    "c1": dict(kind="laplace", P=2, rep=1, L=3, m=8, eta=1.6, kappa=0j, matvecs=100, near=8760, far=27456),
    "c2": dict(kind="laplace", P=3, rep=1, L=6, m=4, eta=1.6, kappa=0j, matvecs=100, near=560232, far=2057544),
    "c3": dict(kind="helmholtz", P=3, rep=1, L=7, m=8, eta=1.6, kappa=4 * np.pi + 0j, matvecs=100,
               near=2237784, far=8094432),
    "c4": dict(kind="maxwell", P=2, rep=1, L=5, m=8, eta=1.6, kappa=2 * np.pi + 0j, matvecs=100,
               near=140232, far=515904),
    "c5": dict(kind="laplace", P=4, rep=1, L=8, m=5, eta=1.6, kappa=0j, matvecs=1000, near=8947080, far=32153256),
}
DEFAULT_CONFIG = "c5"
FP64_PEAK_TFLOPS = 36.85  # DFMA microbenchmark on this pool's B200 (profiles/r01_fp64_peak_probe.txt)
DATA = "synthetic (built-in make_sphere geometry, seeded uniform[-1,1] x)"


def workload_name(name, c):
    return (f"{name}: {c['kind']} single layer, make_sphere, L={c['L']}, ref P={c['P']}, rep={c['rep']}, "
            f"m={c['m']}, eta={c['eta']}; step = H2 assembly + {c['matvecs']} matvecs")


def config_dict(name, c, dofs, world=1):
    """The `config` of both arms (identical dicts)."""
    return {"workload": workload_name(name, c), "dofs": int(dofs), "parallelism": f"row clusters x{world}",
            "l2": "operator (near blocks + moments) >> 126 MB L2: every matvec streams from HBM, no flush needed"}


def metric_name(name, c):
    return f"{name} H2 assembly + {c['matvecs']} matvecs throughput"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def load_traffic(name):
    """per-launch DRAM bytes of the graph's kernels from the committed ncu capture"""
    try:
        with open(os.path.join(ROOT, "profiles", f"r02_ncu_traffic_{name}.json")) as f:
            return json.load(f)["kernels"]
    except Exception:
        return {}


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


def algorithmic_bytes(near, far, ne, nn, dofs, nl, m, nch, sw):
    """Reference-format bytes one apply streams: near blocks,
    couplings, moments (twice: forward + backward), x / y and up / down."""
    mm = m * m
    return (near * nl * nl + far * mm * mm + 2 * ne * nch * mm * nl + 2 * dofs + 4 * nn * mm * nch) * sw


class RefSample:
    """Bounded sample of the reference's own CPU path at a config (declared
    extrapolation; the full c5 step is ~10 CPU-hours and its couplings alone
    are 161 GB):

    * near-field blocks: the reference's pair_block (pair_integration.hpp:139-148,
      the code H2Matrix's ctor runs per near pair, h2.cpp:236-243) at the
      config's full quadrature orders on a seeded sample of ordered pairs per
      class -- coincident / edge / vertex / regular -- of the full-size mesh,
      each classified by the reference's classify_pair; per-pair time x the
      full-size class counts (singular from the sphere's mesh topology:
      coincident ne, edge 4 ne, vertex 4 ne - 24; regular = near - singular);
    * the rest of the ctor (cluster tree, traversal, couplings, moments): the
      reference's H2Matrix ctor at the config's P and m on level Ls = min(L, 5)
      with 1-point quadrature rules, scaled by the far-pair ratio;
    * apply: the reference's apply on that level-Ls operator, scaled by the
      ratio of reference-format algorithmic bytes."""

    def __init__(self, c):
        self.c = c
        self.impl, self.kind = cpu_impl()
        k = c
        t0 = time.perf_counter()
        self.disc = self.impl.Discretization(k["kind"], k["P"], k["rep"], k["L"], kappa=k["kappa"])
        self.t_disc = time.perf_counter() - t0
        self.ls = min(k["L"], 5)
        self.disc_s = self.disc if self.ls == k["L"] else \
            self.impl.Discretization(k["kind"], k["P"], k["rep"], self.ls, kappa=k["kappa"])
        self.cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
        ne = self.disc.element_count
        self.counts = {"coincident": ne, "edge": 4 * ne, "vertex": 4 * ne - 24}
        self.counts["regular"] = k["near"] - sum(self.counts.values())
        self.x_s = np.random.default_rng(20261019).uniform(-1, 1, self.disc_s.dof_count)
        if self.disc_s.is_complex:
            self.x_s = self.x_s + 0j
        self.small = None

    def pairs(self, cls, n, seed):
        """n ordered pairs of class `cls` around seeded interior elements of
        random patches (orientation alternating), asserted by classify_pair"""
        L = self.c["L"]
        side = 1 << L
        rng = np.random.default_rng(seed)
        want = {"coincident": 3, "edge": 2, "vertex": 1, "regular": 0}[cls]
        out = []
        while len(out) < n:
            p = int(rng.integers(0, self.disc.patch_count))
            ix, iy = (int(v) for v in rng.integers(0, max(side - 2, 1), 2))
            e = p * side * side + ix + side * iy
            if cls == "coincident":
                a, b = e, e
            elif cls == "edge":
                a, b = e, e + (1 if len(out) % 2 else side)
            elif cls == "vertex":
                a, b = (e, e + side + 1) if len(out) % 2 else (e + 1, e + side)
            else:
                a, b = e, e + 2 + (side if len(out) % 2 else 0)
            if side < 4 and cls == "regular":
                raise RuntimeError("level too small for the regular sample")
            if len(out) % 4 >= 2:
                a, b = b, a
            if self.disc.classify_pair(a, b)[0] != want:
                continue
            out.append((a, b))
        return np.asarray(out, dtype=np.int32)

    def step(self, seed=0):
        """One bounded sample: returns the extrapolated full step (s) + details."""
        c = self.c
        per = {}
        nsamp = {"coincident": 2 * self.cores, "edge": 2 * self.cores, "vertex": 2 * self.cores,
                 "regular": 8 * self.cores}
        for cls in ("coincident", "edge", "vertex", "regular"):
            pr = self.pairs(cls, nsamp[cls], seed * 7 + len(per))
            t0 = time.perf_counter()
            self.disc.pair_blocks(pr)
            per[cls] = (time.perf_counter() - t0) / len(pr)
        t_near = sum(self.counts[k] * per[k] for k in per)
        if self.small is None:  # level-Ls operator, 1-point rules (ctor time measured once per sample object)
            t0 = time.perf_counter()
            self.small = self.impl.H2Matrix(self.disc_s, m=c["m"], eta=c["eta"], far_order=1, sing_order=1)
            self.t_small_ctor = time.perf_counter() - t0
        hs = self.small
        t0 = time.perf_counter()
        hs.apply(self.x_s)
        t_apply_s = time.perf_counter() - t0
        sw = 16 if self.disc.is_complex else 8
        nl = self.disc.local_count
        nch = 4 if c["kind"] == "maxwell" else 1
        nn_full = 6 * (4 ** (c["L"] + 1) - 1) // 3
        b_full = algorithmic_bytes(c["near"], c["far"], self.disc.element_count, nn_full, self.disc.dof_count,
                                   nl, c["m"], nch, sw)
        b_small = algorithmic_bytes(hs.near_count, hs.far_count, self.disc_s.element_count, hs.node_count,
                                    self.disc_s.dof_count, nl, c["m"], nch, sw)
        t_rest = self.t_small_ctor * c["far"] / max(hs.far_count, 1)
        t_apply = t_apply_s * b_full / b_small
        step = t_near + t_rest + c["matvecs"] * t_apply
        sample = (f"{'reference igabem core (Eigen-subset shim)' if self.kind == 'reference' else 'oracle port'}, "
                  f"{self.cores} OpenMP threads: pair_block at full order on "
                  f"{', '.join(f'{nsamp[k]} {k}' for k in per)} ordered pairs of the L={c['L']} mesh x full-size "
                  f"class counts ({t_near:.0f} s); H2Matrix ctor at L={self.ls} (1-point rules) "
                  f"{self.t_small_ctor:.2f} s x far-pair ratio {c['far'] / max(hs.far_count, 1):.1f} "
                  f"({t_rest:.1f} s); apply at L={self.ls} {t_apply_s * 1e3:.1f} ms x algorithmic-bytes ratio "
                  f"{b_full / b_small:.1f} = {t_apply:.2f} s per matvec")
        return step, dict(near_s=t_near, rest_s=t_rest, matvec_s=t_apply, per_pair_s=per, sample=sample)


def run_reference(args, c, name):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    rs = RefSample(c)
    for w in range(args.warmup):
        rs.step(seed=1000 + w)
    vals, info = [], None
    for k in range(args.steps):
        s, info = rs.step(seed=k)
        vals.append(s)
    step = statistics.mean(vals)
    value = c["matvecs"] * rs.disc.dof_count / step / 1e9
    line = {"metric": metric_name(name, c), "value": value, "unit": "GDOF/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config_dict(name, c, rs.disc.dof_count, args.gpus),
            "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": rs.cores, "kind": rs.kind,
                             "sample": info["sample"]},
            "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "breakdown_s": {k: info[k] for k in ("near_s", "rest_s", "matvec_s")}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ B200 arm
def make_disc(igb, c):
    if c["kind"] == "laplace":
        pde = igb.Pde.laplace()
    elif c["kind"] == "helmholtz":
        pde = igb.Pde.helmholtz(c["kappa"])
    else:
        pde = igb.Pde.maxwell(c["kappa"])
    return igb.Discretization(igb.make_sphere(), pde, c["P"], c["rep"], c["L"])


def load_pipes(name):
    """ncu-measured FP64 / DMMA pipe utilisation of the kernels (committed capture)"""
    try:
        with open(os.path.join(ROOT, "profiles", f"r02_ncu_pipes_{name}.json")) as f:
            return json.load(f)["kernels"]
    except Exception:
        return {}


def kernel_rooflines(h, c, disc, prof, iters, peaks, src, traffic):
    """Rooflines of the matvec graph's own kernels (timed serialised, CUDA
    events): algorithmic work per launch / average launch time."""
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    mm = c["m"] ** 2
    sym = h.far_sym_counts()
    near_bytes = h.device_bytes()["near"]
    out = {}

    def fp64(key, evals, ms, note):
        fl = evals * 16  # Laplace kernel 12 flop + 2 per product it feeds (K up[s] and K^T up[t])
        out[key] = {"bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "peak_source": "measured DFMA probe (profiles/r01_fp64_peak_probe.txt)",
                    "flops_per_launch": fl, "kernel_evals": evals, "ms": ms, "note": note}

    blk_pairs, blk_bytes, stream_bytes = h.leaf_blocks()
    if "far_near" in prof:  # k_leaf_ws: far field of every level + near rows + leaf blocks in one launch
        ms = prof["far_near"] / iters
        fp64("far_near", (sym["leaf"] + sym["coarse"]) * mm * mm, ms,
             "warp-specialised kernel: far warps evaluate the couplings of the unordered far pairs of every level "
             "(m^4 evaluations each), stream warps move the near rows and the leaf blocks (bulk copies)")
        r = out["far_near"]
        r["fp64_frac"] = r["achieved"] / r["peak"]
        r["hbm_bytes_per_launch"] = stream_bytes  # block rows: near field (once per unordered pair) + leaf blocks
        r["hbm_achieved_gbs"] = stream_bytes / (ms * 1e-3) / 1e9
        r["hbm_frac"] = r["hbm_achieved_gbs"] / hbm
        r["leaf_block_pairs"] = blk_pairs
        if r["hbm_frac"] > r["fp64_frac"]:  # report the roofline the kernel sits closer to
            r.update({"bound": "hbm", "achieved": r["hbm_achieved_gbs"], "peak": hbm, "unit": "GB/s",
                      "peak_source": src})
    if "far_leaf_near" in prof:
        ms = prof["far_leaf_near"] / iters
        fp64("far_leaf_near", sym["leaf"] * mm * mm, ms,
             "leaf-level far field (unordered leaf pairs x m^4 evaluations, couplings recomputed) fused with all "
             "near-field rows and the leaf blocks")
        out["far_leaf_near"]["hbm_achieved_gbs"] = (near_bytes + blk_bytes) / (ms * 1e-3) / 1e9
        out["far_leaf_near"]["hbm_frac"] = out["far_leaf_near"]["hbm_achieved_gbs"] / hbm
        out["far_leaf_near"]["near_bytes_per_launch"] = near_bytes + blk_bytes
    if "far_leaf" in prof:
        fp64("far_leaf", sym["leaf"] * mm * mm, prof["far_leaf"] / iters, "leaf-level far field")
    if "far_coarse" in prof:
        fp64("far_coarse", sym["coarse"] * mm * mm, prof["far_coarse"] / iters, "far field above the leaf level")
    if "far" in prof:  # plain graph: one far-field phase (stored couplings streamed, or evaluated symmetrically)
        ms = prof["far"] / iters
        far_bytes = h.device_bytes()["far"]
        if far_bytes > 0:
            out["far"] = {"bound": "hbm", "achieved": far_bytes / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                          "peak_source": src, "bytes_per_launch": far_bytes, "ms": ms,
                          "note": "stored couplings (reference format) streamed once per matvec"}
        else:
            cplx = c["kind"] != "laplace"
            evals = h.far_count // 2 * mm * mm * (4 if c["kind"] == "maxwell" else 1)
            fl = evals * (80 if cplx else 16)
            out["far"] = {"bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "peak_source": "measured DFMA probe (profiles/r01_fp64_peak_probe.txt)",
                          "flops_per_launch": fl, "kernel_evals": evals, "ms": ms,
                          "note": "couplings evaluated once per unordered pair; complex kernel counted as 80 flop "
                                  "per evaluation (~40 FP64 instructions), real as 16"}
    if "near_rows" in prof:
        ms = prof["near_rows"] / iters
        out["near_rows"] = {"bound": "hbm", "achieved": near_bytes / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                            "peak_source": src, "bytes_per_launch": near_bytes, "ms": ms}
    for k, r in out.items():
        r["frac"] = r["achieved"] / r["peak"]
        t = traffic.get(k)
        r["traffic"] = t
    return out


def run_b200(args, c, name):
    import torch
    import paper_1906_00785_b200 as igb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))
    dev = local
    disc = make_disc(igb, c)
    opts = igb.H2Options(m=c["m"], eta=c["eta"])
    N = disc.dof_count()
    mv = c["matvecs"]
    if dist is not None:
        return run_dist(args, c, name, igb, torch, dist, disc, opts, world, rank, dev)
    # -- setup: first assembly (plan + upload + kernels)
    h = igb.H2Matrix(disc, opts, device=dev)
    if (h.near_count, h.far_count) != (c["near"], c["far"]):
        raise RuntimeError(f"partition counts {h.near_count}/{h.far_count} differ from the reference's "
                           f"{c['near']}/{c['far']}")
    t_first = h.assembly_times()
    for _ in range(args.warmup):
        h.bench_steps(1, mv)
    torch.cuda.synchronize(dev)
    with ClockSampler(dev) as clk:
        total_ms, asm_ms = h.bench_steps(args.steps, mv)
    torch.cuda.synchronize(dev)
    ms_step = total_ms / args.steps
    asm_step = asm_ms / args.steps
    mv_ms = (ms_step - asm_step) / mv
    value = mv * N / (ms_step * 1e-3) / 1e9
    clocks = clk.summary()
    # -- per-kernel times: assembly kernels (CUDA events of the last assembly)
    # and the matvec graph's own kernels launched serialised (best of three)
    times = h.assembly_times()
    iters = 20
    try:
        h.profile_kernels(3)
        runs = [h.profile_kernels(iters) for _ in range(3)]
    except igb.LogicError:  # no level-split graph (complex kinds, m > 6): the phases of the plain graph
        h.profile_apply(3)
        runs = [{k: v for k, v in h.profile_apply(iters).items() if v > 0} for _ in range(3)]
    prof = {k: min(r[k] for r in runs) for k in runs[0]}
    peaks, src = load_peaks()
    kernels = {"singular_edge": times["edge_ms"], "singular_vertex": times["vertex_ms"],
               "singular_coincident": times["coincident_ms"], "regular_near": times["regular_ms"],
               "element_moments": times["elements_ms"], "images": times["images_ms"],
               "singular_scatter": times["scatter_ms"]}
    for k, v in prof.items():
        kernels["matvec_" + k] = v / iters * mv
    dominant = max(kernels, key=kernels.get)
    rooflines = kernel_rooflines(h, c, disc, prof, iters, peaks, src, load_traffic(name))
    sing_pts = singular_points(h, c)
    for cls, key in (("edge", "edge_ms"), ("vertex", "vertex_ms"), ("coincident", "coincident_ms")):
        ms = times[key]
        if ms > 0:
            fl = sing_pts[cls] * flops_per_point(c, disc)
            rooflines["singular_" + cls] = {
                "bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "peak_source": "measured DFMA probe", "flops_per_launch": fl, "ms": ms, "points": sing_pts[cls],
                "note": "per-point flop model of the unfactorised evaluation (bench.flops_per_point)",
                "frac": fl / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, "traffic": None}
    for k, v in load_pipes(name).items():  # hardware measure next to the model fractions
        if k in rooflines:
            rooflines[k]["ncu_fp64_pipe_pct"] = v["fp64_pipe_pct"]
            rooflines[k]["ncu_dmma_pipe_pct"] = v["dmma_pipe_pct"]
    dom_key = dominant[len("matvec_"):] if dominant.startswith("matvec_") else dominant
    if dom_key not in rooflines:
        dom_key = next((k for k in ("far_near", "far_leaf_near") if k in rooflines), next(iter(rooflines)))
    roof = {k: rooflines[dom_key][k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
    roof["kernel"] = dom_key
    n_asm_k, n_mv_k = h.launch_counts()
    launches = args.steps * (n_asm_k + mv * n_mv_k)
    # -- e2e through the public API with host buffers: H2Matrix(disc) (host
    # plan + uploads + kernels) + mv x apply(host x) (H2D x, graph, D2H y)
    # x and y in page-locked host memory (the contract's pinned host buffers)
    tdt = torch.complex128 if h.dtype == np.complex128 else torch.float64
    x_host = torch.from_numpy(np.random.default_rng(20261019).uniform(-1, 1, N)).to(tdt).pin_memory().numpy()
    y_host = torch.empty(N, dtype=tdt).pin_memory().numpy()
    upload = h.upload_bytes()
    del h
    e2e_times = []
    e2e_steps = max(1, min(args.steps, 3))
    for it in range(e2e_steps + 1):
        t0 = time.perf_counter()
        he = igb.H2Matrix(disc, opts, device=dev)
        for _ in range(mv):
            y = he.apply(x_host, out=y_host)
        _ = float(y[0].real)
        dt = time.perf_counter() - t0
        if it > 0:
            e2e_times.append(dt)
        del he
    e2e_step = statistics.mean(e2e_times)
    sw = 16 if np.iscomplexobj(x_host) else 8
    e2e = {"value": mv * N / e2e_step / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_step * 1e3,
           "steps": e2e_steps, "h2d_bytes_per_step": int(upload + mv * N * sw), "d2h_bytes_per_step": int(mv * N * sw)}
    cpu = None
    if not args.no_cpu:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
        rs = RefSample(c)
        s, info = rs.step(seed=0)
        cpu = {"value": mv * N / s / 1e9, "unit": "GDOF/s", "cores": rs.cores, "kind": rs.kind,
               "sample": info["sample"], "step_s": s}
    return {"metric": metric_name(name, c), "value": value, "unit": "GDOF/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": DATA, "config": config_dict(name, c, N, 1),
            "assembly_ms": asm_step, "matvec_ms": mv_ms, "matvec_gdofs": N / (mv_ms * 1e-3) / 1e9,
            "first_assembly": t_first, "matvec_kernel_ms": {k: v / iters for k, v in prof.items()},
            "kernel_ms_per_step": kernels, "dominant_kernel": dominant, "roofline": roof, "rooflines": rooflines,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}


def run_dist(args, c, name, igb, torch, dist, disc, opts, world, rank, dev):
    """N > 1: the row-cluster partition (DistH2Matrix): each rank assembles the
    block rows of 24/N level-1 clusters; a matvec all-gathers the up moments
    and all-reduces y over NCCL.  Strong scaling: the operator is fixed."""
    N = disc.dof_count()
    mv = c["matvecs"]
    D = igb.DistH2Matrix(disc, opts, device=dev)
    dt = D.dtype
    gen = torch.Generator(device="cpu").manual_seed(20261019)
    x = torch.rand(N, dtype=torch.float64, generator=gen).mul_(2).sub_(1).to(f"cuda:{dev}").to(dt)
    y = torch.empty_like(x)

    def step():
        torch.cuda.synchronize(dev)  # the assembly rewrites what queued matvecs read
        a = D.h.reassemble()[0]
        for _ in range(mv):
            D.apply(x, y)
        return a

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record()
        asm = 0.0
        for _ in range(args.steps):
            asm += step()
        e1.record()
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, asm], device=f"cuda:{dev}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, asm_step = float(t[0]) / args.steps, float(t[1]) / args.steps
    # e2e: public API with host buffers (plan + assembly + mv x (H2D x, matvec, D2H y))
    x_host = torch.from_numpy(np.random.default_rng(20261019).uniform(-1, 1, N)).to(dt).pin_memory()
    e2e_t = []
    for it in range(2):
        dist.barrier()
        t0 = time.perf_counter()
        De = igb.DistH2Matrix(disc, opts, device=dev)
        xs = torch.empty(N, dtype=De.dtype, device=f"cuda:{dev}")
        for _ in range(mv):
            xs.copy_(x_host, non_blocking=True)
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
    return {"metric": metric_name(name, c), "value": mv * N / (ms_step * 1e-3) / 1e9,
            "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config_dict(name, c, N, world),
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
    """FP64 flops of one singular quadrature point, direct (unfactorised)
    evaluation (FMA = 2): 2 rational degree-4 jets (4 homogeneous components x
    55 FMA + rational/normal ~30 flops), kernel ~12, weights 6, shapes
    2*(2*(q+1)*q + (q+1)^2) FMA-ish, staging nl multiplies, and the nl^2 FMA
    outer product."""
    nl = disc.local_count()
    q = int(round(nl ** 0.5)) - 1
    jet = 4 * 55 * 2 + 30
    shapes = 2 * (2 * (q + 1) * q * 2 + (q + 1) ** 2)
    return 2 * jet + 12 + 6 + shapes + nl + 2 * nl * nl


def self_launch(args):
    """--gpus N without a torchrun environment: re-run this script as N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--force-dist", action="store_true",
                    help="test aid: run the multi-GPU (NCCL) path even at one rank (under torchrun)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args, c, args.config)
    out = run_b200(args, c, args.config)
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
