#!/usr/bin/env python
"""bench.py — one JSON line for the driver.

Step = one pass of the whole hot path on one batch of synthetic input:
sph_build_cells (binning, radix sort, hierarchy, interaction slots, 13-direction
lists) + sph_density (h iteration to N_ngb = 48, ghost) + sph_force, cold h0 as the
config specifies. Metric = SPH pair interactions per second: 2F per step (F unordered
pairs with r < max(h_i,h_j), once for density and once for force) over
the whole step's device time.

  python bench.py [--gpus N --steps K --warmup W] [--impl sph|reference] [--config C4]

N > 1 runs under torch.distributed.run: one process per GPU, strong scaling of C5
(134,217,728 clustered particles, BASELINE configs[4]) over a slab decomposition (SURVEY
§8(e)); two NCCL halo exchanges per step; the time is the max over ranks, value = all
ranks' pairs / that time.
--impl reference times the fp64 oracle (oracle/) on a bounded sample of the same
workload on this host's CPU cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPH pair interactions/s (density+force), whole step"
UNIT = "pair-interactions/s"
# FLOP per unit: density 27 per unordered pair + 25 per directed
# contribution (first full pass); force 74 per unordered pair.
FLOP_DENS_PAIR, FLOP_DENS_DIR, FLOP_FORCE_PAIR = 27, 25, 74
# neighbour finding: one distance test = 3 sub + 1 mul + 2 FMA = 8 FLOP per recorded entry;
# h iteration (Eq. 3 and its h-derivatives), per list entry per evaluation of N(h): q = r/h 1,
# f, f', f'' of the spline 7 (outer branch; the inner one is 10, credit the smaller), the
# sums S0 += f 1, S1 += q f' 2 (FMA), S2 += q^2 f'' 3 -> 14 FLOP, times the device-counted
# entry evaluations (sph_stats.n_h_evals)
FLOP_TEST, FLOP_HEVAL = 8, 14
# FP32 ALU peak derived from the unit counts and clock (B200_PROFILING.md: 148 SMs,
# clocks.max.sm 1965 MHz; 128 FP32 lanes/SM, FMA = 2 FLOP). Measured: 72.6 TFLOP/s
# (tools/fp32_peak.cu, profiles/round1/fp32_peak.json).
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12

CONFIG_TUNING = dict(split_count=48, split_fraction=0.0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sph", choices=["sph", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--calls", default="step", choices=["step", "three"],
                    help="one step = sph_step (default) or sph_build_cells + sph_density + sph_force")
    ap.add_argument("--no-warm", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ref-budget-s", type=float, default=90.0,
                    help="--impl reference: wall seconds for the warm-up + timed steps together")
    ap.add_argument("--cpu-frac", type=float, default=0.02, help="cpu_baseline: fraction of the particles timed as targets")
    ap.add_argument("--scale-config", default="C5", help="N > 1 workload: C5 (strong scaling) or C4xN (weak)")
    ap.add_argument("--transport", default="torch", choices=["torch", "libsph", "peer"],
                    help="N > 1 halo exchange: torch.distributed P2P, libsph's NCCL communicator, or peer "
                         "stores (the pack kernels write into the neighbours' CUDA IPC buffers)")
    return ap.parse_args()


# --------------------------------------------------------------------- clocks ---
class Clocks:
    """nvidia-smi samples (every 20 ms, with timestamps) of the SM clock and throttle reasons.
    The sampler runs from construction (before the warm-up, so it is up when the timed region
    starts); `region()` brackets the timed steps and only samples inside it (+-25 ms) count;
    a region shorter than the sampling period reports the samples nearest to it."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.t0 = self.t1 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def wait_running(self, busy, limit_s: float = 5.0):
        """Run `busy` (untimed GPU work) until the sampler has written a sample."""
        t = time.time()
        while self.p is not None and time.time() - t < limit_s:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                return
            busy()

    def start(self):
        import datetime
        self.t0 = datetime.datetime.now()

    def end(self):
        import datetime
        self.t1 = datetime.datetime.now()

    def stop(self):
        import datetime
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi missing"]}
        if self.t1 is None:
            self.end()
        time.sleep(0.05)   # the sample after the region
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        samples = []
        for r in rows:
            r = [x.strip() for x in r]
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f")
                samples.append((ts, float(r[1]), float(r[2]), r[5:9]))
            except (ValueError, IndexError):
                continue
        tol = datetime.timedelta(milliseconds=25)
        t0 = self.t0 or self.t1
        inside = [x for x in samples if t0 - tol <= x[0] <= self.t1 + tol]
        if not inside and samples:   # a region shorter than the sampling period
            mid = t0 + (self.t1 - t0) / 2
            inside = sorted(samples, key=lambda x: abs((x[0] - mid).total_seconds()))[:2]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for x in inside:
            for k, nm in enumerate(names):
                if len(x[3]) > k and x[3][k].lower().startswith("active"):
                    reasons.add(nm)
        sm = [x[1] for x in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(x[2] for x in inside) if inside else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- oracle ---
# ---- cpu_baseline: the oracle on a seeded 2% subset of the headline input itself ----------
_G = {}   # inherited by the forked pool workers (x, v, m, box, tree, h and state of all particles)


def _w_density(idx):
    """Pool worker, phase 1: the oracle's own h root (Eq. 3), density (Eq. 2) and particle
    state for a chunk of targets. Returns (idx, h, rho, A, c, f, seconds)."""
    import numpy as np

    import oracle
    import oracle.neighbours as nb
    nb.WORKERS = 1
    g = _G
    t0 = time.perf_counter()
    hT = oracle.solve_h(g["x"], g["box"], targets=idx, tree=g["tree"])
    h = g["h"].copy()
    h[idx] = hT
    den = oracle.density_at(g["x"], g["v"], g["m"], h, g["box"], targets=idx, tree=g["tree"])
    st = oracle.particle_state(den["rho"], den["omega"], g["u"][idx], hT, den["div"], den["curl"])
    return idx, hT, den["rho"], st["A"], st["c"], st["f"], time.perf_counter() - t0


def _w_force(idx):
    """Pool worker, phase 2: the oracle's force (Eq. 4-5 + viscosity) for a chunk of targets.
    Returns (directed force pairs, seconds)."""
    import oracle
    import oracle.neighbours as nb
    nb.WORKERS = 1
    g = _G
    t0 = time.perf_counter()
    fo = oracle.force_at(g["x"], g["v"], g["m"], g["h"], g["rho"], g["A"], g["c"], g["f"], g["box"], targets=idx,
                         tree=g["tree"])
    return int(fo["n_nbr_force"].sum()), time.perf_counter() - t0


def _w_closure(T):
    """Pool worker of the reference arm: the oracle's full evaluation for targets T of the
    workload itself, from nothing but positions, velocities, masses and energies. The targets'
    force sums need h, rho, A, c, f of every force partner j (r < max(h_i, h_j)); a partner
    by its own h has h_j > r, and h_j <= hb[j] (the bound below), so the closure C = T + every
    j within h_i or within hb[j] of a target holds them all: the oracle solves h on C, the
    density and state on the partners, the force on T. Returns (pair interactions: the
    targets' directed force pairs = their share of 2F, the bench metric's count; seconds)."""
    import numpy as np

    import oracle
    import oracle.neighbours as nb
    from scipy.spatial import cKDTree
    nb.WORKERS = 1
    g = _G
    x, box, n = g["x"], g["box"], g["x"].shape[0]
    t0 = time.perf_counter()
    hT = oracle.solve_h(x, box, targets=T, tree=g["tree"])
    _, j1, _, _ = nb.ball_pairs(x, box, x[T], hT, tree=g["tree"])
    j2, _, _, _ = nb.ball_pairs(x[T], box, x, g["hb"], tree=cKDTree(x[T], boxsize=box))
    C = np.union1d(np.union1d(j1, j2), T)
    h = np.zeros(n)
    h[C] = oracle.solve_h(x, box, targets=C, tree=g["tree"])
    _, fj, _, _ = oracle.sph.force_pairs(x, h, box, T, tree=g["tree"])
    S = np.union1d(fj, T)   # within C: a partner outside it has h = 0 and r >= h_i
    den = oracle.density_at(x, g["v"], g["m"], h, box, targets=S, tree=g["tree"])
    st = oracle.particle_state(den["rho"], den["omega"], g["u"][S], h[S], den["div"], den["curl"])
    rho, A, c, f = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(n)
    rho[S], A[S], c[S], f[S] = den["rho"], np.nan_to_num(st["A"]), st["c"], st["f"]
    fo = oracle.force_at(x, g["v"], g["m"], h, rho, A, c, f, box, targets=T, tree=g["tree"])
    work = int(fo["n_nbr_force"].sum())   # the targets' share of 2F (the metric's count)
    if g.get("keep"):   # tests: the targets' results
        g["kept"] = dict(h=h[T], rho=rho[T], a=fo["a"], dudt=fo["dudt"])
    return work, time.perf_counter() - t0


def oracle_closure_setup(p):
    """Untimed setup of the reference arm on the workload itself: the tree and, per particle, an
    upper bound of its h. N(h) >= (32/3)(1 + 0.25 k) with k the other particles within h/2
    (f(q) >= 0.25 for q <= 1/2), so N(h) = 48 allows at most 14 of them: h <= 2 d_15, with d_15
    the distance to the 15th nearest other particle."""
    import numpy as np
    from scipy.spatial import cKDTree

    import oracle.neighbours as nb
    x = p.x.astype(np.float64)
    box = np.asarray(p.box, np.float64)
    tree = cKDTree(x, boxsize=box)
    d, _ = tree.query(x, k=16, workers=-1)
    hb = 2.0 * d[:, 15] * (1.0 + 1e-9)
    _G.clear()
    _G.update(x=x, v=p.v.astype(np.float64), m=p.m.astype(np.float64), u=p.u.astype(np.float64), box=box,
              tree=tree, hb=hb)
    return nb


def oracle_closure_step(p, k, procs, seed):
    """One reference step: k targets of the workload in `procs` compact blobs (the k/procs
    particles nearest to a seeded random particle: blobs sample the particles, and a blob's
    closure adds only a shell of partners), one blob per process."""
    import multiprocessing as mp

    import numpy as np
    rng = np.random.default_rng(seed)
    kb = max(1, k // procs)
    centres = rng.choice(p.n, procs, replace=False)
    _, idx = _G["tree"].query(_G["x"][centres], k=kb, workers=-1)
    chunks = [np.sort(np.asarray(r).reshape(-1)) for r in np.atleast_2d(idx)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(chunks)) as pool:
        res = pool.map(_w_closure, chunks)
    return time.perf_counter() - t0, sum(r[0] for r in res)


def oracle_subset_rate(p, gpu, frac=0.02, procs=None, seed=140423098):
    """Time the fp64 oracle (as it stands, oracle/) on the headline input itself: a seeded
    `frac` subset of its particles as targets, every particle a source. Per target the oracle
    does its full work: h root of Eq. 3, density, particle state, force. Neighbours outside the
    subset take their h and state (rho, A, c, f) from the GPU run's outputs (they are inputs of
    the targets' force sums, not timed work). Targets are split over a process pool (fork, one
    cKDTree thread per process); the rate is directed force pairs of the targets (their share
    of 2F) over the wall time of the two pool phases. Also a 1-process figure on one chunk."""
    import multiprocessing as mp

    import numpy as np
    from scipy.spatial import cKDTree

    import oracle
    procs = procs or cores_used()
    x = p.x.astype(np.float64)
    box = np.asarray(p.box, np.float64)
    st = oracle.particle_state(gpu["rho"], gpu["omega"], p.u, gpu["h"], gpu["div"], gpu["curl"])
    _G.clear()
    _G.update(x=x, v=p.v.astype(np.float64), m=p.m.astype(np.float64), u=p.u.astype(np.float64), box=box,
              tree=cKDTree(x, boxsize=box), h=gpu["h"].astype(np.float64), rho=gpu["rho"].astype(np.float64),
              A=np.nan_to_num(st["A"], posinf=0.0), c=st["c"], f=st["f"])
    rng = np.random.default_rng(seed)
    T = np.sort(rng.choice(p.n, int(frac * p.n), replace=False))
    chunks = np.array_split(T, procs * 2)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_w_density, chunks)
    for idx, hT, rho, A, c, f, _ in res:
        _G["h"][idx], _G["rho"][idx], _G["A"][idx], _G["c"][idx], _G["f"][idx] = hT, rho, np.nan_to_num(A), c, f
    with ctx.Pool(procs) as pool:
        res2 = pool.map(_w_force, chunks)
    wall = time.perf_counter() - t0
    pairs = sum(r[0] for r in res2)
    # one process, one chunk: the single-thread figure
    _, _, _, _, _, _, t1a = _w_density(chunks[0])
    p1, t1b = _w_force(chunks[0])
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": pairs / wall, "unit": UNIT, "cores": procs, "kind": "oracle",
            "sample": (f"{p.name} itself ({p.n} particles, every one a source): seeded {frac:.0%} subset of "
                       f"{T.size} targets (seed {seed}), full oracle work per target (h root + density + state + "
                       f"force, fp64 numpy/scipy), {procs} processes x 1 thread, wall {wall:.1f} s; neighbours' h "
                       f"and state from the GPU outputs (inputs, untimed); rate = the targets' directed force "
                       f"pairs / wall"),
            "one_thread": {"value": p1 / (t1a + t1b), "targets": int(chunks[0].size), "seconds": t1a + t1b},
            "cpu_model": cpu}


def measured_hbm():
    """HBM copy bandwidth (GB/s) from MEASURED_PEAKS.json (driver-written), else the profiling
    guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6550.7, "fallback (B200_PROFILING.md)"


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def arm_config(args, p, world, n_ngb_tol):
    """The `config` object of the bench line: the same for this arm and the reference arm
    (which evaluates a sample of the same workload)."""
    import numpy as np
    cold = not bool(np.any(p.h0 > 0))
    return {"workload": f"{args.config}: {p.n} particles ({p.name} generator, seeds in workloads/), "
                        f"cold h0" + (" (library guess)" if cold else ""),
            "N": p.n, "box": list(p.box), "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": "replicas" if world > 1 else "single GPU",
            "split_count": CONFIG_TUNING["split_count"], "split_fraction": CONFIG_TUNING["split_fraction"],
            "n_ngb": 48, "n_ngb_tol": n_ngb_tol,
            "step_call": "sph_step" if args.calls == "step" else "sph_build_cells + sph_density + sph_force"}


def reference_config(args, p):
    import numpy as np
    return arm_config(args, p, 1, float(np.float32(1e-4)))   # sph_config_default's n_ngb_tol


def run_reference(args, rank, world):
    """The reference arm: the fp64 oracle as it stands on the host cores, on this arm's
    workload itself (args.config, every particle a source); each step the full oracle work
    for a seeded sample of targets (oracle_closure_step). The sample size is calibrated so
    that a step takes about cpu_budget_s / (steps + warmup) of wall time."""
    if rank != 0:
        return
    import workloads
    p = workloads.make(args.config)
    oracle_closure_setup(p)
    procs = cores_used()
    budget = args.ref_budget_s / max(1, args.steps + args.warmup)
    # t(k) = a + b k: each process's queries over all particles (partners reaching in by
    # their own h) are a fixed cost per step; two calibration steps fit a and b
    k0, k1 = 1024 * procs, 4096 * procs
    t0_, _ = oracle_closure_step(p, k0, procs, seed=140423100)
    t1_, _ = oracle_closure_step(p, k1, procs, seed=140423100)
    b = max((t1_ - t0_) / (k1 - k0), 1e-9)
    a = max(t0_ - b * k0, 0.0)
    k = int(min(max(k0, (budget - a) / b), p.n // 4))
    for w in range(args.warmup):
        oracle_closure_step(p, k, procs, seed=140423101 + w)
    ts, ws = [], []
    for s_ in range(args.steps):
        t, wk = oracle_closure_step(p, k, procs, seed=140423200 + s_)
        ts.append(t)
        ws.append(wk)
    T = sum(ts)
    value = sum(ws) / T
    sample = (f"{p.name} itself ({p.n} particles, every one a source): per step {k} targets in {procs} compact "
              f"blobs (the particles nearest to seeded random particles); the oracle solves h on the blobs' "
              f"closure (every possible force partner: within max(h_i, h_j), h_j bounded by twice the 15th-"
              f"neighbour distance), the density and state of the partners and the targets' force, fp64 "
              f"numpy/scipy, {procs} processes x 1 thread; value = the targets' directed force pairs (their "
              f"share of 2F) / wall")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": reference_config(args, p),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours -----
def traffic_from_profiles(kernel: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel)
    except (OSError, ValueError):
        return None


ISSUE_PEAK_GINST = 148 * 4 * 1.965   # warp-instructions per ns: 148 SMs x 4 schedulers x 1/clock


def issue_from_profiles(kernel: str, ms: float):
    """Issue-rate utilisation: the kernel's executed warp instructions (ncu, profiles/issue.json)
    over its live launch time, against one warp-instruction per scheduler per clock."""
    try:
        inst = json.load(open(os.path.join(ROOT, "profiles", "issue.json"))).get(kernel)
    except (OSError, ValueError):
        return None
    if not inst or ms <= 0:
        return None
    ach = inst / (ms * 1e6)
    return {"warp_inst_per_launch": inst, "achieved_ginst_s": ach, "peak_ginst_s": ISSUE_PEAK_GINST,
            "frac": ach / ISSUE_PEAK_GINST, "source": "profiles/issue.json (ncu executed instructions, round-2 final code)"}


def run_sph(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1404_2303_b200 as sph
    import workloads

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = world > 1
    if dist:
        import torch.distributed as td
    p = workloads.make(args.config)
    N = p.n
    stream = torch.cuda.current_stream(dev)
    cfg = sph.default_config(p.box, **CONFIG_TUNING)
    ctx = sph.Context(cfg, device=local_rank, stream=stream.cuda_stream)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
    h0 = t(p.h0) if np.any(p.h0 > 0) else None
    out_d = dict(h=torch.empty(N, device=dev), rho=torch.empty(N, device=dev))
    out_f = dict(a=torch.empty(N, 3, device=dev), dudt=torch.empty(N, device=dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(xx, hh, vv, mm, uu, od, of):
        if args.calls == "step":   # the whole-step call (sph_step): no host round trips between phases
            d, f = ctx.step(xx, vv, mm, uu, hh, out=dict(h=od["h"], rho=od["rho"], a=of["a"], dudt=of["dudt"]))
            return d.stats, f.stats
        ctx.build_cells(xx, hh)
        d = ctx.density(vv, mm, uu, out=od)
        f = ctx.force(vv, out=of)
        return d.stats, f.stats

    for _ in range(args.warmup):
        step(x, h0, v, m, u, out_d, out_f)
    torch.cuda.synchronize()

    def step_e2e(xx, hh, vv, mm, uu, od, of):
        # the whole step in one public call (sph_step): host copies overlapped with the work
        d, f = ctx.step(xx, vv, mm, uu, hh, out=dict(h=od["h"], rho=od["rho"], a=of["a"], dudt=of["dudt"]))
        return d.stats, f.stats

    def timed(inputs, outs_d, outs_f, stepf=step):
        stats = []
        total_ms = 0.0
        if dist:
            td.barrier()
        torch.cuda.synchronize()
        clk = Clocks(local_rank)
        clk.wait_running(lambda: stepf(*inputs, outs_d, outs_f))   # untimed steps until sampling
        torch.cuda.synchronize()
        l0 = ctx.kernel_launches
        clk.start()
        for _ in range(args.steps):
            flush.zero_()                       # evict the inputs from L2 between steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sd, sf = stepf(*inputs, outs_d, outs_f)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            stats.append((sd, sf))
        clk.end()
        clocks = clk.stop()
        torch.cuda.synchronize()
        if dist:
            td.barrier()
        return total_ms, stats, ctx.kernel_launches - l0, clocks

    total_ms, stats, launches, clocks = timed((x, h0, v, m, u), out_d, out_f)
    F = stats[-1][1]["n_pairs"]
    D = stats[-1][0]["n_directed"]
    # e2e: the same steps through the C ABI's whole-step call (sph_step) with pinned HOST buffers
    # (copies inside the region, overlapped with the work where the step allows)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hx, hv, hm, hu = pin(p.x), pin(p.v), pin(p.m), pin(p.u)
        hh0 = pin(p.h0) if h0 is not None else None
        hod = dict(h=torch.empty(N).pin_memory(), rho=torch.empty(N).pin_memory())
        hof = dict(a=torch.empty(N, 3).pin_memory(), dudt=torch.empty(N).pin_memory())
        for _ in range(max(1, args.warmup)):   # host-staging buffers are allocated on first use
            step_e2e(hx, hh0, hv, hm, hu, hod, hof)
        e2e_ms, e2e_stats, _, _ = timed((hx, hh0, hv, hm, hu), hod, hof, stepf=step_e2e)
        h2d = sum(a.numel() * 4 for a in (hx, hv, hm, hu)) + (hh0.numel() * 4 if hh0 is not None else 0)
        d2h = sum(a.numel() * 4 for a in (*hod.values(), *hof.values()))
        e2e = {"t_ms": e2e_ms, "pairs": 2.0 * sum(s[1]["n_pairs"] for s in e2e_stats),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        # the host path must reproduce the device path bit for bit
        assert torch.equal(hod["rho"], out_d["rho"].cpu()) and torch.equal(hof["a"], out_f["a"].cpu())

    # warm start: h0 = converged h x (1 + 0.05 U(-1,1)), seeded; the regime of a
    # time-step loop that carries h between steps. Reported beside the cold headline.
    warm = None
    if not args.no_warm:
        rng = np.random.default_rng(140423099)
        hw = out_d["h"].cpu().numpy() * (1.0 + 0.05 * rng.uniform(-1.0, 1.0, N)).astype(np.float32)
        hw_d = t(hw.astype(np.float32))
        for _ in range(2):
            step(x, hw_d, v, m, u, out_d, out_f)
        warm_ms, wstats, _, _ = timed((x, hw_d, v, m, u), out_d, out_f)
        warm = {"ms_per_step": warm_ms / args.steps, "value": 2.0 * wstats[-1][1]["n_pairs"] * args.steps / (warm_ms * 1e-3),
                "h0": "converged h x (1 + 0.05 U(-1,1)), seed 140423099",
                "regrow_particles": wstats[-1][0]["n_rebuilds"], "h_iters": wstats[-1][0]["h_iters"]}
    pairs_local = 2.0 * sum(s[1]["n_pairs"] for s in stats)
    t_max = total_ms
    pairs_all = pairs_local
    e2e_tmax = e2e["t_ms"] if e2e else None
    e2e_pairs = e2e["pairs"] if e2e else None
    if dist:
        tt = torch.tensor([total_ms, e2e_tmax or 0.0], dtype=torch.float64, device=dev)
        td.all_reduce(tt, op=td.ReduceOp.MAX)
        pp = torch.tensor([pairs_local, e2e_pairs or 0.0], dtype=torch.float64, device=dev)
        td.all_reduce(pp)
        t_max, e2e_tmax = float(tt[0]), float(tt[1])
        pairs_all, e2e_pairs = float(pp[0]), float(pp[1])
    if rank != 0:
        ctx.close()
        return

    sd = [s[0] for s in stats]
    sfo = [s[1] for s in stats]
    med = lambda key, arr: statistics.median(a[key] for a in arr)
    k_force_ms = med("ms_kernel_force", sfo)
    k_dens_ms = med("ms_kernel_density_full", sd)
    flop_force = FLOP_FORCE_PAIR * F
    flop_dens = FLOP_DENS_PAIR * F + FLOP_DENS_DIR * D
    ms_density = med("ms_density", sd)
    ms_force = med("ms_force", sfo)
    ms_build = med("ms_build", sd)

    def roof(name, flop, ms, what):
        ach = flop / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        return {"kernel": name, "bound": "alu", "achieved": ach, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP32_PEAK_TFLOPS, "traffic": traffic_from_profiles(name),
                "flop_per_step": flop, "ms_per_step": ms, "work": what, "issue": issue_from_profiles(name, ms),
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (measured FFMA 72.6)"}

    # per-phase kernel time, CUDA events on the ctx stream around every launch of the phase
    # (summed over the phase's launches within one step)
    nb_entries = med("n_nb_entries", sd)
    h_evals = med("n_h_evals", sd)
    # the h iteration runs fused in the NB walk's epilogue; stand-alone solves (pool lists,
    # repeated calls) add k_hsolve time, so the phase is credited over both kernels' time
    ms_nb = med("ms_kernel_walk_nb", sd) + med("ms_kernel_hsolve", sd)
    kern = {
        "k_walk (neighbour lists + h solve)": roof("k_walk<MODE_NB>", FLOP_TEST * nb_entries + FLOP_HEVAL * h_evals,
                                                   ms_nb,
                                                   f"{FLOP_TEST} FLOP per recorded neighbour entry (r^2 < h_build^2), "
                                                   f"{int(nb_entries)} entries, + {FLOP_HEVAL} FLOP per entry "
                                                   f"evaluation of the h iteration (fused in the walk's epilogue), "
                                                   f"{int(h_evals)} evaluations "
                                                   f"({h_evals / max(nb_entries, 1):.2f} per entry)"),
        "k_force": roof("k_force", flop_force, k_force_ms, f"{FLOP_FORCE_PAIR} FLOP x F"),
        "k_density": roof("k_density", flop_dens, k_dens_ms, f"{FLOP_DENS_PAIR} FLOP x F + {FLOP_DENS_DIR} x D"),
        "k_walk (interaction lists)": roof("k_walk<MODE_FILL>", FLOP_TEST * sfo[-1]["n_pair_slots"],
                                           med("ms_kernel_walk_union", sd),
                                           f"{FLOP_TEST} FLOP per interaction-list entry"),
    }
    order = sorted(kern.values(), key=lambda r: -r["ms_per_step"])
    dominant, secondary = order[0], order[1:]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # every output of one more (untimed) evaluation: the neighbours' state for the oracle
        d = ctx.density(v, m, u)
        gpu = {k: getattr(d, k).cpu().numpy().astype(np.float64) for k in ("h", "rho", "omega", "div", "curl")}
        cpu = oracle_subset_rate(p, gpu, frac=args.cpu_frac)
    # a1-a3 (binning + sort + permute) against HBM: SURVEY 8(d)'s algorithmic bytes per particle,
    # (28 + 24 x passes + 8 + 80), over the CUDA-event time of those kernels in the step
    passes = sd[-1]["sort_passes"]
    bpp = 28 + 24 * passes + 8 + 80
    ms_sort = med("ms_kernel_sort", sd)
    hbm = measured_hbm()
    ach_bin = N * bpp / (ms_sort * 1e-3) / 1e9 if ms_sort > 0 else 0.0
    roof_bin = {"kernels": "k_keys + k_radix_pass x passes + k_pack + k_validate_pack_vmu + k_gather_vmu",
                "bound": "hbm", "achieved": ach_bin, "peak": hbm[0], "unit": "GB/s", "frac": ach_bin / hbm[0],
                "traffic": None, "bytes_per_particle": bpp, "sort_passes": passes,
                "sort_key_bits": sd[-1]["sort_key_bits"], "ms_per_step": ms_sort, "peak_source": hbm[1],
                "note": ("C4's 2.1M-particle arrays are L2-resident per pass (126 MB L2), so this is not an HBM "
                         "measurement; the shard-size run is tools/binning_run.py (profiles/round2/binning_16M.md)")}
    value = pairs_all / (t_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": arm_config(args, p, world, cfg.n_ngb_tol),
        "roofline": dominant,
        "roofline_others": secondary,
        "roofline_binning": roof_bin,
        "cpu_baseline": cpu,
        "e2e": ({"value": e2e_pairs / (e2e_tmax * 1e-3), "unit": UNIT,
                 "h2d_bytes_per_step": e2e["h2d_bytes_per_step"], "d2h_bytes_per_step": e2e["d2h_bytes_per_step"]}
                if e2e else None),
        "gpu_launches": launches,
        "clocks": clocks,
        "breakdown": {"F_pairs": F, "D_directed": D, "ms_build": ms_build, "ms_density": ms_density,
                      "ms_force": ms_force, "ms_kernel_density_full": k_dens_ms, "ms_kernel_force": k_force_ms,
                      "rate_loops_2F_over_tdens_plus_tforce": 2.0 * F / ((ms_density + ms_force) * 1e-3),
                      "ms_kernel_walk_nb": med("ms_kernel_walk_nb", sd), "ms_kernel_hsolve": med("ms_kernel_hsolve", sd),
                      "ms_kernel_walk_union": med("ms_kernel_walk_union", sd), "nb_entries": nb_entries,
                      "walk_launches": sd[-1]["n_walk_launches"],
                      "h_iters": sd[-1]["h_iters"], "regrow_particles": sd[-1]["n_rebuilds"],
                      "warm_start": warm,
                      "cand_density_full": sd[-1]["n_candidates_density_full"],
                      "cand_force": sfo[-1]["n_candidates"], "levels": sd[-1]["n_levels"],
                      "cells": sd[-1]["n_cells"]},
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def run_slab(args, rank, world, local_rank):
    """N > 1: strong scaling on BASELINE configs[4] (north_star: "measured at 1, 2, 4 and 8
    GPUs on the 134M-particle case"): C5, 134,217,728 clustered particles (512 clumps), split
    into N count-quantile slabs along x; each rank exchanges halos with its two neighbours over
    NCCL before the density and before the force loop (paper_1404_2303_b200/slab.py; the send
    rows packed by libsph's k_halo_pack). --scale-config C4xN selects the former weak-scaling
    workload (the C4 recipe in an (N,1,1) box)."""
    import numpy as np
    import torch
    import torch.distributed as td

    import paper_1404_2303_b200 as sph
    import workloads
    from paper_1404_2303_b200 import slab

    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    p = workloads.c4_weak(world) if args.scale_config == "C4xN" else workloads.make(args.scale_config)
    strong = args.scale_config != "C4xN"
    Lx = p.box[0]
    cfg0 = sph.default_config(p.box, **CONFIG_TUNING)
    ctx0 = sph.Context(cfg0, device=local_rank, stream=stream.cuda_stream)
    # count-quantile cuts from the global x histogram (each rank histograms its initial slab)
    own0 = np.nonzero((p.x[:, 0] >= rank * Lx / world) & (p.x[:, 0] < (rank + 1) * Lx / world))[0]
    hist = ctx0.x_histogram(torch.from_numpy(np.ascontiguousarray(p.x[own0])).to(dev), 0.0, Lx, 8192)
    td.all_reduce(hist)
    edges = slab.slab_cuts(hist.cpu().numpy(), 0.0, Lx, world)
    lo, hi = edges[rank], edges[rank + 1]
    own = np.nonzero((p.x[:, 0] >= lo) & (p.x[:, 0] < hi))[0]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    x, v, m, u, h0 = t(p.x[own]), t(p.v[own]), t(p.m[own]), t(p.u[own]), t(p.h0[own])
    # halo width: twice the largest occupancy guess of h anywhere (allreduce), <= slab width
    gmax = torch.tensor([float(ctx0.guess_h(x).max())], dtype=torch.float64, device=dev)
    td.all_reduce(gmax, op=td.ReduceOp.MAX)
    wmin = torch.tensor([min(e1 - e0 for e0, e1 in zip(edges, edges[1:]))], dtype=torch.float64, device=dev)
    width = float(min(2.0 * gmax.item(), wmin.item()))
    ctx0.close()
    cfg = sph.default_config(p.box, **CONFIG_TUNING, rank=rank, nranks=world, slab_lo=lo, slab_hi=hi,
                             halo_width=width)
    ctx = sph.Context(cfg, device=local_rank, stream=stream.cuda_stream)
    # halo transport: torch.distributed P2P (NCCL) or libsph's own NCCL communicator
    if args.transport == "peer":
        tr = slab.PeerTransport(ctx, rank, world, cap_rows=len(own))
    else:
        tr = slab.LibTransport(ctx, rank, world) if args.transport == "libsph" else slab.DistTransport(rank, world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(inputs):
        if args.transport == "peer":
            return slab.evaluate_rank_peer(ctx, *inputs, lo, hi, width, tr)
        return slab.evaluate_rank(ctx, *inputs, lo, hi, width, tr)

    for _ in range(args.warmup):
        step((x, v, m, u, h0))
    torch.cuda.synchronize()

    def timed(make_inputs, fetch):
        total, res = 0.0, None
        td.barrier()
        torch.cuda.synchronize()
        l0 = ctx.kernel_launches
        clk = Clocks(local_rank)   # (every rank runs the same steps: no per-rank warm-up here)
        clk.start()
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = step(make_inputs())
            fetch(res)
            e1.record(stream)
            e1.synchronize()
            total += e0.elapsed_time(e1)
        clk.end()
        clocks = clk.stop()
        torch.cuda.synchronize()
        td.barrier()
        return total, res, ctx.kernel_launches - l0, clocks

    total_ms, res, launches, clocks = timed(lambda: (x, v, m, u, h0), lambda r: None)
    pairs = 2.0 * res.stats_force["n_pairs"] * args.steps
    # e2e: owned inputs from pinned host memory, outputs back to the host, inside the region
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hx, hv, hm, hu, hh0 = pin(p.x[own]), pin(p.v[own]), pin(p.m[own]), pin(p.u[own]), pin(p.h0[own])
    outs = [torch.empty(len(own)).pin_memory(), torch.empty(len(own)).pin_memory(),
            torch.empty(len(own), 3).pin_memory(), torch.empty(len(own)).pin_memory()]

    def fetch(r):
        for o, s_ in zip(outs, (r.h, r.rho, r.a, r.dudt)):
            o.copy_(s_, non_blocking=True)

    e2e_ms, _, _, _ = timed(lambda: tuple(a.to(dev, non_blocking=True) for a in (hx, hv, hm, hu, hh0)), fetch)
    h2d = sum(a.numel() * 4 for a in (hx, hv, hm, hu, hh0))
    d2h = sum(o.numel() * 4 for o in outs)
    agg = torch.tensor([total_ms, e2e_ms, pairs, float(res.n_halo), float(len(own))], dtype=torch.float64, device=dev)
    mx = agg.clone()
    td.all_reduce(mx, op=td.ReduceOp.MAX)
    sm = agg.clone()
    td.all_reduce(sm)
    if rank == 0:
        t_max, e2e_max = float(mx[0]), float(mx[1])
        line = {
            "metric": METRIC, "value": float(sm[2]) / (t_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"{p.name}: {p.n} particles ({p.meta.get('n_clumps')} clumps), "
                                    f"{world} count-quantile slabs along x, cold h0"),
                       "N": p.n, "parallelism": f"slab{world} (halo exchange over NCCL, 2 per step)",
                       "halo_width": width, "halo_over_owned_mean": float(sm[3]) / float(sm[4]),
                       "l2": "flushed (256 MiB write) before every timed step",
                       "split_count": CONFIG_TUNING["split_count"]},
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": float(sm[2]) / (e2e_max * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local_rank)
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if world > 1:
            run_slab(args, rank, world, local_rank)
        else:
            run_sph(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as td
            td.destroy_process_group()


if __name__ == "__main__":
    main()
