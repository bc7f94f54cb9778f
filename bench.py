"""Benchmark: solver iterations/s and GUPS of A / A^T on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 3 -- the north-star size, 3-D Shepp-Logan 512^3,
720 views of a 616x480 detector, CGLS (SURVEY.md 8(d) geometry rule: SID 749, SDD 1198,
0.43 mm voxels, 0.616 mm pixels).  A "step" is one steady-state solver loop iteration; for
CGLS (solvers.py:339-357): A^T (+||r||^2), fused volume update, A (+||p||^2), fused
projection update (+||e||^2).  ``--config 4`` (or ``--solver lsqr-jacobi``) times LSQR with
Jacobi preconditioning, ``--solver psirt`` PSIRT; ``--precision f64`` the reference-precision
path.  Inputs stay resident in HBM; the working set (0.55 GB volume + 3 x 0.85 GB projection
vectors at config 3) exceeds the 126 MB L2, so no explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--solver S]
                    [--precision f32|f64] [--impl ours|reference]

Prints ONE JSON line on rank 0.  ``--impl reference`` times the reference
algorithm's CPU restatement (oracle/, C + OpenMP, all host threads) on bounded
view samples of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json configs: (N, views, nu, nv, solver, K)
CONFIGS = {
    1: (64, 90, 128, 96, "cgls", 10),
    2: (256, 360, 512, 384, "cgls", 40),
    3: (512, 720, 616, 480, "cgls", 40),
    4: (512, 720, 616, 480, "lsqr-jacobi", 40),
    5: (1024, 1440, 1024, 768, "cgls", 10),
}
# nnz(A) per config, SURVEY.md 8(d) (exact for 1-2, sampled for 3-5); the
# algorithmic unit of the A / A^T roofline.
NNZ = {1: 8.50e7, 2: 2.176e10, 3: 1.312e11, 4: 1.312e11, 5: 1.36e12}
SLOTS_PER_NNZ = 8  # FP32-lane-slot equivalents per nonzero
SMS = 148
LANES = 128


def geometry(cfg: int):
    from paper_2110_13526_b200.geometry import DetectorGeometry, VolumeGeometry, make_circular_trajectory

    N, V, nu, nv, _, _ = CONFIGS[cfg]
    p = 220.16 / N
    vg = VolumeGeometry(N, N, N, (p, p, p))
    pu = 379.456 / nu
    tr = make_circular_trajectory(749.0, 1198.0, V, 0.0, 2 * np.pi, DetectorGeometry(nu, nv, (pu, pu)))
    return vg, tr


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)
        return False

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def committed_traffic(cfg: int) -> dict:
    """DRAM bytes per operator application of the hot kernels from the committed ncu captures of
    this build (profiles/traffic_r2.json; round-1 file as a fallback)."""
    for name in ("traffic_r2.json", "traffic_r1.json"):
        try:
            with open(ROOT / "profiles" / name) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if f"config{cfg}" in d:
            return dict(d[f"config{cfg}"], source=d.get("source"))
    return {}


# ------------------------------------------------------------------ CPU legs --
def _oracle_ops(cfg, k, threads):
    from oracle import oracle as O
    from paper_2110_13526_b200.geometry import make_circular_trajectory

    vg, tr = geometry(cfg)
    sub = make_circular_trajectory(tr.sid, tr.sdd, k, 0.0, k * tr.angular_span / tr.n_views, tr.detector)
    return O, vg, tr, sub


def cpu_time_views(cfg: int, k: int, workers: int, threads: int = 0):
    """One A and one A^T of the reference algorithm (oracle port, C + OpenMP, fp64) on the first
    k views of the workload; returns (t_A, t_AT) in seconds."""
    O, vg, tr, sub = _oracle_ops(cfg, k, threads)
    op = O.OracleOperator(vg, sub, workers=workers, threads=threads)
    x = np.random.default_rng(0).random(op.n)
    y = np.random.default_rng(1).standard_normal(op.m)
    t0 = time.perf_counter()
    op.project(x)
    ta = time.perf_counter() - t0
    t0 = time.perf_counter()
    op.backproject(y)
    tat = time.perf_counter() - t0
    return ta, tat


def cpu_vector_time(cfg: int):
    """Vector work of one CGLS iteration in fp64 numpy (solvers.py:340-355), full size."""
    vg, tr = geometry(cfg)
    n, m = vg.nx * vg.ny * vg.nz, tr.n_rays
    xv, dv, rv = np.zeros(n), np.ones(n), np.ones(n)
    t0 = time.perf_counter()
    _ = float(rv @ rv)
    dv *= 0.5
    dv += rv
    xv += 0.1 * dv
    tv_n = time.perf_counter() - t0
    del xv, dv, rv
    ev, pv = np.ones(m), np.ones(m)
    t0 = time.perf_counter()
    _ = float(pv @ pv)
    ev -= 0.1 * pv
    _ = float(np.linalg.norm(ev))
    tv_m = time.perf_counter() - t0
    return tv_n + tv_m


def cpu_views(cfg: int, threads: int) -> int:
    """Sample size: enough views that the worker-parallel backprojector uses every host thread
    (its parallelism is min(workers, threads), operator.py:219) and that the k -> 2k difference
    (32+ views of traversal) stands clear of the run-to-run noise of A^T's fixed cost."""
    V = CONFIGS[cfg][1]
    return max(1, min(V // 2, max(threads, 32)))


def cpu_workers(cfg: int, threads: int, k: int) -> int:
    """Backprojector workers as the reference deals them (operator.py:219-220): all threads, capped
    so the W private fp64 accumulators stay within 64 GB of host memory."""
    N = CONFIGS[cfg][0]
    return max(1, min(threads, k, int(64e9 // (8 * N ** 3))))


def cpu_extrapolate(cfg: int, k: int, t1, t2):
    """Time of one full-trajectory A and A^T from samples at k and 2k views with the same worker
    count: t(v) = F + v s  ->  full = F + V s, so the fixed cost F is counted once.  A^T's F is
    the W private accumulators' allocation, first-touch page faults and serial merge
    (operator.py:222-233); A has none.  t1 / t2: (t_A, t_AT) medians at k and 2k views."""
    V = CONFIGS[cfg][1]
    out = {}
    for name, a, b in (("t_A", t1[0], t2[0]), ("t_AT", t1[1], t2[1])):
        slope = (b - a) / k
        if slope <= 0.0:  # noise swamped the difference: scale the 2k sample proportionally
            slope, fixed = b / (2 * k), 0.0
        else:
            fixed = max(a - k * slope, 0.0)
        out[name] = fixed + V * slope
        out[name + "_fixed"] = fixed
    return out


def cpu_sample(cfg: int, threads: int = 0):
    """CPU time of one CGLS iteration of the reference algorithm (one A + one A^T + the vector
    updates) on this host, extrapolated from view samples at k and 2k views."""
    from oracle import oracle as O

    threads = int(O.lib().oracle_max_threads()) if threads < 1 else threads
    V = CONFIGS[cfg][1]
    k = cpu_views(cfg, threads)
    workers = cpu_workers(cfg, threads, k)
    t1 = cpu_time_views(cfg, k, workers, threads)
    if 2 * k <= V:
        t2 = cpu_time_views(cfg, 2 * k, workers, threads)
        ex = cpu_extrapolate(cfg, k, t1, t2)
        how = (f"A and A^T timed on {k} and {2 * k} of {V} views (t_A {t1[0]:.2f}/{t2[0]:.2f} s, "
               f"t_AT {t1[1]:.2f}/{t2[1]:.2f} s); full = fixed cost + {V} x per-view slope")
    else:
        ex = {"t_A": t1[0] * V / k, "t_AT": t1[1] * V / k, "t_A_fixed": 0.0, "t_AT_fixed": 0.0}
        how = f"A and A^T on all {V} views"
    tv = cpu_vector_time(cfg)
    return {**ex, "t_vec": tv, "t_iter": ex["t_A"] + ex["t_AT"] + tv, "views_sampled": k, "workers": workers,
            "threads": threads, "sample": how + f"; workers {workers}; vector updates at full size (numpy fp64)",
            "extrapolated": k < V}


def run_reference(args, cfg, rank, world):
    """The reference arm: the reference algorithm's CPU implementation (oracle port, all host
    threads) on rank 0.  One step = one A + one A^T on a k-view sample of the workload; after the
    K timed steps one 2k-view sample gives the per-view slope, and the CGLS iteration time is
    extrapolated to all views (cpu_extrapolate)."""
    if rank != 0:
        return 0
    from oracle import oracle as O

    threads = int(O.lib().oracle_max_threads())
    N, V, nu, nv, solver, K = CONFIGS[cfg]
    k = cpu_views(cfg, threads)
    workers = cpu_workers(cfg, threads, k)
    # warm-up: page in the oracle and the tables on a one-view sample; the timed samples are capped at 6
    # (each is ~11 s at config 3) so the reference arm ends within a few minutes
    for _ in range(args.warmup):
        cpu_time_views(cfg, 1, 1)
    n_samples = max(1, min(args.steps, 6))
    samples = [cpu_time_views(cfg, k, workers) for _ in range(n_samples)]
    t1 = (float(np.median([s[0] for s in samples])), float(np.median([s[1] for s in samples])))
    if 2 * k <= V:
        s2 = [cpu_time_views(cfg, 2 * k, workers) for _ in range(2)]
        t2 = (float(np.median([s[0] for s in s2])), float(np.median([s[1] for s in s2])))
        ex = cpu_extrapolate(cfg, k, t1, t2)
    else:
        t2 = None
        ex = {"t_A": t1[0] * V / k, "t_AT": t1[1] * V / k, "t_A_fixed": 0.0, "t_AT_fixed": 0.0}
    t_iter = ex["t_A"] + ex["t_AT"] + cpu_vector_time(cfg)
    val = 1.0 / t_iter
    sample = (f"A and A^T of the reference algorithm on {k} of {V} views (median of {n_samples} samples: t_A "
              f"{t1[0]:.2f} s, t_AT {t1[1]:.2f} s) and on {2 * k} views (median of 2"
              + (f": t_A {t2[0]:.2f} s, t_AT {t2[1]:.2f} s" if t2 else "") + f"); iteration (one A + one A^T + the vector updates, as every solver's step) = fixed cost + {V} x "
              f"per-view slope; workers {workers}, {threads} OpenMP threads; vector updates at full size (numpy fp64)")
    solver = args.solver or CONFIGS[cfg][4]
    sname = SOLVER_NAME[solver]
    line = {
        "impl": "reference", "metric": f"{sname} iterations/sec", "value": val, "unit": "it/s", "n_gpus": world,
        "steps": n_samples, "warmup": args.warmup, "ms_per_step": t_iter * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{cfg}: Shepp-Logan {N}^3, {V} views of {nu}x{nv}, {sname} step",
                   "solver": solver, "precision": "f64", "parallelism": "cpu-openmp"},
        "gups_A": N ** 3 * V / ex["t_A"] / 1e9, "gups_AT": N ** 3 * V / ex["t_AT"] / 1e9,
        "t_A_s": ex["t_A"], "t_AT_s": ex["t_AT"], "t_AT_fixed_s": ex["t_AT_fixed"],
        # each timed step is a k-view sample (A + A^T), not a full iteration: ms_per_step is the extrapolated
        # full-iteration time, sample_s the measured per-step wall time
        "extrapolated": True, "sample_s": t1[0] + t1[1], "sample_views": k,
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": threads, "kind": "port", "sample": sample,
                         "extrapolated": True},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg --
SOLVER_METHOD = {"cgls": ("cgls", {}), "lsqr-jacobi": ("lsqr", {"jacobi_precondition": True}), "psirt": ("psirt", {})}
SOLVER_NAME = {"cgls": "CGLS", "lsqr-jacobi": "LSQR+Jacobi", "psirt": "PSIRT"}


def _new_run(P, op, b, solver, iters):
    from paper_2110_13526_b200.solvers import ClassicalRun, CglsRun, LsqrRun, SolverConfig

    method, kw = SOLVER_METHOD[solver]
    cfg = SolverConfig(method=method, max_iterations=iters, **kw)
    if method == "cgls":
        return CglsRun(op, b, cfg)
    if method == "lsqr":
        return LsqrRun(op, b, cfg)
    return ClassicalRun(op, b, cfg, method)


def run_ours(args, cfg, rank, world, local_rank):
    """N = 1: one steady-state solver iteration per step (N > 1 goes through run_sharded)."""
    import torch

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import _lib
    from paper_2110_13526_b200.solvers import SolverConfig

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    N, V, nu, nv, _, K = CONFIGS[cfg]
    solver = args.solver or CONFIGS[cfg][4]
    sname = SOLVER_NAME[solver]
    vg, tr = geometry(cfg)
    t_setup = time.perf_counter()
    op = P.CbctOperator(vg, tr, device=dev, precision=args.precision)
    x_int = op.phantom_internal(P.shepp_logan_3d())  # device voxelizer (bit-identical to generate_phantom)
    b_int = op.new_projections()
    op.project_internal(x_int, b_int)  # inverse crime b = A phantom (device)
    del x_int
    b = P.operator.InternalProjections(tr, b_int)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    steps, warmup = args.steps, args.warmup
    stream = torch.cuda.current_stream(dev)
    run = _new_run(P, op, b, solver, steps + warmup + 1)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    device_loop = hasattr(run, "run_device") and run.device_capable()
    if device_loop:
        # CGLS and LSQR run device-resident (scalars and stop tests on the GPU, no host round trip per
        # iteration) as replays of one captured CUDA graph of the iteration (solvers.*Run.run_device)
        done0 = run.updates if solver == "lsqr-jacobi" else run.i
        run.run_device(warmup, graph=True)  # warm-up (captures the graph on its first call)
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk:
            start.record(stream)
            run.run_device(steps, graph=True, collect=False)
            end.record(stream)
            torch.cuda.synchronize()
        run.collect()
        done1 = run.updates if solver == "lsqr-jacobi" else run.i
        assert done1 - done0 == warmup + steps, "the timed loop must run exactly K iterations"
        launches = steps * run.graph_launches  # libcbct kernels per replayed iteration x replays
        loop = f"device-resident {sname}, CUDA-graph replay per iteration"
    else:
        # host-driven loop (the reference's scalar recurrences on the host, fp64): each step is one
        # full iteration including its blocking norm reads
        for _ in range(warmup):
            run.step()
        torch.cuda.synchronize()
        n0 = _lib.lib().cbct_launch_count()
        with ClockSampler(local_rank) as clk:
            start.record(stream)
            for _ in range(steps):
                run.step()
            end.record(stream)
            torch.cuda.synchronize()
        launches = _lib.lib().cbct_launch_count() - n0
        loop = f"host-driven {sname} loop ({args.precision})"
    ms = start.elapsed_time(end)
    # kernel-only durations: CUDA events tight around the launches on this stream
    scratch = op.new_bp_scratch()
    vol_a, proj_a = op.new_volume(), op.new_projections()
    vol_a.copy_(run.x if hasattr(run, "x") else vol_a)
    proj_a.copy_(b_int)

    def kernel_ms(fn, reps=5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        s.record(stream)
        for _ in range(reps):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    reps = 5 if args.precision == "f32" else 2
    out_p, out_v = op.new_projections(), op.new_volume()
    t_a = kernel_ms(lambda: op.project_internal(vol_a, out_p), reps)
    t_at = kernel_ms(lambda: op.backproject_internal(proj_a, out_v, scratch=scratch), reps)
    del out_p, out_v, vol_a, proj_a
    ms_step = ms / steps
    value = 1e3 / ms_step
    e_last = run.history[-1].rel_discrepancy if run.history else None
    del run
    torch.cuda.empty_cache()

    # end to end through the public API: host fp64 b in, host x out, the full solve (setup included)
    b_host = op.proj_from_internal(b_int, torch.float64).cpu().numpy()
    e2e_k = max(steps, 5)
    bstack = P.ProjectionStack(tr, b_host)
    method, kw = SOLVER_METHOD[solver]
    scfg = SolverConfig(method=method, max_iterations=e2e_k, **kw)
    t_solves = []
    n_solves = 3 if args.precision == "f32" else 1
    P.solve(op, bstack, scfg)  # untimed: the pinned staging buffers and copy threads are created on first use
    for _ in range(n_solves):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve(op, bstack, scfg)
        torch.cuda.synchronize()
        t_solves.append(time.perf_counter() - t0)
    t_e2e = float(np.median(t_solves))
    e2e = {"value": rep.iterations / t_e2e, "unit": "it/s",
           "h2d_bytes_per_step": int(op.m * 4 / e2e_k), "d2h_bytes_per_step": int((op.n * 8 + 24 * e2e_k) / e2e_k),
           "note": f"{method}() on a host fp64 ProjectionStack, K={e2e_k}, including its setup "
                   f"({'pre-loop 2 A + 1 A^T' if method == 'cgls' else 'normal_diagonal + pre-loop' if kw else 'pre-loop' if method == 'lsqr' else 'row/col sums + 11-step spectral radius'}) "
                   f"and the pinned-staged host copies (hostcopy.py: b narrowed to the operator precision on the "
                   f"host, x returned in fp64); one untimed warm-up solve; median of {n_solves} solves "
                   f"({', '.join(f'{1e3 * t:.0f}' for t in t_solves)} ms)"}
    del bstack, b_host

    peaks = measured_peaks()
    clocks = clk.summary()
    f_mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    peak_slots = SMS * LANES * f_mhz * 1e6
    nnz = NNZ[cfg]
    dom, t_dom = ("A^T", t_at) if t_at >= t_a else ("A", t_a)
    achieved = SLOTS_PER_NNZ * nnz / (t_dom * 1e-3)
    f32 = args.precision == "f32"
    bp_kernel = "k_bp_sided" if op.info.bp_sided_gs > 0 else "k_bp_boundary"
    kname = {"A^T": bp_kernel if f32 else "k_bp64", "A": "k_project_q" if f32 else "k_project64"}[dom]
    traffic = committed_traffic(cfg) if f32 else {}
    roof = {"bound": "issue", "kernel": f"{dom} ({kname})",
            "achieved": achieved / 1e9, "peak": peak_slots / 1e9, "unit": "Gslot/s", "frac": achieved / peak_slots,
            "traffic": traffic.get(kname),
            "traffic_unit": "B per operator application (DRAM read + write, ncu --set full of this build; A^T "
                            "summed over its view-batch launches)",
            "traffic_A": traffic.get("k_project_q"),
            "traffic_source": traffic.get("source"),
            # the HBM view of the same kernel: measured DRAM bytes per application over the live time,
            # against MEASURED_PEAKS.json hbm_gbs (shows the kernel is not HBM-bound)
            "hbm_gbs": (traffic[kname] / (t_dom * 1e-3) / 1e9) if traffic.get(kname) else None,
            "hbm_peak_gbs": peaks.get("hbm_gbs"),
            "hbm_frac": (traffic[kname] / (t_dom * 1e-3) / 1e9 / peaks["hbm_gbs"])
            if traffic.get(kname) and peaks.get("hbm_gbs") else None,
            "definition": "SURVEY.md 8(d): 8 FP32-lane-slot equivalents per nonzero of A; peak = 148 SM x 128 "
                          f"lanes x f_SM (median SM clock under load, {f_mhz:.0f} MHz)",
            "ncu_utilisation": {k: v for k, v in traffic.get("ncu_utilisation", {}).items() if k != "source"} or None,
            "algorithmic_bytes": 4 * (op.n + op.m),
            "frac_A": SLOTS_PER_NNZ * nnz / (t_a * 1e-3) / peak_slots,
            "frac_AT": SLOTS_PER_NNZ * nnz / (t_at * 1e-3) / peak_slots}
    cpu = None
    if rank == 0 and not args.no_cpu:
        s = cpu_sample(cfg)
        cpu = {"value": 1.0 / s["t_iter"], "unit": "it/s", "cores": s["threads"], "kind": "port",
               "sample": f"{s['sample']}; t_A {s['t_A']:.1f}s t_AT {s['t_AT']:.1f}s (fixed {s['t_AT_fixed']:.2f}s) "
                         f"-> one CGLS iteration of the reference algorithm",
               "extrapolated": s["extrapolated"], "workers": s["workers"]}
    line = {
        "metric": f"{sname} iterations/sec", "value": value, "unit": "it/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"config{cfg}: Shepp-Logan {N}^3, {V} views of {nu}x{nv}, {sname} step",
                   "solver": solver, "precision": args.precision, "parallelism": "single",
                   "l2": "working set > 126 MB L2 (no flush needed)"},
        "gups_A": N ** 3 * V / (t_a * 1e-3) / 1e9, "gups_AT": N ** 3 * V / (t_at * 1e-3) / 1e9,
        "ms_A": t_a, "ms_AT": t_at, "ms_rest_of_step": ms_step - t_a - t_at,
        "loop": loop,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
        "setup_s": t_setup, "plan_table_bytes": int(op.info.table_bytes),
        "plan": {"proj_chunk": int(op.info.proj_chunk), "bp_groups": int(op.info.bp_groups),
                 "bp_view_batches": int(op.info.bp_view_batches), "bp_closed_form": int(op.info.bp_closed_form)},
        "e_last": e_last,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, cfg, rank, world, local_rank):
    """N > 1: one solve (CGLS, LSQR+Jacobi or PSIRT) sharded over the ranks (views for A, cell rows for
    A^T), NCCL all_gathers of the volume and projection vectors before A and A^T
    (paper_2110_13526_b200/distributed.py).  Strong scaling: total work fixed."""
    import torch
    import torch.distributed as dist

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import _lib
    from paper_2110_13526_b200.distributed import (CudaVectors, DistCglsRun, DistClassicalRun, DistLsqrRun,
                                                   ShardedOperator, TorchComm)
    from paper_2110_13526_b200.solvers import SolverConfig

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    N, V, nu, nv, _, K = CONFIGS[cfg]
    solver = args.solver or CONFIGS[cfg][4]
    sname = SOLVER_NAME[solver]
    method, kw = SOLVER_METHOD[solver]
    vg, tr = geometry(cfg)
    comm = TorchComm()
    sop = ShardedOperator(vg, tr, comm, device=dev)
    if args.p2p:  # fused update + all-gather kernels over NVLink peer memory
        sop.enable_p2p()
    op = sop.op
    # inverse crime b = A phantom; each rank projects its own view block (rank-local plan)
    sop._d_full[: op.vol_elems] = op.phantom_internal(P.shepp_logan_3d())
    b_local = torch.zeros(sop.m_loc, device=dev)
    sop.project_local(sop._d_full, b_local)
    vec = CudaVectors(op)
    steps, warmup = args.steps, args.warmup

    def new_run(bl, iters, record=False):
        scfg = SolverConfig(method=method, max_iterations=iters, **kw)
        if method == "cgls":
            return DistCglsRun(sop, vec, bl, scfg, record=record)
        if method == "lsqr":
            return DistLsqrRun(sop, vec, bl, scfg, record=record)
        return DistClassicalRun(sop, vec, bl, scfg, method, record=record)

    run = new_run(b_local, steps + warmup + 1)
    stream = torch.cuda.current_stream(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if method == "cgls":
        # device-resident sharded loop: norm partials all-gathered and summed on the GPU, no host
        # round trip inside the K iterations (distributed.DistCglsRun.run_device)
        run.run_device(warmup)
        dist.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.lib().cbct_launch_count()
        with ClockSampler(local_rank) as clk:
            start.record(stream)
            run.run_device(steps)
            end.record(stream)
            torch.cuda.synchronize()
        assert run.i == warmup + steps, "the timed loop must run exactly K iterations"
    else:
        # host-driven sharded LSQR / PSIRT: rank-ordered fp64 scalar sums between the kernels
        for _ in range(warmup):
            run.step()
        dist.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.lib().cbct_launch_count()
        with ClockSampler(local_rank) as clk:
            start.record(stream)
            for _ in range(steps):
                run.step()
            end.record(stream)
            torch.cuda.synchronize()
    launches = _lib.lib().cbct_launch_count() - launches0
    t = torch.tensor([start.elapsed_time(end)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / steps

    def kernel_ms(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    p_tmp = torch.zeros(sop.m_loc, device=dev)
    r_tmp = torch.zeros(sop.n_loc, device=dev)
    t_a = kernel_ms(lambda: sop.project_local(sop._d_full, p_tmp))
    t_at = kernel_ms(lambda: sop.backproject_local(sop._e_full, r_tmp))
    del p_tmp, r_tmp, run
    tk = torch.tensor([t_a, t_at], device=dev)
    dist.all_reduce(tk, op=dist.ReduceOp.MAX)
    t_a, t_at = (float(v) for v in tk.tolist())
    # end to end: host view block in (pinned), sharded solve, x shards gathered to rank-0 host
    e2e_k = max(steps, 5)
    b_host = b_local.cpu().pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bl = b_host.to(dev, non_blocking=True)
    r2 = new_run(bl, e2e_k)
    if method == "cgls":
        while r2.should_continue():
            r2.run_device(e2e_k - r2.i)
    else:
        while r2.should_continue():
            r2.step()
    _, x_loc = r2.finish()
    x_full = sop.gather_volume(x_loc)
    x_host = x_full[: op.vol_elems].cpu() if rank == 0 else None
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    peaks = measured_peaks()
    clocks = clk.summary()
    f_mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    peak_slots = SMS * LANES * f_mhz * 1e6
    nnz = NNZ[cfg]
    nnz_a = nnz * (sop.v1 - sop.v0) / V  # views are symmetric: nnz splits evenly
    dom, t_dom = ("A^T", t_at) if t_at >= t_a else ("A", t_a)
    nnz_dom = nnz / world if dom == "A^T" else nnz_a
    achieved = SLOTS_PER_NNZ * nnz_dom / (t_dom * 1e-3)
    line = {
        "metric": f"{sname} iterations/sec", "value": 1e3 / ms_step, "unit": "it/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"config{cfg}: Shepp-Logan {N}^3, {V} views of {nu}x{nv}, {sname} step",
                   "solver": solver,
                   "parallelism": f"A by view x{world}, A^T by cell rows x{world}, " +
                                  ("fused d/e updates with NVLink peer stores" if args.p2p else "NCCL all_gather d/e"),
                   "l2": "working set > 126 MB L2 (no flush needed)"},
        "ms_A_local": t_a, "ms_AT_local": t_at,
        "roofline": {"bound": "issue", "kernel": dom, "achieved": achieved / 1e9, "peak": peak_slots / 1e9,
                     "unit": "Gslot/s", "frac": achieved / peak_slots, "traffic": None,
                     "definition": "per-rank share of SURVEY.md 8(d) slots (A^T share approximated as nnz/N)"},
        "cpu_baseline": None,
        "e2e": {"value": e2e_k / float(te.item()), "unit": "it/s", "h2d_bytes_per_step": int(sop.m_loc * 4 / e2e_k),
                "d2h_bytes_per_step": int(op.vol_elems * 4 / e2e_k) if rank == 0 else 0,
                "note": f"sharded solve from pinned host view blocks, K={e2e_k}, incl. pre-loop and x gather"},
        "clocks": clocks, "gpu_launches": int(launches),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--solver", default=None, choices=sorted(SOLVER_METHOD),
                    help="solver of the timed step (default: the config's, BASELINE.json: cgls, config 4 lsqr-jacobi)")
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"],
                    help="operator / vector precision (f64: the reference-precision path, csrc/f64.cu)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--sharded", action="store_true", help="use the sharded (multi-GPU) driver even at N=1")
    ap.add_argument("--p2p", action="store_true",
                    help="sharded driver: fused update + NVLink peer stores instead of NCCL all_gathers of d and e")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, args.config, rank, world)
    if world > 1 or args.sharded:
        import torch

        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        rc = run_sharded(args, args.config, rank, world, local_rank)
        torch.distributed.destroy_process_group()
        return rc
    return run_ours(args, args.config, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
