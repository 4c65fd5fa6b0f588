#!/usr/bin/env python
"""HOOI benchmark for the B200 engine (and the CPU reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A step is one HOOI iteration (one `hooi_sweep`: TTM-tree -> Gram + eigenvectors per leaf -> core) of BASELINE.json
config C (default 5: 1600^3 -> 100^3, the largest single-GPU configuration and the one north_star's target names)
on a seeded synthetic low-rank-plus-noise tensor (SURVEY.md §8d recipe, paper_1707_05594_b200/workloads.py).
Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0      # B200_PROFILING.md fallback
FP64_FALLBACK_TFLOPS = 35.77   # cuBLAS DGEMM 8192^3 measured on this pool (profiles/r01_fp64_peaks.jsonl)
NVLINK_GBS = 770.0             # measured peer copy per direction (B200_PROFILING.md)


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def tree_roofline(spec, tree, cost, p_fp64_tflops, hbm_gbs):
    """Per-TTM roofline of SURVEY.md §8d: flops_u = 2 K_n |In_u|, bytes_u = 8 (|In_u| + |Out_u| + K_n L_n),
    t_roof_u = max(flops_u / P_fp64, bytes_u / BW_hbm)."""
    rows = []
    for node, kind in enumerate(tree.kind):
        if kind != 1:
            continue
        n = tree.mode[node]
        flops = 2 * spec.K[n] * cost.card_in[node]
        nbytes = 8 * (cost.card_in[node] + cost.card_out[node] + spec.K[n] * spec.L[n])
        t_f, t_b = flops / (p_fp64_tflops * 1e12), nbytes / (hbm_gbs * 1e9)
        rows.append(dict(node=node, mode=n, flops=flops, bytes=nbytes, t_roof_s=max(t_f, t_b),
                         bound="tensor" if t_f >= t_b else "hbm"))
    return rows


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md recipe)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1])); power.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        # "under load": the samples above the idle clock
        busy = [s for s in sm if s > 500] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------------------------- workloads
def pinned_array(count):
    from paper_1707_05594_b200._lib import check, lib
    p = ctypes.c_void_p()
    check(lib.tp_host_alloc(ctypes.c_size_t(count * 8), ctypes.byref(p)))
    arr = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(count,))
    return arr, p


def build_on_gpu(ctx, cfg, host_flat, threads):
    """T = X + sigma E assembled on the device from host-generated noise; returns the device tensor and fills
    host_flat with the same bits (so every arm consumes identical input)."""
    from paper_1707_05594_b200 import engine as E, workloads as W
    W.noise_into(cfg, host_flat.reshape(cfg.L), threads)
    dt = E.DeviceTensor.upload_raw(ctx, cfg.L, host_flat.ctypes.data)
    x = E.DeviceTensor.upload(ctx, W.generating_core(cfg))
    for n, a in enumerate(W.generating_factors(cfg)):
        nxt = x.ttm(a, n)
        x.free()
        x = nxt
    dt.axpby(cfg.sigma, 1.0, x)
    x.free()
    dt.download_into(host_flat.ctypes.data)
    return dt


def oracle_tree(tree):
    from oracle import hooi_oracle as ho
    return ho.Tree(tree.n_modes, tree.kind, tree.mode, tree.parent)


def cpu_iteration(t, spec, factors, tree):
    """One HOOI iteration of the CPU restatement (oracle/hooi_oracle.py) with every host BLAS thread."""
    from oracle import hooi_oracle as ho
    timers = {}
    t0 = time.perf_counter()
    core, new = ho.hooi_sweep(t, spec.L, spec.K, factors, oracle_tree(tree), "jacobi", None, timers)
    return time.perf_counter() - t0, core, new, timers


def cpu_single_thread(t, spec, factors, tree, cost, secs_all_cores, cores, budget_s=30.0):
    """The same CPU port on ONE BLAS thread (the reference's own build is single-threaded, proj/CMakeLists.txt:7-20):
    a full iteration where that fits the budget, otherwise the first root product on a slab subset, scaled by MACs."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    from oracle import hooi_oracle as ho
    with threadpool_limits(limits=1):
        if secs_all_cores * cores <= budget_s:
            dt, _, _, _ = cpu_iteration(t, spec, factors, tree)
            return {"value": dt, "unit": "s/iter", "cores": 1, "sample": "1 full iteration, BLAS limited to one thread"}
        node = next(i for i, k in enumerate(tree.kind) if k == 1)          # first root child
        mode = tree.mode[node]
        slab_mode = 0 if mode != 0 else 1
        keep = max(1, spec.L[slab_mode] // 16)
        sl = [slice(None)] * len(spec.L)
        sl[slab_mode] = slice(0, keep)
        sub = np.ascontiguousarray(t[tuple(sl)])
        t0 = time.perf_counter()
        ho.ttm(sub, np.ascontiguousarray(factors[mode].T), mode)
        dt = time.perf_counter() - t0
        macs = spec.K[mode] * sub.size
        est = dt * (cost.total_macs + spec.K[tree.mode[node]] * int(np.prod(spec.L, dtype=object))) / macs
        return {"value": est, "unit": "s/iter", "cores": 1, "kind": "extrapolated",
                "sample": "root product T x_%d on %d of %d slabs of mode %d took %.2f s on one thread (%.1f GMAC/s); "
                          "scaled to the iteration's tree + first core product MACs, eigen-solves not included"
                          % (mode + 1, keep, spec.L[slab_mode], slab_mode + 1, dt, macs / dt / 1e9)}


# --------------------------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU implementation of the path (its Eigen engine cannot be built here — Eigen is absent — so
    this is the oracle port, NumPy/OpenBLAS, all host threads) on the same config and metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1707_05594_b200 import planner as P, workloads as W
    cfg = W.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg, threads=cores)
    factors = W.start_factors(cfg)
    budget_s = 240.0
    wall0 = time.perf_counter()
    dt0, _, factors, _ = cpu_iteration(t, spec, factors, tree)  # first (warm-up) iteration, also sizes the run
    warm_done = 1
    while warm_done < args.warmup and (time.perf_counter() - wall0) + dt0 * (1 + 1) < budget_s:
        _, _, factors, _ = cpu_iteration(t, spec, factors, tree)
        warm_done += 1
    times = []
    phase = {}
    while len(times) < args.steps and (not times or (time.perf_counter() - wall0) + dt0 < budget_s):
        dt, _, factors, timers = cpu_iteration(t, spec, factors, tree)
        times.append(dt)
        for k, v in timers.items():
            phase[k] = phase.get(k, 0.0) + v
    value = float(np.mean(times))
    sample = ("%d full HOOI iteration(s) of %s timed after %d warm-up (asked %d/%d; bounded to ~%.0f s of CPU work)"
              % (len(times), cfg.name, warm_done, args.steps, args.warmup, budget_s))
    line = {
        "impl": "reference", "metric": "hooi_s_per_iter", "value": value, "unit": "s/iter", "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm_done, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "iterations": cfg.iterations, "schedule": "jacobi on optimal_tree"},
        "cpu_baseline": {"value": value, "unit": "s/iter", "cores": cores, "kind": "port", "sample": sample,
                         "phases_s_per_iter": {k: v / len(times) for k, v in phase.items()}},
        "e2e": {"value": value, "unit": "s/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------------------------- B200 arm
def measure_fp64_peak(torch):
    """cuBLAS DGEMM 8192^3, best of 5 (the FP64 roofline denominator; MEASURED_PEAKS.json has no FP64 entry)."""
    try:
        n = 8192
        a = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        b = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        torch.cuda.empty_cache()
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12, "measured live (cuBLAS DGEMM 8192^3, best of 5)"
    except Exception as exc:  # pragma: no cover
        return FP64_FALLBACK_TFLOPS, "fallback (profiles/r01_fp64_peaks.jsonl): %s" % exc


def sin_principal_angle(a, b):
    """sin of the largest principal angle between the column spaces of two orthonormal bases."""
    r = b - a @ (a.T @ b)                       # component of b outside span(a): accurate for tiny angles
    return float(np.linalg.svd(r, compute_uv=False).max())


def run_b200(args):
    import torch
    from paper_1707_05594_b200 import engine as E, planner as P, workloads as W

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.distributed:
        from paper_1707_05594_b200 import distributed as D
        return D.run_bench_rank(args, rank, world, local_rank)

    torch.cuda.set_device(0)
    cfg = W.CONFIGS[args.config]
    spec = cfg.spec
    cores = os.cpu_count() or 1
    hbm_gbs, hbm_src = read_peaks()
    p_fp64, fp64_src = measure_fp64_peak(torch)

    ctx = E.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    opt = P.optimal_tree(spec)
    tree = opt.tree
    cost = P.tree_cost(tree, spec)
    total = int(np.prod(cfg.L, dtype=np.int64))
    host_flat, host_handle = pinned_array(total)
    t_build = time.perf_counter()
    dt = build_on_gpu(ctx, cfg, host_flat, cores)
    t_build = time.perf_counter() - t_build
    f0 = W.start_factors(cfg)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")

    # L2 hygiene: inputs far larger than the 126 MB L2 need nothing; otherwise flush between steps
    small = total * 8 < 4 * 126e6
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda") if small else None

    def one_step(timed):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = plan.sweep(dt)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), st

    # One HOOI run from the random orthonormal start: W untimed warm-up iterations, then the K timed ones continue
    # it ("mean over the config's iterations after one warm-up").  The first iteration of a run is cold
    # (no carried path yet); it is timed separately below and reported in `carried_path`.
    plan.set_factors(f0)
    for _ in range(max(args.warmup, 0)):
        one_step(False)
    ctx.synchronize()
    torch.cuda.synchronize()
    k0, _ = ctx.launch_counts()
    sampler = ClockSampler(0)
    sampler.start()
    step_ms, phases, node_ms_sum = [], {}, None
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        ms, st = one_step(True)
        step_ms.append(ms)
        for k, v in plan.last_timing().items():
            phases[k] = phases.get(k, 0.0) + v
        nm, em = plan.node_timing()
        node_ms_sum = nm if node_ms_sum is None else [a + b for a, b in zip(node_ms_sum, nm)]
    ctx.synchronize()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    k1, lib_calls = ctx.launch_counts()
    steps = len(step_ms)
    ms_per_step = float(np.sum(step_ms)) / steps
    phases = {k: v / steps for k, v in phases.items()}
    node_ms = [v / steps for v in node_ms_sum]
    # fit evaluation, timed separately from the sweep (the reference's CLI also calls it outside)
    w0 = time.perf_counter()
    fit = plan.fit_from_norms(dt)
    fit_norms_ms = (time.perf_counter() - w0) * 1e3
    plan.reconstruction_error(dt)                       # first call pays one-off kernel set-up for new shapes
    w0 = time.perf_counter()
    fit_full = plan.reconstruction_error(dt)
    fit_full_ms = (time.perf_counter() - w0) * 1e3
    final_factors = plan.get_factors()
    evd_info = plan.evd_info()

    # The per-TTM numbers come from a second pass of the same K iterations with the eigen-solves serialised behind
    # the tree instead of beside it: in the overlapped schedule above a TTM's event span also contains whatever
    # eigen-solve kernels shared the SMs with it.  Both tree totals are reported.
    overlapped_node_ms = node_ms
    plan.set_overlap_evd(False)
    plan.set_factors(f0)
    one_step(False)  # cold sweep: afterwards every tree node runs exactly once per sweep (carried path)
    node_ms_sum, serial_ms, serial_phases = None, [], {}
    for _ in range(steps):
        ms, st = one_step(True)
        serial_ms.append(ms)
        for k, v in plan.last_timing().items():
            serial_phases[k] = serial_phases.get(k, 0.0) + v / steps
        nm, em = plan.node_timing()
        node_ms_sum = nm if node_ms_sum is None else [a + b for a, b in zip(node_ms_sum, nm)]
    node_ms = [v / steps for v in node_ms_sum]
    plan.set_overlap_evd(True)

    # Third pass: the same K iterations with the carried path off, i.e. tree + full core chain per iteration as the
    # reference schedules it (hooi.hpp:189-229); reported beside the headline, which uses the engine's default.
    plan.set_carry_path(False)
    plan.set_factors(f0)
    nocarry_ms = [one_step(True)[0] for _ in range(steps)]
    factors_after_k = plan.get_factors()          # K iterations from the start factors
    plan.set_carry_path(True)
    plan.set_factors(f0)
    cold_ms = None
    for i in range(steps):
        ms, _ = one_step(False)
        if i == 0:
            cold_ms = ms                           # first iteration of a run: no carried path yet
    nocarry_same = all(np.array_equal(a, b) for a, b in zip(plan.get_factors(), factors_after_k))

    # TTM-tree phase vs its per-TTM roofline
    rows = tree_roofline(spec, tree, cost, p_fp64, hbm_gbs)
    tree_flops = sum(r["flops"] for r in rows)
    t_roof = sum(r["t_roof_s"] for r in rows)
    ttm_ms = sum(node_ms[r["node"]] for r in rows)
    for r in rows:
        r["ms"] = node_ms[r["node"]]
        r["frac"] = r["t_roof_s"] * 1e3 / r["ms"] if r["ms"] > 0 else None
        r["tflops"] = r["flops"] / (r["ms"] * 1e-3) / 1e12 if r["ms"] > 0 else None
    # `roofline`: the dominant tree node's kernel, timed where the contract asks -- CUDA events on the engine's
    # stream inside the timed region (engine defaults: eigen-solve kernels may share the SMs with it and the grid
    # leaves 2 SMs to them while any are in flight); the serial-pass figure of the same node is reported beside it.
    dom_serial = max(rows, key=lambda r: r["ms"])
    dom = dict(max(rows, key=lambda r: overlapped_node_ms[r["node"]]))
    dom["ms"] = overlapped_node_ms[dom["node"]]
    dom["tflops"] = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
    serial_same = next(r for r in rows if r["node"] == dom["node"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            entry = json.load(f).get(cfg.name, {})
            traffic = entry.get("by_node", {}).get(str(dom["node"]), entry.get("dominant_ttm_dram_bytes_per_launch"))
    except Exception:
        pass
    if dom["bound"] == "tensor":
        roofline = {"bound": "tensor", "achieved": dom["tflops"], "peak": p_fp64, "unit": "TFLOP/s",
                    "frac": dom["tflops"] / p_fp64, "traffic": traffic}
    else:
        gbs = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm_gbs, "unit": "GB/s", "frac": gbs / hbm_gbs,
                    "traffic": traffic}
    serial_achieved = (serial_same["tflops"] if dom["bound"] == "tensor"
                       else serial_same["bytes"] / (serial_same["ms"] * 1e-3) / 1e9)
    roofline.update({"kernel": "ttm_tma_kernel / ttm_dmma_kernel (tree node %d: mode %d, %s)"
                               % (dom["node"], dom["mode"] + 1, "FP64 DMMA pipe" if dom["bound"] == "tensor" else "HBM"),
                     "algorithmic_flops_per_launch": dom["flops"], "algorithmic_bytes_per_launch": dom["bytes"],
                     "avg_launch_ms": dom["ms"], "timed": "CUDA events around the launch, timed region, engine defaults",
                     "serial_pass": {"avg_launch_ms": serial_same["ms"], "achieved": serial_achieved,
                                     "frac": serial_achieved / (p_fp64 if dom["bound"] == "tensor" else hbm_gbs),
                                     "slowest_node_in_serial_pass": dom_serial["node"]},
                     "peak_source": fp64_src if dom["bound"] == "tensor" else hbm_src})

    # e2e: the reference-facing by-value call with HOST buffers (upload T + factors, sweep, download factors + core)
    e2e = None
    if not args.no_e2e:
        host_t = host_flat.reshape(cfg.L)
        d = E.Decomposition(None, f0)
        e2e_steps = args.steps
        E.hooi_sweep(host_t, spec, d, tree, "jacobi", ctx=ctx)  # warm (allocator, page tables)
        ctx.synchronize()
        w0 = time.perf_counter()
        for _ in range(e2e_steps):
            d = E.hooi_sweep(host_t, spec, d, tree, "jacobi", ctx=ctx)
        e2e_s = (time.perf_counter() - w0) / e2e_steps
        fbytes = 8 * sum(l * k for l, k in zip(spec.L, spec.K))
        # the by-value call starts every eigen-solve from the caller's factors, the resident run from its own Ritz
        # vectors: same subspaces to rounding, not the same bits
        agree = max(sin_principal_angle(a, b) for a, b in zip(d.factors, factors_after_k)) if e2e_steps == steps else None
        e2e = {"value": e2e_s, "unit": "s/iter", "h2d_bytes_per_step": total * 8 + fbytes,
               "d2h_bytes_per_step": fbytes + 8 * int(np.prod(spec.K)), "host_memory": "pinned",
               "max_sin_principal_angle_vs_resident_run": agree}

    # CPU baseline: the oracle port on the same host tensor, all cores, a bounded sample (one iteration)
    cpu = None
    if not args.no_cpu:
        host_t = host_flat.reshape(cfg.L)
        secs, ocore, ofac, timers = cpu_iteration(host_t, spec, f0, tree)
        from oracle import hooi_oracle as ho
        plan.set_factors(f0)
        plan.sweep(dt)
        gfac = plan.get_factors()
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(gfac, ofac))
        gnorm, onorm = plan.core_norm(), float(np.sqrt(np.sum(ocore * ocore)))
        single = cpu_single_thread(host_t, spec, f0, tree, cost, secs, cores)
        cpu = {"value": secs, "unit": "s/iter", "cores": cores, "kind": "port", "single_thread": single,
               "sample": "1 full HOOI iteration of %s from the start factors (NumPy/OpenBLAS oracle port)" % cfg.name,
               "phases_s": timers,
               "parity_first_iteration": {"max_sin_principal_angle": angle, "core_norm_rel_diff": abs(gnorm - onorm) / onorm}}

    line = {
        "metric": "hooi_s_per_iter", "value": ms_per_step * 1e-3, "unit": "s/iter", "n_gpus": 1, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "iterations": cfg.iterations, "schedule": "jacobi on optimal_tree",
                   "timed_steps": "iterations W+1..W+K of one HOOI run from the random orthonormal start",
                   "tree": tree.label(), "grid": [1] * spec.n_modes(), "evd": "top-k subspace iteration where certified, else full syevd; on side streams",
                   "core": "chain along a tree path, partial products carried into the next sweep",
                   "l2": "flushed_between_steps" if small else "inputs_larger_than_L2",
                   "noise": "slab-parallel" if cfg.slab_noise else "sequential"},
        "ttm_tree": {"schedule": "serial pass (eigen-solves not overlapped), same K iterations",
                     "tflops": tree_flops / (ttm_ms * 1e-3) / 1e12, "roofline_frac": t_roof * 1e3 / ttm_ms,
                     "measured_ms": ttm_ms, "roofline_ms": t_roof * 1e3, "flops": tree_flops,
                     "p_fp64_tflops": p_fp64, "p_fp64_source": fp64_src, "hbm_gbs": hbm_gbs, "hbm_source": hbm_src,
                     # the same per-TTM roofline against the nominal peaks north_star quotes (report both)
                     "roofline_frac_nominal_peaks": sum(r["t_roof_s"] for r in tree_roofline(spec, tree, cost, 40.0, 8000.0))
                                                    * 1e3 / ttm_ms,
                     "nominal_peaks": {"fp64_tflops": 40.0, "hbm_gbs": 8000.0},
                     "per_node": [{k: r[k] for k in ("node", "mode", "bound", "ms", "tflops", "frac")} for r in rows]},
        "ttm_tree_overlapped_ms": sum(overlapped_node_ms[r["node"]] for r in rows),
        "serial_schedule": {"ms_per_step": float(np.mean(serial_ms)), "phases_ms": serial_phases,
                            "note": "steady state: one cold sweep from the start factors precedes the K timed ones"},
        "carried_path": {"enabled": True, "ms_first_iteration_cold": cold_ms,
                         "ms_per_step_disabled": float(np.mean(nocarry_ms)),
                         "factors_bit_identical_when_disabled": bool(nocarry_same),
                         "note": "the core chain runs along a tree path; its partial products are the next sweep's "
                                 "tree nodes and are not recomputed. The first iteration of a run (first warm-up step "
                                 "here) is cold: tree + whole chain. ms_per_step_disabled: same K iterations from "
                                 "the start factors with the option off (the reference's schedule)."},
        "evd": {"fast_path_leaves": evd_info[0], "redone_with_full_solve_last_sweep": evd_info[1]},
        "phases_ms": phases, "relative_fit": fit,
        "fit_evaluation": {"from_norms": fit, "from_norms_ms": fit_norms_ms, "full_expansion": fit_full,
                           "full_expansion_ms": fit_full_ms,
                           "note": "reconstruction_error (hooi.hpp:232-245) on the device, host wall time incl. "
                                   "allocation of the expansion; not part of the timed sweep"}, "wall_s_timed_region": wall, "build_s": t_build,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(k1 - k0),
        "library_calls": int(lib_calls), "clocks": clocks,
    }
    print(json.dumps(line))
    plan.close()
    dt.free()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--distributed", action="store_true", help="force the grid executor at N=1 (run under torchrun)")
    ap.add_argument("--grid", default=None,
                    help="override the optimal static grid, e.g. 2x2x2; 'dynamic' = per-node grids (optimal_dynamic_scheme)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
