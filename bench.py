#!/usr/bin/env python
"""HOOI benchmark for the B200 engine (and the CPU reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference] [--grid 2x2x2|dynamic]

A step is one HOOI iteration (one `hooi_sweep`: TTM-tree -> Gram + eigenvectors per leaf -> core) of BASELINE.json
config C (default 5: 1600^3 -> 100^3, the largest single-GPU configuration and the one north_star's target names)
on a seeded synthetic low-rank-plus-noise tensor (SURVEY.md §8d recipe, paper_1707_05594_b200/workloads.py).
Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.

N > 1: one process per GPU over NCCL.  Under torchrun (WORLD_SIZE set) this process is one rank; started plainly
(`python bench.py --gpus N`) it re-executes itself under `python -m torch.distributed.run --nproc-per-node N`.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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
PARITY_ANGLE, PARITY_REL = 1e-9, 1e-10   # north_star: subspace angle / core norm and fit, relative


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def shared_config(name, iterations, tree_label, n_gpus, grid, grid_volume, compare_grid=None):
    """The `config` object BOTH arms print for a given (config, N): the workload and the reference's own selections
    for it.  Everything specific to one engine goes under its `engine` key instead, so the driver's same-config
    check compares like with like."""
    return {"workload": name, "iterations": int(iterations), "schedule": "jacobi on optimal_tree",
            "tree": tree_label, "n_gpus": int(n_gpus), "grid": [int(v) for v in grid],
            "grid_volume_elements": int(grid_volume), "compare_grid": compare_grid}


def comparison_grid(n_modes, world, K):
    """north_star: on the largest config the optimal grid is compared with the uniform 2x2x2 grid (8 GPUs, 3 modes)."""
    if world == 8 and n_modes == 3 and all(k >= 2 for k in K):
        return [2, 2, 2]
    return None


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


def cpu_iteration(t, L, K, factors, otree):
    """One HOOI iteration of the CPU restatement (oracle/hooi_oracle.py) with every host BLAS thread."""
    from oracle import hooi_oracle as ho
    timers = {}
    t0 = time.perf_counter()
    core, new = ho.hooi_sweep(t, list(L), list(K), factors, otree, "jacobi", None, timers)
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
            dt, _, _, _ = cpu_iteration(t, spec.L, spec.K, factors, oracle_tree(tree))
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


def oracle_run_with_parity(host_t, spec, tree, f0, iterations, gpu_step, budget_s=60.0):
    """The oracle's HOOI run from the start factors beside the engine's, compared after EVERY iteration.
    gpu_step() advances the engine by one iteration and returns (factors, core_norm, fit).  The oracle runs the
    config's full iteration count unless that would exceed budget_s (then as many as fit, at least one)."""
    from oracle import hooi_oracle as ho
    otree = oracle_tree(tree)
    tnorm2 = float(np.dot(host_t.reshape(-1), host_t.reshape(-1)))
    of = [f.copy() for f in f0]
    rows, secs, phases = [], [], {}
    wall0 = time.perf_counter()
    for it in range(iterations):
        if it and (time.perf_counter() - wall0) + secs[0] > budget_s:
            break
        dt, ocore, of, timers = cpu_iteration(host_t, spec.L, spec.K, of, otree)
        secs.append(dt)
        for k, v in timers.items():
            phases[k] = phases.get(k, 0.0) + v
        gf, gnorm, gfit = gpu_step()
        onorm = float(np.sqrt(np.sum(ocore * ocore)))
        ofit = float(np.sqrt(max(tnorm2 - onorm * onorm, 0.0) / tnorm2))
        rows.append({"iteration": it + 1,
                     "max_sin_principal_angle": max(ho.sin_largest_principal_angle(a, b) for a, b in zip(gf, of)),
                     "core_norm_rel_diff": abs(gnorm - onorm) / onorm,
                     "fit_rel_diff": abs(gfit - ofit) / max(ofit, 1e-3), "fit_oracle": ofit})
    ok = all(r["max_sin_principal_angle"] < PARITY_ANGLE and r["core_norm_rel_diff"] < PARITY_REL and
             r["fit_rel_diff"] < PARITY_REL for r in rows)
    return {"secs": secs, "phases": {k: v / len(secs) for k, v in phases.items()}, "rows": rows, "ok": ok}


# --------------------------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU implementation of the path on the same config and metric.  Its Eigen engine cannot be built
    here (Eigen is absent), so the arithmetic is the oracle port (NumPy/OpenBLAS, all host threads); the inputs and
    the selections (tree, grid) come from the reference's own headers compiled into oracle/_ref/libref_shim.so.  This
    arm maps no product library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref_inputs as R
    index = args.config
    L, K, sigma, iterations, _ = R.CONFIGS[index]
    cores = os.cpu_count() or 1
    otree = R.optimal_tree(L, K)
    grid, volume = R.optimal_static_grid(L, K, otree, args.gpus) if args.gpus > 1 else ([1] * len(L), 0)
    if args.grid and args.grid != "dynamic":
        grid = [int(v) for v in args.grid.split("x")]
        volume = R.static_volume(L, K, otree, grid, args.gpus)
    t = R.build_tensor(index, threads=cores)
    factors = R.start_factors(index)
    budget_s = 240.0
    wall0 = time.perf_counter()
    dt0, _, factors, _ = cpu_iteration(t, L, K, factors, otree)  # first (warm-up) iteration, also sizes the run
    warm_done = 1
    while warm_done < args.warmup and (time.perf_counter() - wall0) + dt0 * (1 + 1) < budget_s:
        _, _, factors, _ = cpu_iteration(t, L, K, factors, otree)
        warm_done += 1
    times = []
    phase = {}
    while len(times) < args.steps and (not times or (time.perf_counter() - wall0) + dt0 < budget_s):
        dt, _, factors, timers = cpu_iteration(t, L, K, factors, otree)
        times.append(dt)
        for k, v in timers.items():
            phase[k] = phase.get(k, 0.0) + v
    value = float(np.mean(times))
    name = R.config_name(index)
    sample = ("%d full HOOI iteration(s) of %s timed after %d warm-up (asked %d/%d; bounded to ~%.0f s of CPU work)"
              % (len(times), name, warm_done, args.steps, args.warmup, budget_s))
    line = {
        "impl": "reference", "metric": "hooi_s_per_iter", "value": value, "unit": "s/iter", "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm_done, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": shared_config(name, iterations, R.tree_label(otree), args.gpus, grid, volume,
                                "x".join(map(str, comparison_grid(len(L), args.gpus, K) or [])) or None),
        "cpu_baseline": {"value": value, "unit": "s/iter", "cores": cores, "kind": "port", "sample": sample,
                         "phases_s_per_iter": {k: v / len(times) for k, v in phase.items()},
                         "inputs": "reference headers compiled into oracle/_ref/libref_shim.so (random_tensor stream, "
                                   "optimal_tree, optimal_static_grid); no product library mapped"},
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
    if world > 1 or args.distributed or args.backend != "cuda":
        from paper_1707_05594_b200 import distributed as D
        return D.run_bench_rank(args, rank, world, local_rank)

    torch.cuda.set_device(0)
    import ctypes
    for item in args.global_option:
        opt, val = item.split("=")
        E.check(E.lib.tp_set_global_option(int(opt), ctypes.c_longlong(int(val))))
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
    for item in args.plan_option:
        opt, val = item.split("=")
        plan.set_option(int(opt), int(val))

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
    # (no carried path yet); the whole series from the start is reported in `run_from_start` below.
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
    graph_replayed = sum(node_ms) == 0.0          # replayed whole-sweep graphs carry no per-node events
    # fit evaluation, timed separately from the sweep (the reference's CLI also calls it outside)
    w0 = time.perf_counter()
    fit = plan.fit_from_norms(dt)
    fit_norms_ms = (time.perf_counter() - w0) * 1e3
    plan.reconstruction_error(dt)                       # first call pays one-off kernel set-up for new shapes
    w0 = time.perf_counter()
    fit_full = plan.reconstruction_error(dt)
    fit_full_ms = (time.perf_counter() - w0) * 1e3
    evd_info = plan.evd_info()

    # The per-TTM numbers come from a second pass of the same K iterations with the eigen-solves serialised behind
    # the tree instead of beside it (which also means plain launches, no replayed graph): in the overlapped schedule
    # a TTM's event span also contains whatever eigen-solve kernels shared the SMs with it.
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
    if graph_replayed:
        overlapped_node_ms = node_ms

    # Third pass: the same K iterations with the carried path off, i.e. tree + full core chain per iteration as the
    # reference schedules it (hooi.hpp:189-229); reported beside the headline, which uses the engine's default.
    plan.set_carry_path(False)
    plan.set_factors(f0)
    nocarry_ms = [one_step(True)[0] for _ in range(steps)]
    factors_nocarry = plan.get_factors()          # K iterations from the start factors
    plan.set_carry_path(True)

    # run_from_start: the workload BASELINE.json names -- the config's iterations from the random orthonormal start --
    # with every iteration timed, the cold first one included.
    plan.set_factors(f0)
    from_start = [one_step(True)[0] for _ in range(max(cfg.iterations, steps))]
    factors_k = None
    if steps <= len(from_start):
        plan.set_factors(f0)
        for _ in range(steps):
            one_step(False)
        factors_k = plan.get_factors()
    nocarry_same = factors_k is not None and all(np.array_equal(a, b) for a, b in zip(factors_k, factors_nocarry))

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
    # Where the timed region replays the whole sweep as one graph (short sweeps), single launches cannot be bracketed
    # by events there and the serial pass of the same iterations supplies the launch time.
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
                     "avg_launch_ms": dom["ms"],
                     "timed": ("CUDA events around the launch, serial pass of the same iterations (the timed region "
                               "replays the sweep as one CUDA graph)" if graph_replayed else
                               "CUDA events around the launch, timed region, engine defaults"),
                     "serial_pass": {"avg_launch_ms": serial_same["ms"], "achieved": serial_achieved,
                                     "frac": serial_achieved / (p_fp64 if dom["bound"] == "tensor" else hbm_gbs),
                                     "slowest_node_in_serial_pass": dom_serial["node"]},
                     "peak_source": fp64_src if dom["bound"] == "tensor" else hbm_src})

    # e2e: the reference-facing by-value call with HOST buffers.  Headline: the whole HOOI run of the config as the
    # reference CLI drives it (tools/tuckerplan_cli.cpp:416-419: hooi_sweep by value in a loop on one tensor) -- every
    # call passes the host tensor and host factors and receives host factors + core; the tensor crosses PCIe in the
    # first call and later calls carry the caller's promise that it has not changed (TP_HOST_TENSOR_UNCHANGED).
    # Timed from the first call (cold context cache, upload included) to the last download, divided by the iterations.
    # Beside it: the same call without the promise (33 GB up every call) and the resident API.
    e2e = None
    if not args.no_e2e:
        host_t = host_flat.reshape(cfg.L)
        fbytes = 8 * sum(l * k for l, k in zip(spec.L, spec.K))
        cbytes = 8 * int(np.prod(spec.K))
        iters = cfg.iterations
        # warm-up call: creates the context's cached plan and device tensor (allocation, handle and kernel set-up are
        # one-off costs of a process, reported separately); the timed run below still moves every byte
        ctx.release_cache()
        w0 = time.perf_counter()
        dw = E.hooi_sweep(host_t, spec, E.Decomposition(None, f0), tree, "jacobi", ctx=ctx)
        first_call_s = time.perf_counter() - w0
        # ... and the rest of one whole warm-up run: the second and third calls of a process pay one-off costs of their
        # own (lazy loading of the kernels only a warm sweep launches, the first recording of a leaf's launch
        # sequence: 140 ms once on C3), which belong to the process, not to an iteration
        for i in range(1, iters):
            dw = E.hooi_sweep(host_t, spec, dw, tree, "jacobi", ctx=ctx, tensor_unchanged=True)
        ctx.synchronize()
        d = E.Decomposition(None, f0)
        w0 = time.perf_counter()
        per_call_ms = []
        for i in range(iters):
            # call 1 makes no promise: the tensor is uploaded (and the start factors make it a cold sweep)
            c0 = time.perf_counter()
            d = E.hooi_sweep(host_t, spec, d, tree, "jacobi", ctx=ctx, tensor_unchanged=i > 0)
            per_call_ms.append((time.perf_counter() - c0) * 1e3)
        run_s = (time.perf_counter() - w0) / iters
        # the by-value run against the resident run of the same iterations: same subspaces to rounding
        plan.set_factors(f0)
        for _ in range(iters):
            plan.sweep(dt)
        agree = max(sin_principal_angle(a, b) for a, b in zip(d.factors, plan.get_factors()))
        # every call uploads (no promise)
        d2 = E.Decomposition(None, f0)
        every_steps = min(args.steps, 3)
        w0 = time.perf_counter()
        for _ in range(every_steps):
            d2 = E.hooi_sweep(host_t, spec, d2, tree, "jacobi", ctx=ctx)
        every_s = (time.perf_counter() - w0) / every_steps
        ctx.release_cache()
        # resident API (DeviceTensor + HooiPlan): per step host factors in, host factors + core out
        plan.set_factors(f0)
        plan.sweep(dt)
        ctx.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            plan.sweep(dt)
            plan.get_factors()
            plan.get_core()
        resident_s = (time.perf_counter() - w0) / args.steps
        e2e = {"value": run_s, "unit": "s/iter",
               "h2d_bytes_per_step": (total * 8) // iters + fbytes, "d2h_bytes_per_step": fbytes + cbytes,
               "host_memory": "pinned",
               "what": "whole run of the config's %d iterations through the by-value C-ABI call, upload of the tensor "
                       "(first call) included, later calls with TP_HOST_TENSOR_UNCHANGED; mean per iteration; process "
                       "warm (one earlier run of the same calls on the same context: allocations, lazily loaded "
                       "kernels; the timed run uploads, starts cold and records its graphs again)" % iters,
               "first_call_of_a_process_s": first_call_s, "per_call_ms": per_call_ms,
               "max_sin_principal_angle_vs_resident_run": agree,
               "by_value_every_call": {"value": every_s, "unit": "s/iter", "h2d_bytes_per_step": total * 8 + fbytes,
                                       "d2h_bytes_per_step": fbytes + cbytes, "calls": every_steps},
               "resident_api": {"value": resident_s, "unit": "s/iter", "h2d_bytes_per_step": 0,
                                "d2h_bytes_per_step": fbytes + cbytes,
                                "what": "tensor resident (DeviceTensor + HooiPlan); factors + core read back each step"}}

    # CPU baseline and parity: the oracle port runs the config's iterations from the start factors on the same host
    # tensor, all cores; the engine runs the same iterations and is compared after every one of them.
    cpu, parity_ok = None, True
    if not args.no_cpu:
        host_t = host_flat.reshape(cfg.L)
        plan.set_factors(f0)

        def gpu_step():
            plan.sweep(dt)
            return plan.get_factors(), plan.core_norm(), plan.fit_from_norms(dt)

        res = oracle_run_with_parity(host_t, spec, tree, f0, cfg.iterations, gpu_step)
        parity_ok = res["ok"]
        secs = float(np.mean(res["secs"]))
        single = cpu_single_thread(host_t, spec, f0, tree, cost, secs, cores)
        cpu = {"value": secs, "unit": "s/iter", "cores": cores, "kind": "port", "single_thread": single,
               "sample": "%d of the %d HOOI iterations of %s from the start factors (NumPy/OpenBLAS oracle port), "
                         "mean per iteration" % (len(res["secs"]), cfg.iterations, cfg.name),
               "phases_s": res["phases"], "parity_per_iteration": res["rows"], "parity_ok": parity_ok,
               "parity_bar": {"max_sin_principal_angle": PARITY_ANGLE, "core_norm_rel_diff": PARITY_REL,
                              "fit_rel_diff": PARITY_REL},
               "parity_first_iteration": {k: res["rows"][0][k] for k in ("max_sin_principal_angle", "core_norm_rel_diff")}}

    line = {
        "metric": "hooi_s_per_iter", "value": ms_per_step * 1e-3, "unit": "s/iter", "n_gpus": 1, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": shared_config(cfg.name, cfg.iterations, tree.label(), 1, [1] * spec.n_modes(), 0),
        "engine": {"timed_steps": "iterations W+1..W+K of one HOOI run from the random orthonormal start",
                   "evd": "certified top-k subspace iteration (one launch for small leaves), else full syevd; on side streams",
                   "core": "chain along a tree path, partial products carried into the next sweep",
                   "sweep_graph": "replayed" if graph_replayed else "plain launches",
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
                     # the FP64 pipe's own ceiling: one DMMA.8x8x4 (512 flop) per 4 cycles per SM at the sampled clock
                     # (37.1 TF/s measured by tools/microbench/fp64_peaks.cu, profiles/r01_fp64_peaks.jsonl)
                     "dmma_issue_ceiling_tflops": (torch.cuda.get_device_properties(0).multi_processor_count * 128
                                                   * (clocks.get("sm_mhz") or 1965.0) * 1e6 / 1e12),
                     "per_node": [{k: r[k] for k in ("node", "mode", "bound", "ms", "tflops", "frac")} for r in rows]},
        "ttm_tree_overlapped_ms": sum(overlapped_node_ms[r["node"]] for r in rows),
        "serial_schedule": {"ms_per_step": float(np.mean(serial_ms)), "phases_ms": serial_phases,
                            "note": "steady state: one cold sweep from the start factors precedes the K timed ones"},
        # what of the leaf solves is NOT hidden behind the tree: the timed step minus the serial pass's tree, Gram
        # and core time (the summed evd_ms of the serial pass counts every leaf in full; on the side streams they
        # overlap each other and the tree, and only this remainder is on the critical path)
        "critical_path": {"step_ms": ms_per_step, "tree_ms": serial_phases.get("tree_ms"),
                          "gram_ms": serial_phases.get("gram_ms"), "core_ms": serial_phases.get("core_ms"),
                          "leaf_solves_summed_ms": serial_phases.get("evd_ms"),
                          "leaf_solves_exposed_ms": max(0.0, ms_per_step - serial_phases.get("tree_ms", 0.0)
                                                        - serial_phases.get("gram_ms", 0.0) - serial_phases.get("core_ms", 0.0))},
        "run_from_start": {"per_iteration_ms": from_start, "iterations": len(from_start),
                           "mean_ms": float(np.mean(from_start[:cfg.iterations])),
                           "note": "one HOOI run from the random orthonormal start, every iteration timed (CUDA "
                                   "events); iteration 1 is cold: no carried products, eigen-solves from the caller's "
                                   "factors. mean_ms is over the config's %d iterations" % cfg.iterations},
        "carried_path": {"enabled": True, "ms_first_iteration_cold": from_start[0],
                         "ms_per_step_disabled": float(np.mean(nocarry_ms)),
                         "factors_bit_identical_when_disabled": bool(nocarry_same),
                         "note": "the core chain runs along a tree path; its partial products are the next sweep's "
                                 "tree nodes and are not recomputed. ms_per_step_disabled: the first K iterations "
                                 "from the start factors with the option off (the reference's schedule)."},
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
    if not parity_ok:
        print("bench.py: parity against the oracle FAILED, see cpu_baseline.parity_per_iteration", file=sys.stderr)
        return 3
    return 0


# --------------------------------------------------------------------------------------------- in-process grid
def run_inprocess_grid(args):
    """`--executor inprocess`: the C++ grid executor (tp_grid_*, csrc/grid_executor.cu) drives all N GPUs from this one
    process over peer memory -- what a C++ caller of the reference API gets.  With fewer devices than ranks
    (--virtual-ranks) several ranks share a GPU: a functional run of the same code path, not a scaling measurement."""
    import torch
    from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
    cfg = W.CONFIGS[args.config]
    spec = cfg.spec
    world = args.gpus
    n_dev = torch.cuda.device_count()
    if world > n_dev and not args.virtual_ranks:
        print("bench.py: %d ranks but %d GPU(s); pass --virtual-ranks for a functional run" % (world, n_dev), file=sys.stderr)
        return 2
    devices = [r % n_dev for r in range(world)]
    tree = P.optimal_tree(spec).tree
    cost = P.tree_cost(tree, spec)
    scheme = None
    if args.grid == "dynamic":
        scheme = P.optimal_dynamic_scheme(tree, spec, world).scheme
        q = list(scheme.root)
    else:
        q = [int(v) for v in args.grid.split("x")] if args.grid else list(P.optimal_static_grid(tree, spec, world).grid)
    volume = (P.scheme_volume(tree, spec, scheme, world).total if scheme else P.static_volume(tree, spec, q, world).total)
    hbm_gbs, hbm_src = read_peaks()
    torch.cuda.set_device(0)
    p_fp64, fp64_src = measure_fp64_peak(torch)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    host_t = W.build_tensor_host(cfg, cores)
    f0 = W.start_factors(cfg)
    grid = E.GridHooi(spec, tree, q, devices, node_grids=scheme.node_grids if scheme else None)
    grid.set_tensor(host_t)
    build_s = time.perf_counter() - t0
    grid.set_factors(f0)
    for _ in range(max(args.warmup, 0)):
        grid.sweep()
    k0, _ = grid.launch_counts()
    sampler = ClockSampler(0)
    sampler.start()
    step_ms, node_sum, volumes = [], None, None
    for _ in range(args.steps):
        grid.sweep()
        total_ms, per_node, _ = grid.last_timing()
        step_ms.append(total_ms)
        node_sum = per_node if node_sum is None else [a + b for a, b in zip(node_sum, per_node)]
        volumes = grid.last_volumes()
    clocks = sampler.stop()
    k1, lib_calls = grid.launch_counts()
    ms_per_step = float(np.mean(step_ms))
    node_ms = [v / args.steps for v in node_sum]
    fit = grid.fit_from_norms()

    cpu, parity_ok = None, True
    if not args.no_cpu:
        grid.set_factors(f0)

        def step():
            grid.sweep()
            return grid.get_factors(), grid.norms()[1], grid.fit_from_norms()

        res = oracle_run_with_parity(host_t, spec, tree, f0, cfg.iterations, step)
        parity_ok = res["ok"]
        cpu = {"value": float(np.mean(res["secs"])), "unit": "s/iter", "cores": cores, "kind": "port",
               "sample": "%d of the %d HOOI iterations of %s from the start factors (NumPy/OpenBLAS oracle port)"
                         % (len(res["secs"]), cfg.iterations, cfg.name),
               "phases_s": res["phases"], "parity_per_iteration": res["rows"], "parity_ok": parity_ok}

    node_q = (lambda node: scheme.node_grids[node]) if scheme else (lambda node: q)
    rows, t_roof, flops_total = [], 0.0, 0
    for node, kind in enumerate(tree.kind):
        if kind != 1:
            continue
        n = tree.mode[node]
        flops = 2 * spec.K[n] * cost.card_in[node]
        qn = node_q(node)[n]
        local_bytes = 8 * (cost.card_in[node] + qn * cost.card_out[node]) / world + 8 * spec.K[n] * spec.L[n]
        link_bytes = 8 * (qn - 1) * cost.card_out[node] / world
        t = max(flops / world / (p_fp64 * 1e12), local_bytes / (hbm_gbs * 1e9)) + link_bytes / (NVLINK_GBS * 1e9)
        t_roof += t
        flops_total += flops
        rows.append({"node": node, "mode": n, "ms": node_ms[node], "roofline_ms": t * 1e3,
                     "frac": t * 1e3 / node_ms[node] if node_ms[node] else None, "nvlink_bytes_per_gpu": link_bytes,
                     "shipped_elements": volumes[0][node], "regrid_elements": volumes[1][node]})
    ttm_ms = sum(r["ms"] for r in rows)
    dom = max(rows, key=lambda r: r["ms"])
    dom_flops = 2 * spec.K[dom["mode"]] * cost.card_in[dom["node"]]
    achieved = dom_flops / (dom["ms"] * 1e-3) / 1e12 if dom["ms"] else None
    compare_q = comparison_grid(spec.n_modes(), world, spec.K)
    line = {
        "metric": "hooi_s_per_iter", "value": ms_per_step * 1e-3, "unit": "s/iter", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": shared_config(cfg.name, cfg.iterations, tree.label(), world, q, volume if world > 1 else 0,
                                "x".join(map(str, compare_q)) if compare_q else None),
        "engine": {"executor": "in-process grid executor (tp_grid_*): peer-memory reduce-scatter from the TTM epilogue, "
                               "owner-rank leaf solves", "devices": devices, "virtual_ranks": world > n_dev,
                   "node_grids": {str(k): list(v) for k, v in scheme.node_grids.items()} if scheme else None},
        "ttm_tree": {"tflops": flops_total / (ttm_ms * 1e-3) / 1e12 if ttm_ms else None,
                     "roofline_frac": t_roof * 1e3 / ttm_ms if ttm_ms else None, "measured_ms": ttm_ms,
                     "roofline_ms": t_roof * 1e3, "flops": flops_total, "p_fp64_tflops": p_fp64,
                     "p_fp64_source": fp64_src, "hbm_gbs": hbm_gbs, "hbm_source": hbm_src, "nvlink_gbs": NVLINK_GBS,
                     "per_node": rows},
        "shipped_elements_per_sweep": sum(volumes[0]) + sum(volumes[1]), "relative_fit": fit, "build_s": build_s,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": p_fp64 * min(world, n_dev), "unit": "TFLOP/s",
                     "frac": achieved / (p_fp64 * min(world, n_dev)) if achieved else None, "traffic": None,
                     "kernel": "ttm kernel (tree node %d, mode %d) across %d rank(s)" % (dom["node"], dom["mode"] + 1, world),
                     "peak_source": fp64_src},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(k1 - k0), "library_calls": int(lib_calls), "clocks": clocks,
    }
    print(json.dumps(line))
    grid.close()
    return 0 if parity_ok else 3


# --------------------------------------------------------------------------------------------- launch
def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args, argv):
    """`python bench.py --gpus N` started plainly: become N ranks, one per GPU (the command the driver itself uses
    when it launches the ranks).  NCCL's communicator lines stay on stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // args.gpus)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
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
    ap.add_argument("--no-grid-comparison", action="store_true")
    ap.add_argument("--executor", default="ranks", choices=["ranks", "inprocess"],
                    help="N > 1: 'ranks' = one process per GPU over NCCL (torch.distributed); 'inprocess' = the C++ grid "
                         "executor (tp_grid_*) driving all GPUs from one process over peer memory")
    ap.add_argument("--peer-slots", action="store_true",
                    help="with --executor ranks: reduce-scatters as direct stores into NVLink-mapped symmetric-memory "
                         "slots (torch.distributed._symmetric_memory) instead of grouped send/recv")
    ap.add_argument("--virtual-ranks", action="store_true",
                    help="with --executor inprocess: allow more ranks than GPUs (functional run on a small box)")
    ap.add_argument("--backend", default="cuda", choices=["cuda", "numpy-test"],
                    help="numpy-test: CONTRACT TEST ONLY -- the grid executor's rank program over gloo with the tests' "
                         "NumPy stand-in for the local kernels (tests/numpy_ops.py); not a measurement")
    ap.add_argument("--global-option", action="append", default=[], metavar="ID=VALUE",
                    help="A/B switch: tp_set_global_option(ID, VALUE) before the run (include/tuckerplan_b200.h, "
                         "TP_GLOBAL_OPT_*), e.g. 4=0 keeps the TMA kernel's last row tile on a padded DMMA")
    ap.add_argument("--plan-option", action="append", default=[], metavar="ID=VALUE",
                    help="A/B switch: tp_plan_set_option(ID, VALUE) on the timed plan (TP_OPT_*), e.g. 10=0 sends a long "
                         "chain product beside running eigen-solves out as one launch")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be at least 1")
    if args.impl == "reference":
        return run_reference(args)
    if args.executor == "inprocess":
        return run_inprocess_grid(args) if int(os.environ.get("RANK", "0")) == 0 else 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args, argv)
    if args.backend == "numpy-test" and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args, argv)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
