"""Profiling driver: build config C, run `--sweeps` serial-schedule HOOI sweeps (no eigen-solve overlap) so that
ncu sees each kernel alone.  Usage: python tools/profile_sweep.py --config 2 --sweeps 2
With --profiler-range the last sweep alone lies between cudaProfilerStart/Stop (ncu --profile-from-start off), so a
capture holds the sweep's own launches and not those of the input assembly."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--overlap", type=int, default=0)
ap.add_argument("--profiler-range", action="store_true")
args = ap.parse_args()
cfg = W.CONFIGS[args.config]
ctx = E.Context(0)
host, handle = bench.pinned_array(int(np.prod(cfg.L, dtype=np.int64)))
dt = bench.build_on_gpu(ctx, cfg, host, os.cpu_count() or 1)
tree = P.optimal_tree(cfg.spec).tree
plan = E.HooiPlan(ctx, cfg.spec, tree, "jacobi")
plan.set_overlap_evd(bool(args.overlap))
plan.set_factors(W.start_factors(cfg))
for i in range(args.sweeps):
    ranged = args.profiler_range and i == args.sweeps - 1
    if ranged:
        import torch
        ctx.synchronize()
        torch.cuda.profiler.start()
    plan.sweep(dt)
    if ranged:
        ctx.synchronize()
        torch.cuda.profiler.stop()
    print(i, plan.last_timing(), [round(x * 1e3) for x in plan.node_timing()[0]])
print("fit", plan.fit_from_norms(dt))
