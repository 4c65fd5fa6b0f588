"""Kernel timeline of one steady-state HOOI sweep with the engine's defaults (eigen-solves overlapped), taken with the
CUPTI activity records behind torch.profiler (nsys is not in this image): which kernel ran when on which stream.
python tools/timeline_sweep.py --config 5 --out gpurun_out/timeline_c5.json   (prints a per-stream digest)"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--warm", type=int, default=5)
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--plan-option", action="append", default=[], metavar="ID=VALUE", help="tp_plan_set_option before the run")
ap.add_argument("--min-us", type=float, default=20.0, help="digest: kernels at least this long")
args = ap.parse_args()
cfg = W.CONFIGS[args.config]
ctx = E.Context(0)
host, handle = bench.pinned_array(int(np.prod(cfg.L, dtype=np.int64)))
dt = bench.build_on_gpu(ctx, cfg, host, os.cpu_count() or 1)
tree = P.optimal_tree(cfg.spec).tree
plan = E.HooiPlan(ctx, cfg.spec, tree, "jacobi")
for item in args.plan_option:
    plan.set_option(int(item.split("=")[0]), int(item.split("=")[1]))
plan.set_factors(W.start_factors(cfg))
for _ in range(args.warm):
    plan.sweep(dt)
ctx.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    plan.sweep(dt)
    ctx.synchronize()
    torch.cuda.synchronize()
prof.export_chrome_trace(args.out + ".chrome")
ev = [e for e in json.load(open(args.out + ".chrome"))["traceEvents"]
      if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
t0 = min(e["ts"] for e in ev)
rows = sorted(({"start_us": round(e["ts"] - t0, 1), "dur_us": round(e["dur"], 1), "stream": e["args"].get("stream"),
                "grid": e["args"].get("grid"), "name": e["name"][:70]} for e in ev), key=lambda r: r["start_us"])
json.dump(rows, open(args.out, "w"), indent=0)
os.remove(args.out + ".chrome")
print("kernels", len(rows), "span_us", round(max(r["start_us"] + r["dur_us"] for r in rows), 1))
for r in rows:
    if r["dur_us"] >= args.min_us:
        print("%10.1f %9.1f  s%-3s %-16s %s" % (r["start_us"], r["dur_us"], r["stream"], r["grid"], r["name"]))
