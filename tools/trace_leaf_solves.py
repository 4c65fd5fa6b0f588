"""Per-sweep certificate margins and sweep times of a BASELINE config (TP_CTX_OPT_TRACE_EVD on): which leaves take
the one-launch kernel, how many power steps the launch-sequence solves settle at, when the sweep graph starts to
replay.  python tools/trace_leaf_solves.py --config 3 --sweeps 14"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B
from paper_1707_05594_b200 import engine as E
from paper_1707_05594_b200 import planner as P
from paper_1707_05594_b200 import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--sweeps", type=int, default=14)
    args = ap.parse_args()
    cfg = W.CONFIGS[args.config]
    ctx = E.Context(0)
    ctx.set_option(2, 1)
    stream = torch.cuda.ExternalStream(ctx.stream)
    tree = P.optimal_tree(cfg.spec).tree
    total = int(np.prod(cfg.L, dtype=np.int64))
    host_flat, _ = B.pinned_array(total)
    dt = B.build_on_gpu(ctx, cfg, host_flat, os.cpu_count() or 1)
    plan = E.HooiPlan(ctx, cfg.spec, tree, "jacobi")
    plan.set_factors(W.start_factors(cfg))
    for i in range(args.sweeps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.sweep(dt)
        e1.record(stream)
        e1.synchronize()
        print(f"sweep {i + 1}: {e0.elapsed_time(e1):.3f} ms  {plan.sweep_info()}", file=sys.stderr)


if __name__ == "__main__":
    main()
