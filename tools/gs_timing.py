"""Gauss-Seidel sweeps (hooi.hpp:206-225, chain-input tree -- the reference CLI's default schedule) on the B200:
ms per iteration in steady state, with and without the carried chain.  usage: python tools/gs_timing.py [configs...]"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench as B
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W

ctx = E.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
for index in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    cfg = W.CONFIGS[index]
    spec = cfg.spec
    tree = P.chain_tree(spec)
    total = int(np.prod(cfg.L, dtype=np.int64))
    host_flat, handle = B.pinned_array(total)
    dt = B.build_on_gpu(ctx, cfg, host_flat, os.cpu_count() or 1)
    f0 = W.start_factors(cfg)
    out = {"workload": cfg.name, "schedule": "gauss_seidel on chain_tree(input order)",
           "tree_macs": P.tree_cost(tree, spec).total_macs}
    for carry in (True, False):
        plan = E.HooiPlan(ctx, spec, tree, "gauss_seidel")
        plan.set_carry_path(carry)
        plan.set_factors(f0)
        for _ in range(3):
            plan.sweep(dt)
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.sweep(dt)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        out["ms_per_iter_carried_chain" if carry else "ms_per_iter_plain"] = float(np.mean(ms))
        out["fast_leaves, redone"] = plan.evd_info()
        plan.close()
    dt.free()
    print(json.dumps(out), flush=True)
