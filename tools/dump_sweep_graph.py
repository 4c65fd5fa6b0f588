import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import bench
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
cfg = W.CONFIGS[int(sys.argv[1])]
ctx = E.Context(0)
ctx.set_option(3, 1)
host, handle = bench.pinned_array(int(np.prod(cfg.L, dtype=np.int64)))
dt = bench.build_on_gpu(ctx, cfg, host, os.cpu_count() or 1)
plan = E.HooiPlan(ctx, cfg.spec, P.optimal_tree(cfg.spec).tree, "jacobi")
plan.set_factors(W.start_factors(cfg))
for _ in range(6):
    plan.sweep(dt)
ctx.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
os.system("cp /tmp/tpb_sweep_graph.dot gpurun_out/sweep_graph_c%s.dot" % sys.argv[1])
