import os, sys, time, json
import numpy as np
sys.path.insert(0, "/root/repo")
import bench
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
cfg = W.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
spec = cfg.spec
ctx = E.Context(0)
total = int(np.prod(cfg.L, dtype=np.int64))
host, handle = bench.pinned_array(total)
dt = bench.build_on_gpu(ctx, cfg, host, os.cpu_count() or 1)
tree = P.optimal_tree(spec).tree
f0 = W.start_factors(cfg)
host_t = host.reshape(cfg.L)
E.hooi_sweep(host_t, spec, E.Decomposition(None, f0), tree, "jacobi", ctx=ctx)
ctx.synchronize()
out = []
for rep in range(30):
    d = E.Decomposition(None, f0)
    calls = []
    for i in range(cfg.iterations):
        w0 = time.perf_counter()
        d = E.hooi_sweep(host_t, spec, d, tree, "jacobi", ctx=ctx, tensor_unchanged=i > 0)
        calls.append(round((time.perf_counter() - w0) * 1e3, 2))
    out.append(calls)
    print(rep, calls, flush=True)
