"""Does the eigen-solve enqueue block the host?  Host wall time of the call vs time until the stream drains."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05594_b200 import engine as E, distributed as D, hostgen
ctx = E.Context(0)
ops = D.GpuOps(ctx)
for n, k in ((1600, 100), (400, 40), (200, 20), (108, 20)):
    a = hostgen.random_tensor([n, n], 1)
    g = a @ a.T
    for rep in range(3):
        buf = ops.from_host(g)
        ctx.synchronize()
        t0 = time.perf_counter()
        f, st = ops.leaf_solve(buf, n, k)
        t1 = time.perf_counter()
        ctx.synchronize()
        t2 = time.perf_counter()
    print("syevd n=%d: host call %.3f ms, until drained %.3f ms" % (n, (t1 - t0) * 1e3, (t2 - t0) * 1e3))
