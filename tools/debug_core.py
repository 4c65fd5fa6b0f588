import sys, os, numpy as np
sys.path.insert(0, '.')
from oracle import hooi_oracle as ho
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
ctx = E.Context(0)
cfg = W.scaled_config(5, [768, 720, 704], [24, 20, 16], 3)
spec = cfg.spec
tree = P.optimal_tree(spec).tree
print(tree.label())
t = W.build_tensor_host(cfg)
f0 = W.start_factors(cfg)
dt = E.DeviceTensor.upload(ctx, t)
ot = ho.Tree(tree.n_modes, tree.kind, tree.mode, tree.parent)
for overlap, fast in ((1, 0),):
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.set_overlap_evd(bool(overlap)); plan.set_fast_evd(bool(fast))
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    for it in range(3):
        plan.sweep(dt)
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, ot, "jacobi")
        gf = plan.get_factors(); gc = plan.get_core()
        # core from the GPU factors by the oracle: isolates the core chain from the factors
        ref = ho.core_from_factors(t, gf)
        d = np.abs(gc - ref)
        bad = np.argwhere(d > 1e-9 * np.max(np.abs(ref)))
        print("overlap", overlap, "fast", fast, "it", it, "evd_info", plan.evd_info(), "core maxdiff", d.max(), "nbad", len(bad), bad[:4].tolist(),
              "angles", ["%.1e" % ho.sin_largest_principal_angle(a, b) for a, b in zip(gf, of)],
              "norm rel", abs(np.linalg.norm(gc) - np.linalg.norm(ocore)) / np.linalg.norm(ocore))
    plan.close()
