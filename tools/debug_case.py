import sys, numpy as np
sys.path.insert(0, '.')
from oracle import hooi_oracle as ho
from paper_1707_05594_b200 import engine as E, planner as P, workloads as W
ctx = E.Context(0)
cfg = W.scaled_config(3, [33, 17, 9, 5], [7, 2, 3, 1], 2)
spec = cfg.spec
tree = P.optimal_tree(spec).tree
print(tree.label())
t = W.build_tensor_host(cfg)
f0 = W.start_factors(cfg)
dt = E.DeviceTensor.upload(ctx, t)
plan = E.HooiPlan(ctx, spec, tree, "jacobi"); plan.set_factors(f0)
st = plan.sweep(dt)
ot = ho.Tree(tree.n_modes, tree.kind, tree.mode, tree.parent)
ocore, of = ho.hooi_sweep(t, spec.L, spec.K, f0, ot, "jacobi")
gf = plan.get_factors()
for n in range(4):
    print(n, ho.sin_largest_principal_angle(gf[n], of[n]))
# leaf-level check: walk the tree on the oracle and compare gram + leaf factor per leaf
def visit(node, tensor):
    for c in ot.children[node]:
        m = ot.mode[c]
        if ot.kind[c] == 2:
            d = E.DeviceTensor.upload(ctx, tensor)
            g = d.gram(m); u = ho.unfold(tensor, m); want = u @ u.T
            v, deg = d.leaf_factor(m, spec.K[m]); ov, odeg = ho.leading_from_gram(want, spec.K[m])
            ev = np.linalg.eigvalsh(want)
            print("leaf", m, tensor.shape, "gram err", np.max(np.abs(g - want)), "angle", ho.sin_largest_principal_angle(v, ov), "eig top", ev[::-1][:spec.K[m]+1])
            d.free()
        else:
            nxt = ho.ttm(tensor, f0[m].T, m)
            d = E.DeviceTensor.upload(ctx, tensor); z = d.ttm(f0[m].T, m); got = z.download(); z.free(); d.free()
            print("ttm", m, tensor.shape, np.max(np.abs(got - nxt)))
            visit(c, nxt)
visit(0, t)
