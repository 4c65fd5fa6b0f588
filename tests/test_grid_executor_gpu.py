"""The C++ grid executor (csrc/grid_executor.cu, C ABI tp_grid_*) as virtual ranks on one B200: every rank is its own
context and stream on device 0, the data plane is the same peer-pointer code that runs across NVLink on a multi-GPU
box.  Compared with the single-process oracle after every sweep; the elements it ships per node must equal the
reference's volume model (grid_volume.hpp:32-46, grid_dynamic.hpp:37-62) and traced regrid counts
(simulate.hpp:97-113) exactly."""
import numpy as np
import pytest

from oracle import hooi_oracle as ho
from paper_1707_05594_b200 import Errc, TuckerplanError, engine as E, hostgen, planner as P, workloads as W

pytestmark = pytest.mark.gpu


def otree(tree):
    return ho.Tree(tree.n_modes, tree.kind, tree.mode, tree.parent)


def run_grid(L, K, q, sweeps=3, node_grids=None, seed_config=1):
    cfg = W.scaled_config(seed_config, L, K, sweeps)
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    procs = int(np.prod(q))
    grid = E.GridHooi(spec, tree, q, [0] * procs, node_grids=node_grids)
    grid.set_tensor(t)
    grid.set_factors(f0)
    of = [f.copy() for f in f0]
    tnorm = ho.frobenius_norm(t)
    out = []
    for _ in range(sweeps):
        st = grid.sweep()
        ost = ho.SweepStats()
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi", ost)
        assert (st.tree_macs, st.core_macs, st.peak_live, st.degenerate) == \
               (ost.tree_macs, ost.core_macs, ost.peak_live, ost.degenerate)
        gf, gcore = grid.get_factors(), grid.get_core()
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(gf, of))
        on = float(np.sqrt(np.sum(ocore * ocore)))
        tn, cn = grid.norms()
        assert abs(tn - tnorm) <= 1e-13 * tnorm
        assert abs(cn - float(np.sqrt(np.sum(gcore * gcore)))) <= 1e-13 * cn
        assert angle < 1e-9, angle
        assert abs(cn - on) <= 1e-10 * on
        ofit = np.sqrt(max(tnorm ** 2 - on ** 2, 0.0)) / tnorm
        assert abs(grid.fit_from_norms() - ofit) <= 1e-10 * max(ofit, 1e-3)
        out.append(grid.last_volumes())
    # the core itself (not only its norm): same subspaces give the same core up to the factors' column signs, which
    # the sign rule fixes identically on both sides
    assert np.max(np.abs(np.abs(gcore) - np.abs(ocore))) <= 1e-7 * np.max(np.abs(ocore))
    grid.close()
    return spec, tree, out


GRIDS = [
    ([40, 36, 32], [6, 5, 4], [1, 1, 1]),
    ([40, 36, 32], [6, 5, 4], [1, 1, 2]),
    ([40, 36, 32], [6, 5, 4], [2, 1, 2]),
    ([40, 36, 32], [6, 5, 4], [2, 2, 2]),
    ([41, 37, 33], [7, 5, 3], [1, 3, 1]),           # uneven cuts: 37 -> 12, 12, 13; 5 -> 1, 2, 2
    ([24, 20, 18, 16], [4, 3, 3, 2], [2, 1, 3, 1]),
    ([24, 20, 18, 16], [4, 3, 3, 2], [1, 2, 1, 2]),
    ([12, 10, 9, 8, 7], [3, 2, 2, 2, 2], [1, 2, 1, 1, 2]),
    ([64, 48], [5, 5], [2, 4]),              # two modes (K_0 = K_1: both leaves have full rank), both split
]


@pytest.mark.parametrize("L,K,q", GRIDS, ids=lambda v: "x".join(map(str, v)))
def test_static_grids_match_oracle_and_volume_model(L, K, q):
    spec, tree, volumes = run_grid(L, K, q)
    model = P.static_volume(tree, spec, q, int(np.prod(q)))
    want = list(model.per_node)
    for ttm, regrid in volumes:               # every sweep ships exactly the model's volume per node
        assert ttm == want, (ttm, want)
        assert sum(regrid) == 0
    assert sum(volumes[0][0]) == model.total


def test_optimal_static_grids_of_scaled_configs():
    for index, L, K, procs in ((3, [80, 20, 20, 10], [8, 4, 4, 2], 4), (1, [40, 40, 40], [8, 8, 8], 8)):
        spec = P.ProblemSpec(L, K)
        tree = P.optimal_tree(spec).tree
        best = P.optimal_static_grid(tree, spec, procs)
        _, _, volumes = run_grid(L, K, list(best.grid), sweeps=2, seed_config=index)
        assert sum(volumes[-1][0]) == best.report.total


def test_dynamic_scheme_with_regrids():
    """A per-node scheme (grid_dynamic.hpp): nodes whose grid differs from their parent's redistribute their input;
    shipped elements per node equal the traced counts of the reference's simulator."""
    L, K, procs = [16, 12, 10, 8], [4, 3, 2, 2], 4
    spec = P.ProblemSpec(L, K)
    tree = P.optimal_tree(spec).tree
    dyn = P.optimal_dynamic_scheme(tree, spec, procs)
    scheme = dyn.scheme
    # force at least one regrid if the optimum has none: flip one node's grid to another valid one
    node_grids = {k: list(v) for k, v in scheme.node_grids.items()}
    if all(list(g) == list(scheme.root) for g in node_grids.values()):
        grids = P.enumerate_grids(procs, spec)
        other = next(g for g in grids if list(g) != list(scheme.root))
        first = sorted(node_grids)[0]
        node_grids[first] = list(other)
    _, _, volumes = run_grid(L, K, list(scheme.root), sweeps=3, node_grids=node_grids, seed_config=2)
    sch = P.DynamicGridScheme(list(scheme.root), node_grids)
    model = P.scheme_volume(tree, spec, sch, procs)
    ttm, regrid = volumes[-1]
    for node in node_grids:
        assert ttm[node] == model.per_node_ttm[node]
        up = tree.parent[node]
        src = list(scheme.root) if tree.kind[up] == P.ROOT else node_grids[up]
        ext = list(spec.L)                      # the node's input: K on the modes multiplied above it
        at = up
        while at > 0:
            ext[tree.mode[at]] = spec.K[tree.mode[at]]
            at = tree.parent[at]
        assert regrid[node] == P.count_moved(ext, src, node_grids[node])
    assert any(regrid)


def test_errors():
    spec = P.ProblemSpec([8, 8, 8], [2, 2, 2])
    tree = P.optimal_tree(spec).tree
    with pytest.raises(TuckerplanError) as err:
        E.GridHooi(spec, tree, [4, 1, 1], [0, 0, 0, 0])          # q_0 > K_0
    assert err.value.code == Errc.invalid_grid
    with pytest.raises(TuckerplanError) as err:
        E.GridHooi(spec, tree, [2, 1, 1], [0, 0, 0])             # grid does not multiply out to the rank count
    assert err.value.code == Errc.invalid_grid
    g = E.GridHooi(spec, tree, [2, 1, 1], [0, 0])
    with pytest.raises(TuckerplanError) as err:
        g.sweep()                                                # nothing set yet
    assert err.value.code == Errc.bad_argument
    with pytest.raises(TuckerplanError) as err:
        E.GridHooi(spec, tree, [2, 1, 1], [0, 0], use_nccl=True)  # NCCL refuses two ranks on one device
    assert err.value.code == Errc.nccl
    g.close()


def test_nccl_transport_world_size_one():
    """TP_GRID_NCCL with a single rank: ncclCommInitAll, all-reduce and broadcast are exercised end to end (the only
    NCCL configuration a one-GPU box allows)."""
    L, K = [40, 36, 32], [6, 5, 4]
    cfg = W.scaled_config(1, L, K, 2)
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    try:
        grid = E.GridHooi(spec, tree, [1, 1, 1], [0], use_nccl=True)
    except TuckerplanError as exc:
        if exc.code == Errc.nccl and "could not be loaded" in str(exc):
            pytest.skip("no libnccl.so.2 on this box")
        raise
    grid.set_tensor(t)
    grid.set_factors(f0)
    of = [f.copy() for f in f0]
    for _ in range(2):
        grid.sweep()
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi", None)
    assert max(ho.sin_largest_principal_angle(a, b) for a, b in zip(grid.get_factors(), of)) < 1e-9
    grid.close()
