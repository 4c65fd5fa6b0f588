"""Planner parity: every selection (tree shape and node ids, MAC ledger, grids, volumes, cut points) must be
bit-identical to the reference's, as recorded in tests/golden/planner_golden.json by the reference itself
(tests/golden/make_golden.py -> oracle/_ref/ref_tools)."""
import json
import os

import numpy as np
import pytest

from paper_1707_05594_b200 import Errc, TuckerplanError
from paper_1707_05594_b200 import planner as P


def _tree_eq(tree: P.TtmTree, gold: dict):
    assert tree.kind == gold["kind"]
    assert tree.mode == gold["mode"]
    assert tree.parent == gold["parent"]


def _check_tree(tree, gold, spec):
    _tree_eq(tree, gold)
    cost = P.tree_cost(tree, spec)
    assert cost.total_macs == gold["total_macs"]
    assert cost.per_node_macs == gold["per_node_macs"]
    assert cost.n_internal == gold["n_internal"]
    assert cost.depth == gold["depth"]
    assert cost.card_in == gold["card_in"]
    assert cost.card_out == gold["card_out"]
    assert P.is_canonical(tree) == gold["canonical"]
    assert P.tree_depth(tree) == gold["depth"]
    P.validate_tree(tree, spec)


def test_all_golden_cases(planner_golden):
    n_ok = 0
    for case in planner_golden["cases"]:
        spec = P.ProblemSpec(case["L"], case["K"])
        if "error" in case:
            with pytest.raises(TuckerplanError) as e:
                P.optimal_tree(spec)
            assert int(e.value.code) == case["error"] + 1
            assert e.value.mode == case["error_mode"]
            continue
        opt = P.optimal_tree(spec)
        assert opt.total_macs == case["opt_total_macs"]
        assert opt.dp_states == case["dp_states"]
        _check_tree(opt.tree, case["opt"], spec)
        assert P.optimal_cost_reuse_greedy(spec) == case["reuse_greedy_macs"]
        _check_tree(P.chain_tree(spec, P.CHAIN_INPUT), case["chain_input"], spec)
        _check_tree(P.chain_tree(spec, P.CHAIN_BY_COST), case["chain_by_cost"], spec)
        _check_tree(P.chain_tree(spec, P.CHAIN_BY_RATIO), case["chain_by_ratio"], spec)
        _check_tree(P.balanced_tree(spec), case["balanced"], spec)
        _check_tree(P.canonicalize(P.chain_tree(spec)), case["canonical_chain"], spec)
        _tree_eq(P.build_tree(spec, "opt"), case["opt"])
        _tree_eq(P.build_tree(spec, "chain-k"), case["chain_by_cost"])
        _tree_eq(P.build_tree(spec, "chain-h"), case["chain_by_ratio"])
        for procs, g in case["grids"].items():
            procs = int(procs)
            grids = P.enumerate_grids(procs, spec)
            assert grids == g["enumerated"]
            if not grids:
                with pytest.raises(TuckerplanError) as e:
                    P.optimal_static_grid(opt.tree, spec, procs)
                assert e.value.code == Errc.no_valid_grid
                continue
            for threads in (1, 3):
                best = P.optimal_static_grid(opt.tree, spec, procs, threads)
                assert best.grid == g["best"]
                assert best.report.total == g["best_volume"]
                assert [best.report.per_node[i] for i in g["per_node_ids"]] == g["per_node_ttm"]
                # the reference's traced reduce-scatter count agrees with the model (acceptance.cpp:199-240)
                assert g["traced_ttm"] == g["per_node_ttm"]
            assert [P.static_volume(opt.tree, spec, q, procs).total for q in grids] == g["volumes"]
        n_ok += 1
    assert n_ok > 150


def test_baseline_config_selections(planner_golden):
    """The SURVEY §8d / BASELINE.md §2 table, spelled out."""
    want = {
        (200, 200, 200): ("T(M2(M3(F1)), M1(M3(F2), M2(F3)))", 368000000, {2: [1, 1, 2], 4: [1, 1, 4], 8: [1, 1, 8]}),
        (96, 96, 96, 96): ("T(M3(M4(M2(F1), M1(F2))), M1(M2(M4(F3), M3(F4))))", 1912504320,
                           {2: [1, 1, 1, 2], 4: [1, 2, 1, 2], 8: [1, 2, 1, 4]}),
        (400, 100, 100, 50): ("T(M2(M3(M4(F1), M1(F4)), M4(M1(F3))), M4(M3(M1(F2))))", 4320000000,
                              {2: [2, 1, 1, 1], 4: [4, 1, 1, 1], 8: [8, 1, 1, 1]}),
        (48,) * 5: ("T(M3(M4(M5(M2(F1), M1(F2)))), M1(M2(M4(M5(F3)), M3(M5(F4), M4(F5)))))", 4973395968,
                    {2: [1, 1, 1, 1, 2], 4: [1, 1, 1, 1, 4], 8: [1, 1, 1, 1, 8]}),
        (1600,) * 3: ("T(M2(M3(F1)), M1(M3(F2), M2(F3)))", 896000000000, {2: [1, 1, 2], 4: [1, 1, 4], 8: [1, 1, 8]}),
    }
    ks = {(200,) * 3: [20] * 3, (96,) * 4: [10] * 4, (400, 100, 100, 50): [40, 10, 20, 5], (48,) * 5: [8] * 5,
          (1600,) * 3: [100] * 3}
    for L, (label, macs, grids) in want.items():
        spec = P.ProblemSpec(list(L), ks[L])
        opt = P.optimal_tree(spec)
        assert opt.tree.label() == label
        assert opt.total_macs == macs
        for procs, q in grids.items():
            assert P.optimal_static_grid(opt.tree, spec, procs).grid == q
    spec = P.ProblemSpec([1600] * 3, [100] * 3)
    tree = P.optimal_tree(spec).tree
    assert P.static_volume(tree, spec, [2, 2, 2], 8).total == 560000000
    assert P.static_volume(tree, spec, [1, 1, 8], 8).total == 224000000


def test_reference_integer_goldens():
    cube = P.ProblemSpec([4, 4, 4], [2, 2, 2])
    assert P.tree_cost(P.chain_tree(cube), cube).total_macs == 576          # test_trees.cpp:60-70
    assert len(P.chain_tree(cube).kind) == 10
    assert P.optimal_tree(cube).total_macs == 448                           # test_tree_search.cpp:80-88
    assert P.tree_cost(P.canonicalize(P.chain_tree(cube)), cube).total_macs == 448  # test_trees.cpp:163-174
    full = P.ProblemSpec([4, 3, 5], [4, 3, 5])
    assert P.tree_cost(P.chain_tree(P.ProblemSpec([2, 2, 2], [2, 2, 2])), P.ProblemSpec([2, 2, 2], [2, 2, 2])).total_macs > 0
    assert P.optimal_tree(full).total_macs > 0
    pinned = P.ProblemSpec([11, 7, 7, 11, 4], [3, 1, 2, 7, 1])                # test_tree_search.cpp:177-189
    assert P.optimal_tree(pinned).total_macs == 87659
    assert P.optimal_cost_reuse_greedy(pinned) == 89606
    chain = P.chain_tree(cube)
    vol = P.static_volume(chain, cube, [2, 2, 2], 8)                         # test_grids.cpp:106-115
    assert vol.total == 144 and vol.per_node[1] == 32 and vol.per_node[2] == 16
    best = P.optimal_static_grid(chain, cube, 4)                             # test_grids.cpp:117-124
    assert best.grid == [1, 2, 2] and best.report.total == 80
    with pytest.raises(TuckerplanError) as e:
        P.optimal_static_grid(chain, cube, 7)
    assert e.value.code == Errc.no_valid_grid
    assert P.enumerate_grids(4, cube) == [[1, 2, 2], [2, 1, 2], [2, 2, 1]]    # test_grids.cpp:59-72
    hcci = P.ProblemSpec([672, 672, 627, 16], [279, 279, 153, 14])            # README.md:65-72
    opt = P.optimal_tree(hcci)
    assert opt.total_macs == 3016394906112 and P.tree_depth(opt.tree) == 3
    g = P.optimal_static_grid(opt.tree, hcci, 32)
    assert g.grid == [4, 2, 4, 1] and g.report.total == 9784331982
    assert P.tree_cost(P.chain_tree(hcci, P.CHAIN_BY_COST), hcci).total_macs == 4637749483584  # README.md:103-104
    for n, count in {1: 0, 2: 2, 3: 5, 4: 8, 5: 12, 6: 16, 8: 24}.items():   # test_trees.cpp:100-111
        s = P.ProblemSpec([4] * n, [2] * n)
        assert P.tree_cost(P.balanced_tree(s), s).n_internal == count


def test_psi_and_blocks(planner_golden):
    for key, want in planner_golden["psi"].items():
        p, n = map(int, key.split(","))
        assert P.grid_count(p, n) == want
    # acceptance.cpp:62-75 spot values
    assert P.grid_count(32, 7) == 462
    for b in planner_golden["blocks"]:
        assert P.block_bounds(b["len"], b["parts"]) == b["cuts"]
        assert [P.block_of(c, b["len"], b["parts"]) for c in range(b["len"])] == b["block_of"]
    cuts = P.block_bounds(100, 8)
    assert [cuts[i + 1] - cuts[i] for i in range(8)] == [12, 13, 12, 13, 12, 13, 12, 13]


def test_spec_and_tree_error_codes():
    def code(fn):
        with pytest.raises(TuckerplanError) as e:
            fn()
        return e.value.code

    assert code(lambda: P.validate_spec(P.ProblemSpec([], []))) == Errc.bad_dims
    assert code(lambda: P.validate_spec(P.ProblemSpec([2] * 17, [1] * 17))) == Errc.bad_dims
    assert code(lambda: P.validate_spec(P.ProblemSpec([3, 0], [1, 1]))) == Errc.bad_dims
    assert code(lambda: P.validate_spec(P.ProblemSpec([3, 3], [1, 4]))) == Errc.k_too_large
    assert code(lambda: P.validate_spec(P.ProblemSpec([3, 3], [0, 1]))) == Errc.k_too_large
    assert code(lambda: P.validate_spec(P.ProblemSpec([2 ** 31] * 3, [1] * 3))) == Errc.overflow
    s = P.ProblemSpec([4, 4, 4], [2, 2, 2])
    good = P.optimal_tree(s).tree
    P.validate_tree(good, s)
    assert code(lambda: P.validate_tree(good, P.ProblemSpec([4, 4], [2, 2]))) == Errc.shape_mismatch
    # malformed trees (tests/test_trees.cpp:124-161): missing leaf, duplicate leaf, repeated mode, wrong path
    def tree(kind, mode, parent):
        return P.TtmTree(3, kind, mode, parent)
    assert code(lambda: P.validate_tree(tree([0, 1, 1, 2], [-1, 1, 2, 0], [-1, 0, 1, 2]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([0, 1, 1, 2, 2], [-1, 1, 2, 0, 0], [-1, 0, 1, 2, 2]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([0, 1, 1, 2], [-1, 1, 1, 0], [-1, 0, 1, 2]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([0, 1, 2], [-1, 1, 0], [-1, 0, 1]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([1, 1, 2], [-1, 1, 0], [-1, 0, 1]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([0, 1, 0], [-1, 1, 0], [-1, 0, 1]), s)) == Errc.bad_tree
    assert code(lambda: P.validate_tree(tree([0, 1, 1], [-1, 1, 2], [-1, 0, 1]), s)) == Errc.bad_tree  # childless mode
    assert code(lambda: P.validate_grid([1, 3, 1], s, 3)) == Errc.invalid_grid
    assert code(lambda: P.validate_grid([1, 2, 1], s, 4)) == Errc.invalid_grid
    assert code(lambda: P.optimal_static_grid(good, s, 16)) == Errc.no_valid_grid
    assert code(lambda: P.grid_count(0, 3)) == Errc.bad_argument
    assert code(lambda: P.build_tree(s, 9)) == Errc.bad_argument


# ---- per-node grids (grid_dynamic.hpp / simulate.hpp), pinned to the reference through tests/golden/dynamic_golden.json
def _dynamic_cases():
    with open(os.path.join(os.path.dirname(__file__), "golden", "dynamic_golden.json")) as f:
        return json.load(f)


def _tree_by_name(name, spec):
    return {"opt": lambda: P.optimal_tree(spec).tree, "chain": lambda: P.chain_tree(spec),
            "chain_by_cost": lambda: P.chain_tree(spec, P.CHAIN_BY_COST), "balanced": lambda: P.balanced_tree(spec)}[name]()


def test_dynamic_schemes_match_reference():
    cases = _dynamic_cases()
    assert len(cases) >= 200
    regridding = 0
    for c in cases:
        spec = P.ProblemSpec(c["L"], c["K"])
        if "error" in c:
            with pytest.raises(TuckerplanError) as e:
                P.optimal_dynamic_scheme(_tree_by_name(c["tree_name"], spec), spec, c["procs"])
            assert int(e.value.code) == c["error"] + 1          # C status = Errc ordinal + 1
            continue
        tree = _tree_by_name(c["tree_name"], spec)
        assert (tree.kind, tree.mode, tree.parent) == (c["tree"]["kind"], c["tree"]["mode"], c["tree"]["parent"])
        for key, legacy in (("scheme", False), ("legacy", True)):
            want = c[key]
            got = P.optimal_dynamic_scheme(tree, spec, c["procs"], legacy)
            assert got.scheme.root == want["root"], (c["L"], c["K"], c["procs"], key)
            assert [got.scheme.node_grids[i] for i in want["nodes"]] == want["node_grids"]
            assert sorted(got.scheme.node_grids) == want["nodes"]
            assert got.report.total == want["total"]
            assert [got.report.per_node_ttm[i] for i in want["nodes"]] == want["ttm"]
            assert [got.report.per_node_regrid[i] for i in want["nodes"]] == want["regrid"]
            # scheme_volume of the returned scheme reproduces the report
            again = P.scheme_volume(tree, spec, got.scheme, c["procs"])
            assert (again.total, again.per_node_ttm, again.per_node_regrid) == \
                   (got.report.total, got.report.per_node_ttm, got.report.per_node_regrid)
            if "traced_regrid" in want:   # the reference's element-by-element owner comparison (simulate.hpp:104-121)
                cards_in = c["tree"]["card_in"]
                for node, traced in zip(want["nodes"], want["traced_regrid"]):
                    parent = tree.parent[node]
                    pg = got.scheme.root if tree.kind[parent] == P.ROOT else got.scheme.node_grids[parent]
                    ext = list(spec.L)
                    at = parent
                    while at > 0:
                        ext[tree.mode[at]] = spec.K[tree.mode[at]]
                        at = tree.parent[at]
                    if got.scheme.node_grids[node] != pg:
                        assert P.count_moved(ext, pg, got.scheme.node_grids[node]) == traced
                        assert traced <= cards_in[node]
                        regridding += 1
                    else:
                        assert traced == 0
        # a uniform scheme on the best static grid costs what static_volume says
        best = P.optimal_static_grid(tree, spec, c["procs"])
        assert best.report.total == c["static_total"]
        uni = P.scheme_volume(tree, spec, P.uniform_scheme(tree, best.grid), c["procs"])
        assert uni.total == c["static_total"] and not any(uni.per_node_regrid)
        assert c["scheme"]["total"] <= c["static_total"]
    assert regridding >= 20


def test_config4_dynamic_scheme_of_the_survey():
    """C4 at P = 8 is the one configuration where regridding pays: 9 437 184 elements with 3 regrids
    against 11 010 048 on the best static grid."""
    spec = P.ProblemSpec([48] * 5, [8] * 5)
    tree = P.optimal_tree(spec).tree
    r = P.optimal_dynamic_scheme(tree, spec, 8)
    assert r.report.total == 9437184
    assert sum(1 for v in r.report.per_node_regrid if v) == 3
    assert P.optimal_static_grid(tree, spec, 8).report.total == 11010048


def test_scheme_volume_error_codes():
    spec = P.ProblemSpec([6, 5, 4], [3, 2, 2])
    tree = P.optimal_tree(spec).tree
    scheme = P.uniform_scheme(tree, [2, 2, 1])
    del scheme.node_grids[max(scheme.node_grids)]
    with pytest.raises(TuckerplanError) as e:
        P.scheme_volume(tree, spec, scheme, 4)
    assert e.value.code == Errc.missing_assignment             # grid_dynamic.hpp:46-48
    bad = P.uniform_scheme(tree, [2, 2, 1])
    bad.node_grids[min(bad.node_grids)] = [4, 1, 1]            # q_0 = 4 > K_0 = 3
    with pytest.raises(TuckerplanError) as e:
        P.scheme_volume(tree, spec, bad, 4)
    assert e.value.code == Errc.invalid_grid
    with pytest.raises(TuckerplanError) as e:
        P.optimal_dynamic_scheme(tree, P.ProblemSpec([5, 4, 3], [1, 1, 1]), 2)
    assert e.value.code == Errc.no_valid_grid
    assert P.count_moved([6, 5, 4], [2, 2, 1], [2, 2, 1]) == 0
    assert P.count_moved([6, 5, 4], [2, 2, 1], [1, 2, 2]) > 0


def test_count_moved_known_answers():
    """tests/test_simulate.cpp:162-167: the two regrids of the reference's hand-built scenario."""
    assert P.count_moved([8, 8, 16, 64], [1, 1, 1, 64], [8, 8, 1, 1]) == 64512
    assert P.count_moved([16, 16, 8, 64], [1, 1, 1, 64], [2, 4, 8, 1]) == 129024
    # block-overlap counting against an element-by-element owner walk (what the reference does)
    rng = np.random.default_rng(41)
    for _ in range(20):
        ext = [int(rng.integers(2, 8)) for _ in range(3)]
        grids = P.enumerate_grids(int(rng.choice([2, 4, 6, 8])), P.ProblemSpec(ext, ext))
        if len(grids) < 2:
            continue
        a, b = grids[int(rng.integers(0, len(grids)))], grids[int(rng.integers(0, len(grids)))]
        moved = 0
        for idx in np.ndindex(*ext):
            ra = rb = 0
            for m, c in enumerate(idx):
                ra = ra * a[m] + P.block_of(c, ext[m], a[m])
                rb = rb * b[m] + P.block_of(c, ext[m], b[m])
            moved += ra != rb
        assert P.count_moved(ext, a, b) == moved
