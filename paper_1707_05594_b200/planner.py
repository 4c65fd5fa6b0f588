"""Host planner, mirroring the reference's planner API names over the C ABI.

Reference: proj/include/tuckerplan/{problem,ttm_tree,tree_cost,tree_opt,tree_builders,grid,grid_volume}.hpp.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence

from ._lib import Errc, TuckerplanError, check, int_array, lib, u64, u64_array

ROOT, MODE, LEAF = 0, 1, 2
CHAIN_INPUT, CHAIN_BY_COST, CHAIN_BY_RATIO = 0, 1, 2
STRATEGIES = {"chain-input": 0, "chain-k": 1, "chain-h": 2, "balanced": 3, "opt": 4}  # bench.hpp:117-126


@dataclass
class ProblemSpec:
    """problem.hpp:24-29."""
    L: List[int]
    K: List[int]

    def n_modes(self) -> int:
        return len(self.L)

    def _c(self):
        return len(self.L), u64_array(self.L), u64_array(self.K)


@dataclass
class TtmTree:
    """ttm_tree.hpp:36-57 as flat arrays (parent-first; children in stored order)."""
    n_modes: int
    kind: List[int]
    mode: List[int]
    parent: List[int]
    children: List[List[int]] = field(default_factory=list)

    def __post_init__(self):
        self.children = [[] for _ in self.kind]
        for i, p in enumerate(self.parent):
            if 0 <= p < len(self.kind) and p != i:
                self.children[p].append(i)

    def _c(self):
        return len(self.kind), int_array(self.kind), int_array(self.mode), int_array(self.parent)

    def label(self, node: int = 0) -> str:
        """serialize.hpp:50-66 labels: T, M<i>, F<i> (1-based)."""
        k = self.kind[node]
        name = "T" if k == ROOT else ("M%d" % (self.mode[node] + 1) if k == MODE else "F%d" % (self.mode[node] + 1))
        kids = self.children[node]
        return name + ("(" + ", ".join(self.label(c) for c in kids) + ")" if kids else "")


def _same_modes(t: "TtmTree", s: ProblemSpec) -> None:
    """ttm_tree.hpp:104-105: the tree carries its own mode count."""
    if t.n_modes != s.n_modes():
        raise TuckerplanError(int(Errc.shape_mismatch), "tree and spec mode counts differ")


def validate_spec(s: ProblemSpec) -> None:
    n, L, K = s._c()
    check(lib.tp_validate_spec(n, L, K))


def partial_cardinality(s: ProblemSpec, done_mask: int) -> int:
    n, L, K = s._c()
    out = u64()
    check(lib.tp_partial_cardinality(n, L, K, ctypes.c_uint32(done_mask), ctypes.byref(out)))
    return out.value


def _tree_out(fn, s: ProblemSpec, *extra):
    n, L, K = s._c()
    cap = 4096
    kind, mode, parent = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_int * cap)()
    count = ctypes.c_int()
    check(fn(n, L, K, *extra, cap, kind, mode, parent, ctypes.byref(count)))
    c = count.value
    return TtmTree(n, list(kind[:c]), list(mode[:c]), list(parent[:c]))


@dataclass
class OptimalTreeResult:
    tree: TtmTree
    total_macs: int
    dp_states: int


def optimal_tree(s: ProblemSpec) -> OptimalTreeResult:
    """tree_opt.hpp:126-138."""
    n, L, K = s._c()
    cap = 4096
    kind, mode, parent = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_int * cap)()
    count, macs, states = ctypes.c_int(), u64(), u64()
    check(lib.tp_optimal_tree(n, L, K, cap, kind, mode, parent, ctypes.byref(count), ctypes.byref(macs),
                              ctypes.byref(states)))
    c = count.value
    return OptimalTreeResult(TtmTree(n, list(kind[:c]), list(mode[:c]), list(parent[:c])), macs.value, states.value)


def optimal_cost_reuse_greedy(s: ProblemSpec) -> int:
    n, L, K = s._c()
    out = u64()
    check(lib.tp_reuse_greedy_cost(n, L, K, ctypes.byref(out)))
    return out.value


def chain_tree(s: ProblemSpec, order: int = CHAIN_INPUT) -> TtmTree:
    return _tree_out(lib.tp_chain_tree, s, order)


def balanced_tree(s: ProblemSpec) -> TtmTree:
    return _tree_out(lib.tp_balanced_tree, s)


def build_tree(s: ProblemSpec, strategy) -> TtmTree:
    if isinstance(strategy, str):
        strategy = STRATEGIES[strategy]
    return _tree_out(lib.tp_build_tree, s, strategy)


def validate_tree(t: TtmTree, s: ProblemSpec) -> None:
    n, L, K = s._c()
    _same_modes(t, s)
    nn, kind, mode, parent = t._c()
    check(lib.tp_validate_tree(n, L, K, nn, kind, mode, parent))


def is_canonical(t: TtmTree) -> bool:
    nn, kind, mode, parent = t._c()
    out = ctypes.c_int()
    check(lib.tp_tree_is_canonical(nn, kind, mode, parent, ctypes.byref(out)))
    return bool(out.value)


def canonicalize(t: TtmTree) -> TtmTree:
    nn, kind, mode, parent = t._c()
    cap = 4096
    ok, om, op = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_int * cap)()
    count = ctypes.c_int()
    check(lib.tp_canonicalize(t.n_modes, nn, kind, mode, parent, cap, ok, om, op, ctypes.byref(count)))
    c = count.value
    return TtmTree(t.n_modes, list(ok[:c]), list(om[:c]), list(op[:c]))


def tree_depth(t: TtmTree) -> int:
    nn, kind, mode, parent = t._c()
    out = ctypes.c_int()
    check(lib.tp_tree_depth(nn, kind, mode, parent, ctypes.byref(out)))
    return out.value


@dataclass
class CostReport:
    """tree_cost.hpp:43-48 plus NodeCards (:20-23)."""
    total_macs: int
    per_node_macs: List[int]
    n_internal: int
    depth: int
    card_in: List[int]
    card_out: List[int]


def tree_cost(t: TtmTree, s: ProblemSpec) -> CostReport:
    n, L, K = s._c()
    nn, kind, mode, parent = t._c()
    total, ni, depth = u64(), ctypes.c_int(), ctypes.c_int()
    per, cin, cout = (u64 * nn)(), (u64 * nn)(), (u64 * nn)()
    _same_modes(t, s)
    check(lib.tp_tree_cost(n, L, K, nn, kind, mode, parent, ctypes.byref(total), per, cin, cout, ctypes.byref(ni),
                           ctypes.byref(depth)))
    return CostReport(total.value, list(per), ni.value, depth.value, list(cin), list(cout))


def node_cardinalities(t: TtmTree, s: ProblemSpec):
    c = tree_cost(t, s)
    return c.card_in, c.card_out


def grid_count(procs: int, n_modes: int) -> int:
    out = u64()
    check(lib.tp_grid_count(u64(procs), n_modes, ctypes.byref(out)))
    return out.value


def validate_grid(q: Sequence[int], s: ProblemSpec, procs: int) -> None:
    n, L, K = s._c()
    if len(q) != n:
        raise TuckerplanError(int(Errc.invalid_grid), "grid and spec mode counts differ")
    check(lib.tp_validate_grid(n, L, K, u64_array(q), u64(procs)))


def enumerate_grids(procs: int, s: ProblemSpec) -> List[List[int]]:
    n, L, K = s._c()
    count = ctypes.c_size_t()
    cap = 1 << 16
    buf = (u64 * (cap * n))()
    check(lib.tp_enumerate_grids(n, L, K, u64(procs), ctypes.c_size_t(cap), buf, ctypes.byref(count)))
    return [list(buf[i * n:(i + 1) * n]) for i in range(count.value)]


def block_bounds(length: int, parts: int) -> List[int]:
    cuts = (u64 * (parts + 1))()
    check(lib.tp_block_bounds(u64(length), u64(parts), cuts))
    return list(cuts)


def block_of(c: int, length: int, parts: int) -> int:
    out = u64()
    check(lib.tp_block_of(u64(c), u64(length), u64(parts), ctypes.byref(out)))
    return out.value


@dataclass
class VolumeReport:
    total: int
    per_node: List[int]  # indexed by node id; 0 for root and leaves


def static_volume(t: TtmTree, s: ProblemSpec, q: Sequence[int], procs: int) -> VolumeReport:
    n, L, K = s._c()
    nn, kind, mode, parent = t._c()
    total, per = u64(), (u64 * nn)()
    check(lib.tp_static_volume(n, L, K, nn, kind, mode, parent, u64_array(q), u64(procs), ctypes.byref(total), per))
    return VolumeReport(total.value, list(per))


@dataclass
class StaticGridResult:
    grid: List[int]
    report: VolumeReport


def optimal_static_grid(t: TtmTree, s: ProblemSpec, procs: int, threads: int = 1) -> StaticGridResult:
    n, L, K = s._c()
    nn, kind, mode, parent = t._c()
    q, total, per = (u64 * n)(), u64(), (u64 * nn)()
    check(lib.tp_optimal_static_grid(n, L, K, nn, kind, mode, parent, u64(procs), threads, q, ctypes.byref(total),
                                     per))
    return StaticGridResult(list(q), VolumeReport(total.value, list(per)))


# ---- per-node grids (grid_dynamic.hpp) ---------------------------------------------------------------------
@dataclass
class DynamicGridScheme:
    """grid_dynamic.hpp:32-35: the root's anchor grid + one grid per TTM node (node id -> grid)."""
    root: List[int]
    node_grids: dict


@dataclass
class SchemeVolumeReport:
    total: int
    per_node_ttm: List[int]      # indexed by node id, 0 for root / leaves
    per_node_regrid: List[int]


@dataclass
class DynamicSchemeResult:
    scheme: DynamicGridScheme
    report: SchemeVolumeReport


def uniform_scheme(t: TtmTree, q: Sequence[int]) -> DynamicGridScheme:
    """simulate.hpp:53-61: one grid everywhere."""
    return DynamicGridScheme(list(q), {i: list(q) for i in range(len(t.kind)) if t.kind[i] == MODE})


def _scheme_arrays(t: TtmTree, n: int, scheme: DynamicGridScheme):
    nn = len(t.kind)
    flat = (u64 * (nn * n))()
    for node, grid in scheme.node_grids.items():
        if not 0 <= node < nn or len(grid) != n:
            raise ValueError("scheme entry does not fit the tree")
        for m in range(n):
            flat[node * n + m] = int(grid[m])
    return (u64 * n)(*[int(v) for v in scheme.root]), flat


def scheme_volume(t: TtmTree, s: ProblemSpec, scheme: DynamicGridScheme, procs: int) -> SchemeVolumeReport:
    """grid_dynamic.hpp:37-62."""
    n, L, K = s._c()
    nn, kind, mode, parent = t._c()
    if len(scheme.root) != n:
        raise ValueError("root grid does not fit the spec")
    for node in range(nn):
        if t.kind[node] == MODE and node not in scheme.node_grids:
            raise TuckerplanError(int(Errc.missing_assignment), "no grid for internal node %d" % node)
    root, flat = _scheme_arrays(t, n, scheme)
    total, ttm, regrid = u64(), (u64 * nn)(), (u64 * nn)()
    check(lib.tp_scheme_volume(n, L, K, nn, kind, mode, parent, root, flat, u64(procs), ctypes.byref(total), ttm,
                               regrid))
    return SchemeVolumeReport(total.value, list(ttm), list(regrid))


def optimal_dynamic_scheme(t: TtmTree, s: ProblemSpec, procs: int, legacy_regrid_target: bool = False
                           ) -> DynamicSchemeResult:
    """grid_dynamic.hpp:141-167."""
    n, L, K = s._c()
    nn, kind, mode, parent = t._c()
    root, flat = (u64 * n)(), (u64 * (nn * n))()
    total, ttm, regrid = u64(), (u64 * nn)(), (u64 * nn)()
    check(lib.tp_optimal_dynamic_scheme(n, L, K, nn, kind, mode, parent, u64(procs), 1 if legacy_regrid_target else 0,
                                        root, flat, ctypes.byref(total), ttm, regrid))
    grids = {i: [flat[i * n + m] for m in range(n)] for i in range(nn) if t.kind[i] == MODE}
    return DynamicSchemeResult(DynamicGridScheme(list(root), grids),
                               SchemeVolumeReport(total.value, list(ttm), list(regrid)))


def count_moved(ext: Sequence[int], from_grid: Sequence[int], to_grid: Sequence[int]) -> int:
    """simulate.hpp:104-121: elements whose owner rank differs between the two grids."""
    n = len(ext)
    out = u64()
    check(lib.tp_count_moved(n, (u64 * n)(*map(int, ext)), (u64 * n)(*map(int, from_grid)),
                             (u64 * n)(*map(int, to_grid)), ctypes.byref(out)))
    return out.value
