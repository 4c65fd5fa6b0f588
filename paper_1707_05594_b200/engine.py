"""Device engine: host-side mirror of the reference's dense API (ttm.hpp, hooi.hpp) over the C ABI.

Two levels, as in include/tuckerplan_b200.h:
  * by-value functions with the reference's names and argument meaning (`ttm`, `leading_left_factors`,
    `hooi_sweep`, `reconstruction_error`, `random_decomposition`) — NumPy arrays in, NumPy arrays out, the
    tensor uploaded per call, exactly what the reference signatures imply;
  * handles (`Context`, `DeviceTensor`, `HooiPlan`) that keep the tensor and the factors resident in HBM across
    sweeps — what a caller doing many sweeps should use.

Nothing here computes on the CPU: every call goes to the CUDA library and fails with Errc.cuda without a B200.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from ._lib import TuckerplanError, Errc, check, dbl_p, lib, size_array, u64, u64_array
from .planner import ProblemSpec, TtmTree, validate_spec
from . import hostgen

JACOBI, GAUSS_SEIDEL = 0, 1
_KINDS = {"jacobi": JACOBI, "gauss_seidel": GAUSS_SEIDEL, "gauss-seidel": GAUSS_SEIDEL, JACOBI: JACOBI,
          GAUSS_SEIDEL: GAUSS_SEIDEL}

lib.tp_tensor_device_ptr.restype = ctypes.c_void_p


class _SweepStatsC(ctypes.Structure):
    _fields_ = [("tree_macs", ctypes.c_uint64), ("core_macs", ctypes.c_uint64), ("peak_live", ctypes.c_int),
                ("degenerate", ctypes.c_int)]


class _SweepTimingC(ctypes.Structure):
    _fields_ = [("total_ms", ctypes.c_float), ("tree_ms", ctypes.c_float), ("gram_ms", ctypes.c_float),
                ("evd_ms", ctypes.c_float), ("core_ms", ctypes.c_float)]


@dataclass
class SweepStats:
    """hooi.hpp:125-130."""
    tree_macs: int = 0
    core_macs: int = 0
    peak_live: int = 0
    degenerate: bool = False


@dataclass
class Decomposition:
    """hooi.hpp:78-81: core (extents K, row-major) and factors[n] (L_n x K_n)."""
    core: np.ndarray
    factors: List[np.ndarray]


def _f64(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _colmajor(a: np.ndarray) -> np.ndarray:
    return np.asfortranarray(a, dtype=np.float64)


class Context:
    """One CUDA device + stream + cuSOLVER handle (tp_ctx)."""

    def __init__(self, device: int = 0, flags: int = 0):
        self._h = ctypes.c_void_p()
        check(lib.tp_ctx_create_ex(device, ctypes.c_uint(flags), ctypes.byref(self._h)))

    def set_option(self, option: int, value: int):
        """tp_ctx_set_option: 1 = streamed-upload threshold in bytes, 2 = trace the eigen-solve certificates."""
        check(lib.tp_ctx_set_option(self._h, int(option), ctypes.c_longlong(int(value))))

    def release_cache(self):
        """Frees what by-value hooi_sweep calls keep on the device between calls."""
        check(lib.tp_ctx_release_cache(self._h))

    def close(self):
        if self._h:
            lib.tp_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(lib.tp_ctx_synchronize(self._h))

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(lib.tp_ctx_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def launch_counts(self):
        a, b = u64(), u64()
        check(lib.tp_ctx_launch_counts(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class DeviceTensor:
    """DenseTensor (dense_tensor.hpp:19-30) resident in HBM."""

    def __init__(self, ctx: Context, handle, dims):
        self.ctx, self._h, self.dims = ctx, handle, tuple(int(d) for d in dims)

    @staticmethod
    def upload(ctx: Context, array: np.ndarray) -> "DeviceTensor":
        a = _f64(array)
        h = ctypes.c_void_p()
        check(lib.tp_tensor_upload(ctx._h, a.ndim, size_array(a.shape), a.ctypes.data_as(dbl_p), ctypes.byref(h)))
        return DeviceTensor(ctx, h, a.shape)

    @staticmethod
    def upload_raw(ctx: Context, dims: Sequence[int], host_ptr: int) -> "DeviceTensor":
        h = ctypes.c_void_p()
        check(lib.tp_tensor_upload(ctx._h, len(dims), size_array(dims), ctypes.cast(host_ptr, dbl_p), ctypes.byref(h)))
        return DeviceTensor(ctx, h, dims)

    @staticmethod
    def zeros(ctx: Context, dims: Sequence[int]) -> "DeviceTensor":
        h = ctypes.c_void_p()
        check(lib.tp_tensor_alloc(ctx._h, len(dims), size_array(dims), ctypes.byref(h)))
        return DeviceTensor(ctx, h, dims)

    @property
    def size(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    @property
    def device_ptr(self) -> int:
        return lib.tp_tensor_device_ptr(self._h) or 0

    def download(self) -> np.ndarray:
        out = np.empty(self.dims, dtype=np.float64)
        check(lib.tp_tensor_download(self.ctx._h, self._h, out.ctypes.data_as(dbl_p)))
        return out

    def norm(self) -> float:
        out = ctypes.c_double()
        check(lib.tp_tensor_norm(self.ctx._h, self._h, ctypes.byref(out)))
        return out.value

    def ttm(self, m: np.ndarray, mode: int, macs: Optional[list] = None) -> "DeviceTensor":
        m = _colmajor(m)
        if m.ndim != 2:
            raise TuckerplanError(int(Errc.shape_mismatch), "matrix expected")
        h = ctypes.c_void_p()
        c = u64(macs[0]) if macs is not None else None
        check(lib.tp_ttm(self.ctx._h, self._h, m.ctypes.data_as(dbl_p), ctypes.c_size_t(m.shape[0]),
                         ctypes.c_size_t(m.shape[1]), int(mode), ctypes.byref(c) if c is not None else None,
                         ctypes.byref(h)))
        if macs is not None:
            macs[0] = c.value
        dims = list(self.dims)
        dims[mode] = m.shape[0]
        return DeviceTensor(self.ctx, h, dims)

    def axpby(self, beta: float, alpha: float, x: "DeviceTensor") -> None:
        """self = beta * self + alpha * x (input assembly helper)."""
        check(lib.tp_tensor_axpby(self.ctx._h, self._h, ctypes.c_double(beta), ctypes.c_double(alpha), x._h))

    def download_into(self, host_ptr: int) -> None:
        check(lib.tp_tensor_download(self.ctx._h, self._h, ctypes.cast(host_ptr, dbl_p)))

    def gram(self, mode: int) -> np.ndarray:
        if not 0 <= mode < len(self.dims):
            raise TuckerplanError(int(Errc.bad_mode), "mode out of range", mode)
        rows = self.dims[mode]
        out = np.empty((rows, rows), dtype=np.float64)
        check(lib.tp_gram(self.ctx._h, self._h, int(mode), out.ctypes.data_as(dbl_p)))
        return out

    def leaf_factor(self, mode: int, k: int):
        if not 0 <= mode < len(self.dims):
            raise TuckerplanError(int(Errc.bad_mode), "mode out of range", mode)
        out = np.zeros((self.dims[mode], max(int(k), 0)), dtype=np.float64, order="F")
        deg = ctypes.c_int()
        check(lib.tp_leaf_factor(self.ctx._h, self._h, int(mode), int(k), out.ctypes.data_as(dbl_p), ctypes.byref(deg)))
        return out, bool(deg.value)

    def free(self):
        if self._h:
            lib.tp_tensor_free(self.ctx._h, self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class HooiPlan:
    """hooi_sweep (hooi.hpp:189-229) on a fixed (spec, tree, kind) with everything resident in HBM."""

    def __init__(self, ctx: Context, spec: ProblemSpec, tree: TtmTree, kind="jacobi"):
        self.ctx, self.spec, self.tree = ctx, spec, tree
        if tree.n_modes != spec.n_modes():
            raise TuckerplanError(int(Errc.shape_mismatch), "tree and spec mode counts differ")
        self._h = ctypes.c_void_p()
        n, L, K = spec._c()
        nn, kind_a, mode_a, parent_a = tree._c()
        check(lib.tp_plan_create(ctx._h, n, L, K, nn, kind_a, mode_a, parent_a, _KINDS[kind], ctypes.byref(self._h)))

    def set_overlap_evd(self, on: bool):
        """Jacobi only: eigen-solves on side streams beside the tree (default) or everything serial on one stream."""
        check(lib.tp_plan_set_option(self.ctx._h, self._h, 1, 1 if on else 0))

    def set_fast_evd(self, on: bool):
        """Top-k subspace-iteration eigen-solve on eligible Jacobi leaves (verified; full solve otherwise)."""
        check(lib.tp_plan_set_option(self.ctx._h, self._h, 2, 1 if on else 0))

    def set_carry_path(self, on: bool):
        """Keep the core chain's partial products (they are next sweep's tree nodes along one path) between sweeps."""
        check(lib.tp_plan_set_option(self.ctx._h, self._h, 3, 1 if on else 0))

    def set_option(self, option: int, value: int):
        """tp_plan_set_option: 4/5 spare SMs, 6 whole-sweep graph (0 off, 1 on, 2 auto), 7 leaf graph, 8 one-launch
        leaf solve, 9 forked subtrees (0 off, 1 on, 2 auto)."""
        check(lib.tp_plan_set_option(self.ctx._h, self._h, int(option), int(value)))

    def set_sweep_graph(self, mode: int):
        self.set_option(6, mode)

    def set_fork_subtrees(self, mode: int):
        """TP_OPT_FORK_SUBTREES: sibling subtrees of the TTM tree on streams of their own (0 off, 1 on, 2 auto)."""
        self.set_option(9, mode)

    def sweep_info(self):
        """(last sweep replayed the whole-sweep graph?, leaves on the one-launch solve)."""
        a, b = ctypes.c_int(), ctypes.c_int()
        check(lib.tp_plan_last_sweep_info(self.ctx._h, self._h, ctypes.byref(a), ctypes.byref(b)))
        return bool(a.value), b.value

    def evd_info(self):
        """(leaves eligible for the fast eigen-solve, leaves the last sweep redid with the full solve)."""
        a, b = ctypes.c_int(), ctypes.c_int()
        check(lib.tp_plan_last_evd_info(self.ctx._h, self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def _factor_ptrs(self, arrays):
        return (dbl_p * len(arrays))(*[a.ctypes.data_as(dbl_p) for a in arrays])

    def set_factors(self, factors: Sequence[np.ndarray]):
        if len(factors) != self.spec.n_modes():
            raise TuckerplanError(int(Errc.shape_mismatch), "factor count differs from mode count")
        fs = []
        for f, l, k in zip(factors, self.spec.L, self.spec.K):
            if tuple(f.shape) != (l, k):
                raise TuckerplanError(int(Errc.shape_mismatch), "factor shape differs from L x K")
            fs.append(_colmajor(f))
        check(lib.tp_plan_set_factors(self.ctx._h, self._h, self._factor_ptrs(fs)))

    def get_factors(self) -> List[np.ndarray]:
        outs = [np.zeros((l, k), dtype=np.float64, order="F") for l, k in zip(self.spec.L, self.spec.K)]
        check(lib.tp_plan_get_factors(self.ctx._h, self._h, self._factor_ptrs(outs)))
        return outs

    def init_sthosvd(self, t: DeviceTensor, order: Optional[Sequence[int]] = None):
        """Start factors (and their core) from the sequentially truncated HOSVD of the device tensor."""
        arr = (ctypes.c_int * len(order))(*[int(v) for v in order]) if order is not None else None
        check(lib.tp_plan_init_sthosvd(self.ctx._h, self._h, t._h, arr))

    def get_core(self) -> np.ndarray:
        out = np.empty(tuple(self.spec.K), dtype=np.float64)
        check(lib.tp_plan_get_core(self.ctx._h, self._h, out.ctypes.data_as(dbl_p)))
        return out

    def core_norm(self) -> float:
        out = ctypes.c_double()
        check(lib.tp_plan_core_norm(self.ctx._h, self._h, ctypes.byref(out)))
        return out.value

    def compute_core(self, t: DeviceTensor):
        check(lib.tp_plan_compute_core(self.ctx._h, self._h, t._h))

    def sweep(self, t: DeviceTensor) -> SweepStats:
        st = _SweepStatsC()
        check(lib.tp_plan_sweep(self.ctx._h, self._h, t._h, ctypes.byref(st)))
        return SweepStats(st.tree_macs, st.core_macs, st.peak_live, bool(st.degenerate))

    def last_timing(self) -> dict:
        tm = _SweepTimingC()
        check(lib.tp_plan_last_timing(self.ctx._h, self._h, ctypes.byref(tm)))
        return {"total_ms": tm.total_ms, "tree_ms": tm.tree_ms, "gram_ms": tm.gram_ms, "evd_ms": tm.evd_ms,
                "core_ms": tm.core_ms}

    def node_timing(self):
        """(node_ms, evd_ms) per tree node of the last sweep: TTM launch time for mode nodes, Gram for leaves."""
        nn = len(self.tree.kind)
        a, b = (ctypes.c_float * nn)(), (ctypes.c_float * nn)()
        check(lib.tp_plan_node_timing(self.ctx._h, self._h, nn, a, b))
        return list(a), list(b)

    def reconstruction_error(self, t: DeviceTensor) -> float:
        out = ctypes.c_double()
        check(lib.tp_plan_reconstruction_error(self.ctx._h, self._h, t._h, ctypes.byref(out)))
        return out.value

    def fit_from_norms(self, t: DeviceTensor) -> float:
        out = ctypes.c_double()
        check(lib.tp_plan_fit_from_norms(self.ctx._h, self._h, t._h, ctypes.byref(out)))
        return out.value

    def close(self):
        if self._h:
            lib.tp_plan_destroy(self.ctx._h, self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GridHooi:
    """Jacobi sweeps on a Cartesian processor grid inside this process (tp_grid_*): rank p runs on CUDA device
    devices[p]; naming a device several times gives virtual ranks on one GPU.  `grid` is the root grid, `node_grids`
    (optional, {node id: grid}) a per-node scheme as planner.optimal_dynamic_scheme returns."""

    def __init__(self, spec: ProblemSpec, tree: TtmTree, grid: Sequence[int], devices: Sequence[int],
                 node_grids=None, use_nccl: bool = False):
        self.spec, self.tree = spec, tree
        n, L, K = spec._c()
        nn, kind_a, mode_a, parent_a = tree._c()
        self._nn = nn
        ng = None
        if node_grids is not None:
            flat = [0] * (nn * n)
            for node, g in node_grids.items():
                flat[node * n:(node + 1) * n] = [int(v) for v in g]
            ng = u64_array(flat)
        self._h = ctypes.c_void_p()
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        check(lib.tp_grid_create(len(devices), devs, n, L, K, nn, kind_a, mode_a, parent_a, u64_array(grid), ng,
                                 ctypes.c_uint(1 if use_nccl else 0), ctypes.byref(self._h)))

    def set_tensor(self, t: np.ndarray):
        t = _f64(t)
        _check_engine_shapes(t, self.spec)
        check(lib.tp_grid_set_tensor(self._h, t.ctypes.data_as(dbl_p)))

    def block(self, rank: int):
        n = self.spec.n_modes()
        lo, dims = (ctypes.c_size_t * n)(), (ctypes.c_size_t * n)()
        check(lib.tp_grid_block(self._h, int(rank), lo, dims))
        return list(lo), list(dims)

    def set_factors(self, factors: Sequence[np.ndarray]):
        fs = [_colmajor(f) for f in factors]
        check(lib.tp_grid_set_factors(self._h, (dbl_p * len(fs))(*[a.ctypes.data_as(dbl_p) for a in fs])))

    def get_factors(self) -> List[np.ndarray]:
        outs = [np.zeros((l, k), dtype=np.float64, order="F") for l, k in zip(self.spec.L, self.spec.K)]
        check(lib.tp_grid_get_factors(self._h, (dbl_p * len(outs))(*[a.ctypes.data_as(dbl_p) for a in outs])))
        return outs

    def sweep(self) -> SweepStats:
        st = _SweepStatsC()
        check(lib.tp_grid_sweep(self._h, ctypes.byref(st)))
        return SweepStats(st.tree_macs, st.core_macs, st.peak_live, bool(st.degenerate))

    def get_core(self) -> np.ndarray:
        out = np.empty(tuple(self.spec.K), dtype=np.float64)
        check(lib.tp_grid_get_core(self._h, out.ctypes.data_as(dbl_p)))
        return out

    def norms(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        check(lib.tp_grid_norms(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def fit_from_norms(self) -> float:
        out = ctypes.c_double()
        check(lib.tp_grid_fit_from_norms(self._h, ctypes.byref(out)))
        return out.value

    def last_volumes(self):
        a, b = (ctypes.c_uint64 * self._nn)(), (ctypes.c_uint64 * self._nn)()
        check(lib.tp_grid_last_volumes(self._h, self._nn, a, b))
        return list(a), list(b)

    def last_timing(self):
        total, fast = ctypes.c_float(), ctypes.c_int()
        per = (ctypes.c_float * self._nn)()
        check(lib.tp_grid_last_timing(self._h, ctypes.byref(total), self._nn, per, ctypes.byref(fast)))
        return total.value, list(per), fast.value

    def launch_counts(self):
        a, b = u64(), u64()
        check(lib.tp_grid_launch_counts(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self):
        if self._h:
            lib.tp_grid_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ by-value API (reference signatures)
def ttm(t: np.ndarray, m: np.ndarray, mode: int, macs: Optional[list] = None, ctx: Optional[Context] = None):
    """ttm(t, m, mode, macs*) — ttm.hpp:73-96."""
    ctx = ctx or default_context()
    dt = DeviceTensor.upload(ctx, t)
    try:
        out = dt.ttm(m, mode, macs)
        try:
            return out.download()
        finally:
            out.free()
    finally:
        dt.free()


def leading_left_factors(m: np.ndarray, k: int, ctx: Optional[Context] = None):
    """leading_left_factors(m, k) — hooi.hpp:45-76.  Returns (vectors rows x k, degenerate)."""
    ctx = ctx or default_context()
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2:
        m = m.reshape(m.shape[0] if m.ndim else 0, -1) if m.size else np.zeros((0, 0))
    mf = _colmajor(m)
    rows, cols = mf.shape
    out = np.zeros((rows, max(int(k), 0)), dtype=np.float64, order="F")
    deg = ctypes.c_int()
    check(lib.tp_leading_left_factors(ctx._h, mf.ctypes.data_as(dbl_p), ctypes.c_size_t(rows), ctypes.c_size_t(cols),
                                      int(k), out.ctypes.data_as(dbl_p), ctypes.byref(deg)))
    return out, bool(deg.value)


def _check_engine_shapes(t: np.ndarray, s: ProblemSpec):
    if t.ndim != s.n_modes():
        raise TuckerplanError(int(Errc.shape_mismatch), "tensor and spec mode counts differ")
    for m in range(t.ndim):
        if t.shape[m] != s.L[m]:
            raise TuckerplanError(int(Errc.shape_mismatch), "tensor extent differs from L", m)


def hooi_sweep(t: np.ndarray, s: ProblemSpec, d: Decomposition, tree: TtmTree, kind="jacobi",
               stats: Optional[SweepStats] = None, ctx: Optional[Context] = None,
               tensor_unchanged: bool = False) -> Decomposition:
    """hooi_sweep(t, s, d, tree, kind, stats*) — hooi.hpp:189-229, by value through tp_hooi_sweep_host_ex.
    tensor_unchanged: the caller's promise that `t` (same buffer) is what the previous call uploaded; the device
    copy is then reused (TP_HOST_TENSOR_UNCHANGED)."""
    ctx = ctx or default_context()
    t = _f64(t)
    _check_engine_shapes(t, s)
    if tree.n_modes != s.n_modes():
        raise TuckerplanError(int(Errc.shape_mismatch), "tree and spec mode counts differ")
    # validate_tree precedes the factor-count check in the reference (hooi.hpp:193-195)
    from .planner import validate_tree
    validate_tree(tree, s)
    if len(d.factors) != s.n_modes():
        raise TuckerplanError(int(Errc.shape_mismatch), "factor count differs from mode count")
    fin = [_colmajor(f) for f in d.factors]
    fout = [np.zeros((l, k), dtype=np.float64, order="F") for l, k in zip(s.L, s.K)]
    core = np.empty(tuple(s.K), dtype=np.float64)
    st = _SweepStatsC()
    nn, kind_a, mode_a, parent_a = tree._c()
    n = s.n_modes()
    check(lib.tp_hooi_sweep_host_ex(ctx._h, n, size_array(t.shape), t.ctypes.data_as(dbl_p), u64_array(s.K),
                                    (dbl_p * n)(*[a.ctypes.data_as(dbl_p) for a in fin]), nn, kind_a, mode_a,
                                    parent_a, _KINDS[kind], ctypes.c_uint(1 if tensor_unchanged else 0),
                                    (dbl_p * n)(*[a.ctypes.data_as(dbl_p) for a in fout]),
                                    core.ctypes.data_as(dbl_p), ctypes.byref(st)))
    if stats is not None:
        stats.tree_macs, stats.core_macs = st.tree_macs, st.core_macs
        stats.peak_live, stats.degenerate = st.peak_live, bool(st.degenerate)
    return Decomposition(core, fout)


def core_from_factors(t: np.ndarray, factors: Sequence[np.ndarray], ctx: Optional[Context] = None) -> np.ndarray:
    """detail::core_from_factors — hooi.hpp:93-100."""
    ctx = ctx or default_context()
    dt = DeviceTensor.upload(ctx, t)
    try:
        cur = dt
        for n, f in enumerate(factors):
            nxt = cur.ttm(np.asarray(f).T, n)
            if cur is not dt:
                cur.free()
            cur = nxt
        out = cur.download()
        if cur is not dt:
            cur.free()
        return out
    finally:
        dt.free()


def random_decomposition(t: np.ndarray, s: ProblemSpec, seed: int, ctx: Optional[Context] = None) -> Decomposition:
    """random_decomposition(t, s, seed) — hooi.hpp:106-123."""
    validate_spec(s)
    t = _f64(t)
    _check_engine_shapes(t, s)
    factors = hostgen.random_orthonormal_factors(s.L, s.K, seed)
    return Decomposition(core_from_factors(t, factors, ctx), factors)


def sthosvd(t: np.ndarray, s: ProblemSpec, order: Optional[Sequence[int]] = None, ctx: Optional[Context] = None):
    """Sequentially truncated HOSVD start (tp_sthosvd; no reference counterpart, see the header).  Returns
    (Decomposition, degenerate)."""
    ctx = ctx or default_context()
    validate_spec(s)
    t = _f64(t)
    _check_engine_shapes(t, s)
    dt = DeviceTensor.upload(ctx, t)
    try:
        n = s.n_modes()
        fout = [np.zeros((l, k), dtype=np.float64, order="F") for l, k in zip(s.L, s.K)]
        core = np.empty(tuple(s.K), dtype=np.float64)
        deg = ctypes.c_int()
        arr = (ctypes.c_int * n)(*[int(v) for v in order]) if order is not None else None
        check(lib.tp_sthosvd(ctx._h, dt._h, u64_array(s.K), arr, (dbl_p * n)(*[a.ctypes.data_as(dbl_p) for a in fout]),
                             core.ctypes.data_as(dbl_p), ctypes.byref(deg), None))
        return Decomposition(core, fout), bool(deg.value)
    finally:
        dt.free()


def reconstruction_error(t: np.ndarray, d: Decomposition, ctx: Optional[Context] = None) -> float:
    """reconstruction_error(t, d) — hooi.hpp:232-245."""
    ctx = ctx or default_context()
    t = _f64(t)
    dt = DeviceTensor.upload(ctx, t)
    try:
        out = ctypes.c_double()
        n = t.ndim
        if d.core is None or len(d.factors) != n or np.ndim(d.core) != n:
            # the reference evaluates the norm first (zero_tensor), then fails on the shape
            if dt.norm() == 0.0:
                raise TuckerplanError(int(Errc.zero_tensor), "relative error undefined at zero")
            raise TuckerplanError(int(Errc.shape_mismatch), "reconstruction shape differs")
        core = _f64(d.core)
        fs = [_colmajor(f) for f in d.factors]
        for m, f in enumerate(fs):
            if f.shape != (t.shape[m], core.shape[m]):
                if dt.norm() == 0.0:
                    raise TuckerplanError(int(Errc.zero_tensor), "relative error undefined at zero")
                raise TuckerplanError(int(Errc.shape_mismatch), "reconstruction shape differs")
        check(lib.tp_reconstruction_error(ctx._h, dt._h, size_array(core.shape), core.ctypes.data_as(dbl_p),
                                          (dbl_p * n)(*[a.ctypes.data_as(dbl_p) for a in fs]), ctypes.byref(out)))
        return out.value
    finally:
        dt.free()
