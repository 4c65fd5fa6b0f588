"""TEST INFRASTRUCTURE — not part of the product.

Inputs and selections for the CPU arm taken from the REFERENCE's own code: oracle/_ref/libref_shim.so is compiled by
oracle/Makefile from the reference headers where they lie (dense_tensor.hpp, tree_opt.hpp, tree_cost.hpp,
grid_volume.hpp).  `bench.py --impl reference` uses this module so that the reference arm maps no product library:
tree and grid come from the reference planner, the tensor from the reference's `random_tensor` stream, the start
factors from the `random_decomposition` gaussian stream (hooi.hpp:111-120) + the oracle's thin QR.

The recipe is SURVEY.md §8d (config c: seeds 1000c+1 core, +2 generating factors, +3 noise, +4 start factors), the
same one paper_1707_05594_b200/workloads.py follows on the product side.
"""
from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from typing import List, Sequence

import numpy as np

from . import hooi_oracle as ho

_HERE = os.path.dirname(os.path.abspath(__file__))
SHIM_PATH = os.path.join(_HERE, "_ref", "libref_shim.so")

_u64 = ctypes.c_uint64
_dbl_p = ctypes.POINTER(ctypes.c_double)

# BASELINE.json configs: (L, K, sigma, iterations, slab-parallel noise)
CONFIGS = {
    1: ([200] * 3, [20] * 3, 1e-3, 5, False),
    2: ([96] * 4, [10] * 4, 1e-3, 10, False),
    3: ([400, 100, 100, 50], [40, 10, 20, 5], 1e-2, 10, False),
    4: ([48] * 5, [8] * 5, 1e-3, 10, True),
    5: ([1600] * 3, [100] * 3, 1e-3, 5, True),
}


def config_name(index: int) -> str:
    L, K = CONFIGS[index][0], CONFIGS[index][1]
    return "C%d_%s_to_%s" % (index, "x".join(map(str, L)), "x".join(map(str, K)))


_shim = None


def shim() -> ctypes.CDLL:
    global _shim
    if _shim is None:
        if not os.path.exists(SHIM_PATH):
            raise ImportError("%s is missing: build it with `make -C oracle` where /root/reference exists "
                              "(it ships to the GPU box with the snapshot)" % SHIM_PATH)
        _shim = ctypes.CDLL(SHIM_PATH)
    return _shim


def _check(status: int, what: str):
    if status != 0:
        raise RuntimeError("reference %s failed with status %d" % (what, status))


def _u64s(values):
    values = [int(v) for v in values]
    return (_u64 * len(values))(*values)


def _ints(values):
    values = [int(v) for v in values]
    return (ctypes.c_int * len(values))(*values)


def random_tensor(dims: Sequence[int], seed: int, out: np.ndarray | None = None) -> np.ndarray:
    dims = [int(d) for d in dims]
    total = int(np.prod(dims, dtype=np.int64))
    if out is None:
        out = np.empty(total, dtype=np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= total
    _check(shim().ref_random_tensor(len(dims), (ctypes.c_size_t * len(dims))(*dims), _u64(seed),
                                    out.ctypes.data_as(_dbl_p)), "random_tensor")
    return out.reshape(-1)[:total].reshape(dims)


def gaussians(seed: int, count: int) -> np.ndarray:
    out = np.empty(int(count), dtype=np.float64)
    _check(shim().ref_gaussians(_u64(seed), ctypes.c_size_t(int(count)), out.ctypes.data_as(_dbl_p)), "gaussians")
    return out


def orthonormal_factors(L, K, seed: int) -> List[np.ndarray]:
    stream = gaussians(seed, sum(int(l) * int(k) for l, k in zip(L, K)))
    return [np.asfortranarray(f) for f in ho.orthonormal_from_gaussians(L, K, stream)]


def optimal_tree(L, K) -> ho.Tree:
    n, cap = len(L), 4 * len(L) * len(L) + 8
    kind, mode, parent = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_int * cap)()
    count, macs = ctypes.c_int(), _u64()
    _check(shim().ref_optimal_tree(n, _u64s(L), _u64s(K), cap, kind, mode, parent, ctypes.byref(count),
                                   ctypes.byref(macs)), "optimal_tree")
    c = count.value
    return ho.Tree(n, list(kind[:c]), list(mode[:c]), list(parent[:c]))


def tree_label(tree: ho.Tree) -> str:
    """The on-disk label form with 1-based modes (serialize.hpp:54-56), e.g. T(M2(M3(F1)), M1(M3(F2), M2(F3)))."""
    kids = {i: [] for i in range(len(tree.kind))}
    for i, p in enumerate(tree.parent):
        if p >= 0:
            kids[p].append(i)

    def label(i):
        if tree.kind[i] == 2:
            return "F%d" % (tree.mode[i] + 1)
        inner = ", ".join(label(c) for c in kids[i])
        return ("T(%s)" if tree.kind[i] == 0 else "M%d(%%s)" % (tree.mode[i] + 1)) % inner

    return label(0)


def optimal_static_grid(L, K, tree: ho.Tree, procs: int):
    n = len(L)
    q, total = (_u64 * n)(), _u64()
    _check(shim().ref_optimal_static_grid(n, _u64s(L), _u64s(K), len(tree.kind), _ints(tree.kind), _ints(tree.mode),
                                          _ints(tree.parent), _u64(procs), q, ctypes.byref(total)),
           "optimal_static_grid")
    return list(q), int(total.value)


def static_volume(L, K, tree: ho.Tree, q, procs: int) -> int:
    total = _u64()
    _check(shim().ref_static_volume(len(L), _u64s(L), _u64s(K), len(tree.kind), _ints(tree.kind), _ints(tree.mode),
                                    _ints(tree.parent), _u64s(q), _u64(procs), ctypes.byref(total)), "static_volume")
    return int(total.value)


def build_tensor(index: int, threads: int = 8) -> np.ndarray:
    """T = X + sigma E of config `index` on the host, from the reference's streams."""
    L, K, sigma, _, slab_noise = CONFIGS[index]
    t = np.empty(L, dtype=np.float64)
    seed = 1000 * index + 3
    if slab_noise:
        flat = t.reshape(L[0], -1)
        with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:   # the C call releases the GIL
            list(pool.map(lambda i: random_tensor(L[1:], seed + i, flat[i]), range(L[0])))
    else:
        random_tensor(L, seed, t.reshape(-1))
    t *= sigma
    z = random_tensor(K, 1000 * index + 1).copy()
    for n, a in enumerate(orthonormal_factors(L, K, 1000 * index + 2)):
        z = np.moveaxis(np.tensordot(a, z, axes=(1, n)), 0, n)
    t += z
    return t


def start_factors(index: int) -> List[np.ndarray]:
    L, K = CONFIGS[index][0], CONFIGS[index][1]
    return orthonormal_factors(L, K, 1000 * index + 4)
