"""Seeded host inputs with the reference's streams (dense_tensor.hpp:43-49, hooi.hpp:109-120)."""
from __future__ import annotations

import ctypes
from typing import List, Sequence

import numpy as np

from ._lib import check, dbl_p, lib, size_array, u64, u64_array


def random_tensor(dims: Sequence[int], seed: int, out: np.ndarray | None = None) -> np.ndarray:
    """random_tensor(dims, seed): i.i.d. N(0,1) in storage order."""
    dims = [int(d) for d in dims]
    total = int(np.prod(dims, dtype=np.int64)) if dims else 0
    if out is None:
        out = np.empty(max(total, 0), dtype=np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= total
    check(lib.tp_random_tensor(len(dims), size_array(dims), u64(seed), out.ctypes.data_as(dbl_p)))
    return out[:total].reshape(dims)


def random_orthonormal_factors(L: Sequence[int], K: Sequence[int], seed: int) -> List[np.ndarray]:
    """The factors of random_decomposition(t, spec, seed); each returned array is L_n x K_n (Fortran order,
    i.e. the column-major Eigen::MatrixXd of the reference)."""
    n = len(L)
    outs = [np.zeros((int(l), int(k)), dtype=np.float64, order="F") for l, k in zip(L, K)]
    ptrs = (dbl_p * n)(*[o.ctypes.data_as(dbl_p) for o in outs])
    check(lib.tp_random_orthonormal_factors(n, u64_array(L), u64_array(K), u64(seed), ptrs))
    return outs


def frobenius_norm(t: np.ndarray) -> float:
    t = np.ascontiguousarray(t, dtype=np.float64)
    out = ctypes.c_double()
    check(lib.tp_frobenius_norm_host(ctypes.c_size_t(t.size), t.ctypes.data_as(dbl_p), ctypes.byref(out)))
    return out.value
