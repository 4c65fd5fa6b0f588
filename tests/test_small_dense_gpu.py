"""The single-launch small dense kernels of the top-k eigen-solve (csrc/evd_kernels.cu) against NumPy, through the
C ABI (tp_dev_cholesky / tp_dev_trsm_right_lt / tp_dev_jacobi_eig).  These replace, for the HOOI leaves, parts of what
the reference gets from Eigen's SelfAdjointEigenSolver (hooi.hpp:55); the bar is rounding-level agreement."""
import ctypes

import numpy as np
import pytest

from paper_1707_05594_b200 import Errc, TuckerplanError
from paper_1707_05594_b200._lib import check, lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_1707_05594_b200 import engine as E
    ctx = E.Context(0)

    class Dev:
        def __init__(self):
            self.ctx = ctx
            self.torch = torch

        def up(self, a, dtype=None):
            t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
            torch.cuda.synchronize()
            return t

        def ptr(self, t, ctype=ctypes.c_double):
            return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctype))

        def down(self, t):
            ctx.synchronize()
            return t.cpu().numpy()

    yield Dev()
    ctx.close()


def colmajor(a):
    return np.asfortranarray(a).ravel(order="F")


def spd(rng, b, cond):
    q, _ = np.linalg.qr(rng.standard_normal((b, b)))
    lam = np.logspace(0, -np.log10(cond), b)
    s = (q * lam) @ q.T
    return (s + s.T) / 2


BLOCKS = [1, 2, 3, 9, 13, 16, 18, 28, 29, 48, 64, 77, 108, 111, 112]


@pytest.mark.parametrize("b", BLOCKS)
def test_cholesky_matches_numpy(dev, b):
    rng = np.random.default_rng(b)
    s = spd(rng, b, 1e6)
    d_s, d_l = dev.up(colmajor(s)), dev.up(np.full(b * b, np.nan))
    d_fail = dev.up(np.zeros(2, dtype=np.int32))
    check(lib.tp_dev_cholesky(dev.ctx._h, dev.ptr(d_s), b, dev.ptr(d_l), dev.ptr(d_fail, ctypes.c_int)))
    l = dev.down(d_l).reshape(b, b, order="F")
    assert dev.down(d_fail)[0] == 0
    ref = np.linalg.cholesky(s)
    assert np.all(np.triu(l, 1) == 0.0)
    assert np.max(np.abs(l - ref)) <= 1e-10 * np.max(np.abs(ref))     # cond 1e6 * eps
    assert np.max(np.abs(l @ l.T - s)) <= 8 * b * np.finfo(float).eps * np.max(np.abs(s))


def test_cholesky_flags_indefinite_matrix(dev):
    rng = np.random.default_rng(5)
    b = 20
    s = spd(rng, b, 10.0)
    s -= 0.5 * np.eye(b)                                               # eigenvalues 0.1..1 shifted below zero
    d_s, d_l = dev.up(colmajor(s)), dev.up(np.zeros(b * b))
    d_fail = dev.up(np.zeros(2, dtype=np.int32))
    check(lib.tp_dev_cholesky(dev.ctx._h, dev.ptr(d_s), b, dev.ptr(d_l), dev.ptr(d_fail, ctypes.c_int)))
    assert dev.down(d_fail)[0] == 1
    assert np.all(np.isfinite(dev.down(d_l)))


@pytest.mark.parametrize("rows,b", [(1, 1), (5, 3), (33, 13), (48, 16), (96, 18), (200, 28), (257, 29), (400, 48),
                                    (1600, 108), (2048, 112), (31, 111)])
def test_trsm_makes_cholesky_qr(dev, rows, b):
    rng = np.random.default_rng(rows * 131 + b)
    z = rng.standard_normal((rows, b)) @ np.diag(np.logspace(0, -3, b))
    l = np.linalg.cholesky(z.T @ z + 1e-30 * np.eye(b)) if rows >= b else np.linalg.cholesky(spd(rng, b, 100.0))
    d_z, d_l = dev.up(colmajor(z)), dev.up(colmajor(l))
    check(lib.tp_dev_trsm_right_lt(dev.ctx._h, dev.ptr(d_z), ctypes.c_size_t(rows), b, dev.ptr(d_l)))
    got = dev.down(d_z).reshape(rows, b, order="F")
    import scipy.linalg as sl
    ref = sl.solve_triangular(l, z.T, lower=True).T                     # Z L^{-T}
    assert np.max(np.abs(got - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1.0)
    # backward check, independent of conditioning: got L^T = Z
    assert np.max(np.abs(got @ l.T - z)) <= 64 * b * np.finfo(float).eps * np.max(np.abs(z)) * max(1.0, np.max(np.abs(got)))
    if rows >= b:
        assert np.max(np.abs(got.T @ got - np.eye(b))) < 1e-6           # one Cholesky-QR pass at cond 1e3


@pytest.mark.parametrize("b", BLOCKS)
def test_jacobi_eig_matches_numpy(dev, b):
    rng = np.random.default_rng(1000 + b)
    k = max(1, b - 8)
    q, _ = np.linalg.qr(rng.standard_normal((b, b)))
    lam = np.concatenate([1.0 + 5.0 * rng.random(k), 1e-6 * rng.random(b - k)])    # signal block + noise floor
    h = (q * lam) @ q.T
    h = (h + h.T) / 2
    d_h = dev.up(colmajor(h))
    d_w, d_v = dev.up(np.full(b, np.nan)), dev.up(np.full(b * b, np.nan))
    d_fail = dev.up(np.zeros(2, dtype=np.int32))
    check(lib.tp_dev_jacobi_eig(dev.ctx._h, dev.ptr(d_h), b, dev.ptr(d_w), dev.ptr(d_v), dev.ptr(d_fail, ctypes.c_int)))
    w = dev.down(d_w)
    v = dev.down(d_v).reshape(b, b, order="F")
    fail = dev.down(d_fail)
    assert fail[0] == 0 and fail[1] <= 12, fail
    ref = np.linalg.eigvalsh(h)
    scale = np.max(np.abs(ref))
    assert np.all(np.diff(w) >= 0)
    assert np.max(np.abs(w - ref)) <= 4 * b * np.finfo(float).eps * scale
    assert np.max(np.abs(v.T @ v - np.eye(b))) <= 4 * b * np.finfo(float).eps
    assert np.max(np.abs(h @ v - v * w)) <= 8 * b * np.finfo(float).eps * scale


def test_jacobi_eig_diagonal_and_repeated(dev):
    b = 12
    h = np.diag([3.0, 1.0, 2.0, 2.0, 5.0, 0.0, 1.0, 4.0, 2.0, 9.0, 7.0, 1.0])
    d_h = dev.up(colmajor(h))
    d_w, d_v = dev.up(np.zeros(b)), dev.up(np.zeros(b * b))
    d_fail = dev.up(np.zeros(2, dtype=np.int32))
    check(lib.tp_dev_jacobi_eig(dev.ctx._h, dev.ptr(d_h), b, dev.ptr(d_w), dev.ptr(d_v), dev.ptr(d_fail, ctypes.c_int)))
    w = dev.down(d_w)
    v = dev.down(d_v).reshape(b, b, order="F")
    assert list(dev.down(d_fail)) == [0, 0]                             # already diagonal: no sweep
    assert np.array_equal(w, np.sort(np.diag(h)))
    assert np.array_equal(np.abs(v).sum(axis=0), np.ones(b)) and np.array_equal(h @ v, v * w)   # a permutation


def test_small_dense_argument_checks(dev):
    t = dev.up(np.zeros(4))
    f = dev.up(np.zeros(2, dtype=np.int32))
    for block in (0, 113):
        with pytest.raises(TuckerplanError) as e:
            check(lib.tp_dev_cholesky(dev.ctx._h, dev.ptr(t), block, dev.ptr(t), dev.ptr(f, ctypes.c_int)))
        assert e.value.code == Errc.bad_argument
        with pytest.raises(TuckerplanError) as e:
            check(lib.tp_dev_jacobi_eig(dev.ctx._h, dev.ptr(t), block, dev.ptr(t), dev.ptr(t), dev.ptr(f, ctypes.c_int)))
        assert e.value.code == Errc.bad_argument
    with pytest.raises(TuckerplanError) as e:
        check(lib.tp_dev_trsm_right_lt(dev.ctx._h, None, ctypes.c_size_t(4), 2, dev.ptr(t)))
    assert e.value.code == Errc.bad_argument


def test_async_leaf_solve_pair(dev):
    """tp_dev_leaf_solve_begin / _finish: the solve runs on a side stream; both routes (full solve without a start
    block, certified top-k with one) give the leading eigenvectors with the reference's sign rule (hooi.hpp:60-68)."""
    torch = dev.torch
    rng = np.random.default_rng(11)
    rows, k = 96, 7
    q, _ = np.linalg.qr(rng.standard_normal((rows, rows)))
    lam = np.concatenate([1.0 + 4.0 * rng.random(k), 1e-6 * rng.random(rows - k)])
    gram = (q * lam) @ q.T
    gram = (gram + gram.T) / 2
    w, v = np.linalg.eigh(gram)
    want = v[:, ::-1][:, :k]
    for col in range(k):
        if want[np.argmax(np.abs(want[:, col])), col] < 0:
            want[:, col] = -want[:, col]
    start = want + 1e-3 * rng.standard_normal(want.shape)
    int_p = ctypes.POINTER(ctypes.c_int)
    for lane, use_start in ((0, False), (1, True), (3, True)):
        d_gram = dev.up(colmajor(gram))
        d_start = dev.up(colmajor(np.linalg.qr(start)[0]))
        d_factor = dev.up(np.zeros(rows * k))
        d_status = dev.up(np.zeros(2, dtype=np.int32))
        flag = ctypes.cast(d_status.data_ptr(), int_p)
        info = ctypes.cast(d_status.data_ptr() + 4, int_p)
        check(lib.tp_dev_leaf_solve_begin(dev.ctx._h, dev.ptr(d_gram), ctypes.c_size_t(rows), k,
                                          dev.ptr(d_start) if use_start else None, dev.ptr(d_factor), flag, info, lane))
        with pytest.raises(TuckerplanError) as e:      # one solve in flight per lane
            check(lib.tp_dev_leaf_solve_begin(dev.ctx._h, dev.ptr(d_gram), ctypes.c_size_t(rows), k, None,
                                              dev.ptr(d_factor), flag, info, lane))
        assert e.value.code == Errc.bad_argument
        used = ctypes.c_int(-1)
        check(lib.tp_dev_leaf_solve_finish(dev.ctx._h, lane, dev.ptr(d_factor), flag, info, ctypes.byref(used)))
        got = dev.down(d_factor).reshape(rows, k, order="F")
        assert used.value == (1 if use_start else 0)
        assert list(dev.down(d_status)) == [0, 0]
        assert np.max(np.abs(got - want)) < 1e-8
    with pytest.raises(TuckerplanError) as e:          # nothing in flight
        check(lib.tp_dev_leaf_solve_finish(dev.ctx._h, 2, dev.ptr(d_factor), flag, info, None))
    assert e.value.code == Errc.bad_argument
    with pytest.raises(TuckerplanError) as e:
        check(lib.tp_dev_leaf_solve_begin(dev.ctx._h, dev.ptr(d_gram), ctypes.c_size_t(rows), k, None,
                                          dev.ptr(d_factor), flag, info, 4))
    assert e.value.code == Errc.bad_argument
