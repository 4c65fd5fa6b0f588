"""Times the single-launch small dense kernels (tp_dev_cholesky / tp_dev_trsm_right_lt / tp_dev_jacobi_eig) with CUDA
events on the engine's stream.  usage: python tools/bench_small_dense.py  -> one JSON line per (rows, block)."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1707_05594_b200 import engine as E
from paper_1707_05594_b200._lib import check, lib

ctx = E.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
dp = lambda t, c=ctypes.c_double: ctypes.cast(t.data_ptr(), ctypes.POINTER(c))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


rng = np.random.default_rng(0)
for rows, b in [(48, 16), (96, 18), (200, 28), (400, 48), (1600, 108), (2048, 112)]:
    k = b - 8
    q, _ = np.linalg.qr(rng.standard_normal((b, b)))
    lam = np.concatenate([1 + 5 * rng.random(k), 1e-6 * rng.random(b - k)])
    h = (q * lam) @ q.T
    h = (h + h.T) / 2
    near = np.diag(np.sort(lam)[::-1]) + 1e-4 * (lambda a: (a + a.T) / 2)(rng.standard_normal((b, b)))
    z = rng.standard_normal((rows, b))
    s = z.T @ z
    d = lambda a: torch.from_numpy(np.asfortranarray(a).ravel(order="F").copy()).cuda()
    d_h, d_near, d_s, d_z = d(h), d(near), d(s), d(z)
    d_l, d_w, d_v = torch.zeros(b * b, dtype=torch.float64, device="cuda"), torch.zeros(b, dtype=torch.float64, device="cuda"), torch.zeros(b * b, dtype=torch.float64, device="cuda")
    d_fail = torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    fi = dp(d_fail, ctypes.c_int)
    out = {"rows": rows, "block": b}
    out["cholesky_us"] = timed(lambda: check(lib.tp_dev_cholesky(ctx._h, dp(d_s), b, dp(d_l), fi)))
    out["trsm_us"] = timed(lambda: check(lib.tp_dev_trsm_right_lt(ctx._h, dp(d_z), ctypes.c_size_t(rows), b, dp(d_l))))
    d_fail.zero_(); torch.cuda.synchronize()
    out["jacobi_random_us"] = timed(lambda: check(lib.tp_dev_jacobi_eig(ctx._h, dp(d_h), b, dp(d_w), dp(d_v), fi)))
    ctx.synchronize(); out["jacobi_random_sweeps"] = int(d_fail.cpu()[1])
    d_fail.zero_(); torch.cuda.synchronize()
    out["jacobi_near_diagonal_us"] = timed(lambda: check(lib.tp_dev_jacobi_eig(ctx._h, dp(d_near), b, dp(d_w), dp(d_v), fi)))
    ctx.synchronize(); out["jacobi_near_diagonal_sweeps"] = int(d_fail.cpu()[1])
    print(json.dumps(out))
