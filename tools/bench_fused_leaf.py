"""CUDA-event times and in-kernel phase cycles of the one-launch leaf solve (csrc/leaf_solve_kernels.cu) on the leaf
shapes of BASELINE configs 1-4: a cold solve, then warm solves from the previous Ritz vectors on slightly perturbed
Gram matrices (the steady state of a HOOI run).  One JSON line per shape."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_05594_b200 import engine as E
from paper_1707_05594_b200._lib import check, lib

PHASES = ["start", "gq_products", "small_grams", "cholesky", "trsm", "jacobi", "ritz_residuals", "certificate"]


def ptr(t, ctype=ctypes.c_double):
    return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctype))


def main():
    ctx = E.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    shapes = [(200, 20, 400, 1e-3), (96, 10, 1000, 1e-3), (100, 10, 4000, 1e-2), (100, 20, 2000, 1e-2),
              (50, 5, 8000, 1e-2), (48, 8, 4096, 1e-3), (160, 24, 700, 1e-3)]
    for rows, k, cols, sigma in shapes:
        rng = np.random.default_rng(rows + k)
        b = k + 8
        base = rng.standard_normal((rows, k)) @ rng.standard_normal((k, cols))
        grams = []
        noise = sigma * rng.standard_normal((rows, cols))
        for i in range(6):
            # the perturbation between consecutive matrices shrinks geometrically, as between the sweeps of a
            # converging HOOI run
            y = base + noise + (1e-2 / (100 ** i)) * rng.standard_normal((rows, cols))
            grams.append(torch.from_numpy(np.asfortranarray(y @ y.T).ravel(order="F").copy()).cuda())
        start, _ = np.linalg.qr(rng.standard_normal((rows, k)))
        d_start = torch.from_numpy(np.asfortranarray(start).ravel(order="F").copy()).cuda()
        ritz = torch.zeros(rows * b, dtype=torch.float64, device="cuda")
        theta = torch.zeros(b, dtype=torch.float64, device="cuda")
        factor = torch.zeros(rows * k, dtype=torch.float64, device="cuda")
        ints = torch.zeros(8, dtype=torch.int32, device="cuda")
        diag = torch.zeros(16, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        out = []
        for i, g in enumerate(grams):
            warm = i > 0
            ints.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ip = ptr(ints, ctypes.c_int)
            check(lib.tp_dev_leaf_solve_fused(ctx._h, ptr(g), ctypes.c_size_t(rows), k, ptr(ritz if warm else d_start),
                                              1 if warm else 0, ptr(ritz), ptr(theta), ptr(factor), ip,
                                              ctypes.cast(ctypes.addressof(ip.contents) + 16, ctypes.POINTER(ctypes.c_int)),
                                              ptr(diag)))
            e1.record(stream)
            e1.synchronize()
            iv, dv = ints.cpu().tolist(), diag.cpu().tolist()
            out.append({"warm": warm, "us": e0.elapsed_time(e1) * 1e3, "miss": iv[4], "fail": iv[5],
                        "jacobi_sweeps": iv[6], "power_steps": iv[7], "rounds": dv[3],
                        "phase_us_at_1965MHz": {n: round(c / 1965.0, 1) for n, c in zip(PHASES, dv[4:12])},
                        "jacobi_us_checks_rotations_updates_barriers": [round(c / 1965.0, 1) for c in dv[12:16]]})
        print(json.dumps({"rows": rows, "k": k, "block": b, "runs": out}))
    ctx.close()


if __name__ == "__main__":
    main()
