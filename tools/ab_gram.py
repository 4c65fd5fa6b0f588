"""A/B timing of the Gram kernels on the C5 leaf shapes (1600 rows, 10^4 columns): wide (128 x 128 tiles, TMA) against
narrow (64 x 64, cp.async).  CUDA events around tp_dev_gram on device buffers.  Usage: python tools/ab_gram.py"""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05594_b200 import engine as E

ctx = E.Context(0)
lib = E.lib
stream = torch.cuda.ExternalStream(ctx.stream)
shapes = {"mode0 (1,1600,10000)": (1, 1600, 10000), "mode1 (100,1600,100)": (100, 1600, 100),
          "mode2 (10000,1600,1)": (10000, 1600, 1)}
flush = torch.empty(160 << 20, dtype=torch.float64, device="cuda")   # 1.3 GB > L2
for name, (outer, rows, inner) in shapes.items():
    y = torch.randn(outer * rows * inner, dtype=torch.float64, device="cuda")
    g = torch.empty(rows * rows, dtype=torch.float64, device="cuda")
    ref = None
    for wide in (0, 1):
        E.check(lib.tp_set_global_option(4, ctypes.c_longlong(wide)))
        times = []
        for it in range(8):
            flush.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                E.check(lib.tp_dev_gram(ctx._h, ctypes.c_void_p(y.data_ptr()), ctypes.c_size_t(outer), ctypes.c_size_t(rows),
                                        ctypes.c_size_t(inner), ctypes.c_void_p(g.data_ptr())))
                b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        got = g.clone()
        if ref is None:
            ref = got
        err = float((got - ref).abs().max() / ref.abs().max())
        flops = rows * rows * outer * inner          # half of a full GEMM's 2 m n k
        best = min(times[2:])
        print(json.dumps({"shape": name, "wide": wide, "ms_best": round(best, 4), "ms_median": round(float(np.median(times[2:])), 4),
                          "tflops_syrk": round(flops / best / 1e9, 2), "rel_diff_vs_narrow": err}))
E.check(lib.tp_set_global_option(4, ctypes.c_longlong(1)))
