import sys, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_1707_05594_b200 import engine as E, distributed as D, hostgen
ctx1 = E.Context(0); o1 = D.GpuOps(ctx1)
big = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()
cases = [((552960, 704), 1, 16, "2D KT2 (2 CTA/SM)"), ((768, 720, 704), 1, 20, "3D KT3 (2 CTA/SM)"),
         ((276480, 704), 1, 100, "2D KT13 (1 CTA/SM)"), ((384, 720, 704), 1, 100, "3D KT13 (1 CTA/SM)"),
         ((552960, 704), 1, 40, "2D KT5 (1 CTA/SM)")]
for dims, mode, k, label in cases:
    x = hostgen.random_tensor(dims, 1)
    f = np.asfortranarray(hostgen.random_tensor([k, dims[mode]], 2).T).reshape(-1, order="F")
    xb, fb = o1.from_host(x), o1.from_host(f)
    os.environ["TPB_DISABLE_TMA_NOW"] = "1"
    ref = o1.to_host(o1.ttm_partial(xb, list(dims), mode, fb, dims[mode], 0, k, [0, k]))
    del os.environ["TPB_DISABLE_TMA_NOW"]
    bad = 0
    for rep in range(6):
        ctx1.synchronize(); torch.cuda.synchronize()
        z = o1.ttm_partial(xb, list(dims), mode, fb, dims[mode], 0, k, [0, k])
        with torch.cuda.stream(side):
            for _ in range(50): big.zero_()
        got = o1.to_host(z)
        torch.cuda.synchronize()
        d = np.abs(got - ref).reshape(-1)
        if d.max() > 1e-9:
            bad += 1
    print(label, dims, "bad runs:", bad, "of 6")
    del xb, fb
