import sys, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_1707_05594_b200 import engine as E, distributed as D, hostgen
ctx1, ctx2, ctx3 = E.Context(0), E.Context(0), E.Context(0)
o1, o2, o3 = D.GpuOps(ctx1), D.GpuOps(ctx2), D.GpuOps(ctx3)
dims, mode, k = (552960, 704), 1, 16
g768 = hostgen.random_tensor((768, 768), 4); g768 = g768 @ g768.T
g704 = hostgen.random_tensor((704, 704), 5); g704 = g704 @ g704.T
x = hostgen.random_tensor(dims, 1)
f = np.asfortranarray(hostgen.random_tensor([k, dims[mode]], 2).T).reshape(-1, order="F")
xb, fb = o1.from_host(x), o1.from_host(f)
os.environ["TPB_DISABLE_TMA_NOW"] = "1"
ref = o1.to_host(o1.ttm_partial(xb, list(dims), mode, fb, dims[mode], 0, k, [0, k]))
del os.environ["TPB_DISABLE_TMA_NOW"]
big = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
pinned = torch.empty(8 << 20, dtype=torch.float64, pin_memory=True)
side = torch.cuda.Stream()
def run(kind):
    bad = 0
    for rep in range(4):
        for c in (ctx1, ctx2, ctx3): c.synchronize()
        torch.cuda.synchronize()
        b1, b2 = o2.from_host(g768), o3.from_host(g704)
        if kind in ("two_syevd",):
            o2.leaf_solve(b1, 768, 24)
        z = o1.ttm_partial(xb, list(dims), mode, fb, dims[mode], 0, k, [0, k])
        if kind in ("two_syevd", "syevd_after704"):
            o3.leaf_solve(b2, 704, 16)
        elif kind == "copies":
            with torch.cuda.stream(side):
                for _ in range(20):
                    pinned.copy_(big[:8 << 20], non_blocking=True); big[:8 << 20].copy_(pinned, non_blocking=True)
        elif kind == "malloc":
            for i in range(20):
                t = torch.empty((32 << 20) + i * 4096, dtype=torch.float64, device="cuda"); del t; torch.cuda.empty_cache()
        elif kind == "memset":
            with torch.cuda.stream(side):
                for _ in range(50): big.zero_()
        elif kind == "tiny_kernels":
            with torch.cuda.stream(side):
                s = torch.zeros(1024, device="cuda", dtype=torch.float64)
                for _ in range(2000): s.add_(1.0)
        elif kind == "dgemm":
            with torch.cuda.stream(side):
                a = torch.zeros((2048, 2048), dtype=torch.float64, device="cuda")
                for _ in range(30): torch.matmul(a, a)
        got = o1.to_host(z)
        torch.cuda.synchronize()
        d = np.abs(got - ref).reshape(-1)
        if d.max() > 1e-9:
            bad += 1
            idx = np.flatnonzero(d > 1e-9)
            print("    rep", rep, "n_bad", len(idx), "rows", idx[0] // k, "..", idx[-1] // k, "max", d.max())
    print(kind, "bad runs:", bad, "of 4")
for kind in ("none", "two_syevd", "syevd_after704", "copies", "memset", "tiny_kernels", "dgemm", "malloc"):
    run(kind)
