"""TEST INFRASTRUCTURE: CPU stand-in for paper_1707_05594_b200.distributed.GpuOps built on the oracle's NumPy
kernels, so that the grid executor's host logic (partitioning, exchange pattern, reduction order, schedule) can run
under gloo / as virtual ranks without a GPU.  Buffers are flat torch CPU float64 tensors."""
import numpy as np
import torch

from oracle import hooi_oracle as ho


class NumpyOps:
    def empty(self, count):
        return torch.empty(int(count), dtype=torch.float64)

    def zeros(self, count):
        return torch.zeros(int(count), dtype=torch.float64)

    def from_host(self, array):
        return torch.from_numpy(np.ascontiguousarray(array, dtype=np.float64).reshape(-1).copy())

    def to_host(self, t):
        return t.numpy().copy()

    def ttm_partial(self, x, dims, mode, factor, l_full, l0, k, dest_cuts):
        xs = x.numpy().reshape(dims)
        m = factor.numpy().reshape(k, l_full)[:, l0:l0 + dims[mode]]     # F^T restricted to the local rows of F
        z = ho.ttm(xs, m, mode)
        chunks = []
        for d in range(len(dest_cuts) - 1):
            sl = [slice(None)] * len(dims)
            sl[mode] = slice(dest_cuts[d], dest_cuts[d + 1])
            chunks.append(np.ascontiguousarray(z[tuple(sl)]).reshape(-1))
        return torch.from_numpy(np.concatenate(chunks))

    def ttm_scatter(self, x, dims, mode, factor, l_full, l0, k, dest_cuts, targets):
        part = self.ttm_partial(x, dims, mode, factor, l_full, l0, k, dest_cuts)
        per_row = int(np.prod(dims, dtype=np.int64)) // dims[mode]
        for d, target in enumerate(targets):
            lo, hi = per_row * dest_cuts[d], per_row * dest_cuts[d + 1]
            if hi > lo:
                target.copy_(part[lo:hi])

    def reduce_slots(self, slots, count):
        out = slots[0].clone()
        for s in slots[1:]:
            out += s
        return out

    def assemble(self, dst, outer, full_len, inner, src, l0, count):
        dst.view(outer, full_len, inner)[:, l0:l0 + count, :] = src.view(outer, count, inner)

    def gram(self, y, outer, rows, inner, out=None):
        u = ho.unfold(y.numpy().reshape(outer, rows, inner), 1)
        g = torch.from_numpy((u @ u.T).reshape(-1).copy())
        if out is None:
            return g
        out.copy_(g)
        return out

    def leaf_solve(self, gram, rows, k, start=None):
        vec, deg = ho.leading_from_gram(gram.numpy().reshape(rows, rows), k)
        factor = torch.from_numpy(np.asfortranarray(vec).reshape(-1, order="F").copy())
        return factor, torch.tensor([int(deg), 0], dtype=torch.int32)

    def empty_status(self):
        return torch.zeros(2, dtype=torch.int32)

    def sum_squares(self, x, count):
        v = x.numpy()[:count]
        return torch.tensor([float(np.dot(v, v))], dtype=torch.float64)

    def status_to_host(self, status):
        return int(status[0]), int(status[1])

    def synchronize(self):
        pass
