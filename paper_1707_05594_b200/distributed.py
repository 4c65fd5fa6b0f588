"""HOOI on a Cartesian processor grid: one process per GPU, tensors block-distributed, factors replicated.

This is the paper's distribution scheme executed for real — the reference only
*simulates* it (simulate.hpp) and charges (q_n - 1)|Out_u| elements per TTM (grid_volume.hpp:41):

  * grid q (prod q = P), normally `optimal_static_grid(tree, spec, P)`; rank = row-major rank of the block
    coordinates (simulate.hpp:69-73); every tensor of the sweep is cut along mode n at floor(b * ext_n / q_n)
    (grid.hpp:114-119) with its own extent (L_n before the mode is multiplied, K_n after);
  * TTM along mode n: each rank multiplies its block by its row slice of the replicated factor.  If q_n = 1 that
    is the whole story (no communication).  If q_n > 1 the products are partial sums over the split mode: the
    kernel writes them destination-major, the q_n ranks of the mode-n process group exchange the chunks
    (send/recv, each rank ships (q_n - 1)/q_n of its partial product = the reference's volume) and every rank adds
    the q_n contributions to its K-slice in rank order — a reduce-scatter with a fixed, deterministic summation order;
  * leaf n: Gram of the local block (after gathering the mode-n slices to the group's first rank when q_n > 1),
    all-reduced over all ranks, then the same eigen-solve on every rank (bit-identical input, so the replicated
    factors stay consistent without a broadcast);
  * core: the same distributed TTM chain with the new factors.

The rank program is a generator that *yields* its communication requests.  `run_rank` executes them with
torch.distributed (NCCL on GPUs, gloo in the CPU tests); `run_virtual` steps P rank programs in lock-step inside
one process and moves the data itself — that is how the multi-rank path is exercised on a single GPU.
Local arithmetic goes through a backend: `GpuOps` (the CUDA library, device pointers of torch tensors — torch is
only the allocator and the collective plumbing) or a NumPy backend that lives with the tests.
"""
from __future__ import annotations

import ctypes
import os
import sys
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, Generator, List, Optional, Sequence, Tuple

import numpy as np

from . import planner as P
from ._lib import check, dbl_p, lib, size_array


# ----------------------------------------------------------------------------------------------- layout
class GridLayout:
    """Block distribution induced by one grid (grid.hpp:23-45, 114-125; simulate.hpp:69-73)."""

    def __init__(self, q: Sequence[int]):
        self.q = [int(v) for v in q]
        self.n = len(self.q)
        self.procs = int(np.prod(self.q, dtype=np.int64))

    def coords(self, rank: int) -> List[int]:
        c = [0] * self.n
        for m in range(self.n - 1, -1, -1):
            c[m] = rank % self.q[m]
            rank //= self.q[m]
        return c

    def rank_of(self, coords: Sequence[int]) -> int:
        r = 0
        for m in range(self.n):
            r = r * self.q[m] + int(coords[m])
        return r

    def cuts(self, ext: int, mode: int) -> List[int]:
        return P.block_bounds(int(ext), self.q[mode])

    def local_range(self, rank: int, mode: int, ext: int) -> Tuple[int, int]:
        c = self.coords(rank)[mode]
        cuts = self.cuts(ext, mode)
        return cuts[c], cuts[c + 1]

    def local_dims(self, rank: int, ext: Sequence[int]) -> List[int]:
        return [hi - lo for lo, hi in (self.local_range(rank, m, e) for m, e in enumerate(ext))]

    def slices(self, rank: int, ext: Sequence[int]):
        return tuple(slice(*self.local_range(rank, m, e)) for m, e in enumerate(ext))

    def mode_group(self, rank: int, mode: int) -> List[int]:
        """Ranks that share every coordinate but `mode`, ordered by their mode coordinate."""
        c = self.coords(rank)
        out = []
        for v in range(self.q[mode]):
            c2 = list(c)
            c2[mode] = v
            out.append(self.rank_of(c2))
        return out


# ----------------------------------------------------------------------------------------------- requests
@dataclass
class Exchange:      # point-to-point batch: sends [(peer, tensor)], recvs [(peer, tensor)]
    sends: list
    recvs: list


@dataclass
class AllReduce:     # sum over all ranks, in place
    tensor: object


@dataclass
class Broadcast:     # root's tensor to every rank, in place
    tensor: object
    root: int


@dataclass
class PeerSlots:     # ask the runner for peer-addressable receive slots of one reduce-scatter (fused scatter epilogue)
    key: object      # stable per call site, so that runners can keep the buffers between sweeps
    group: list      # ranks of the mode group in slot order
    me: int          # this rank's position in the group
    count: int       # elements of this rank's chunk = size of each of its receive slots
    counts: list = field(default_factory=list)   # chunk sizes of all group members (what this rank writes to each)


@dataclass
class PeerSlotsReply:
    my_slots: list   # len(group) local buffers of `count` elements; slot s is written by group[s]
    targets: list    # len(group) buffers: targets[d] is group[d]'s slot number `me` (its memory, its size)


@dataclass
class GroupBarrier:  # every group member's stores into peer slots are complete and visible
    group: list


@dataclass
class Volume:        # bookkeeping: elements this rank shipped for a TTM node (checked against the reference model)
    node: int
    elements: int


# ----------------------------------------------------------------------------------------------- backends
class GpuOps:
    """Local kernels on one B200 through the C ABI; buffers are torch CUDA tensors (allocator + NCCL plumbing)."""

    def __init__(self, ctx, device_index: int = 0):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.device = torch.device("cuda", device_index)
        self.stream = torch.cuda.ExternalStream(ctx.stream, device=self.device)
        self.fast_solves = 0   # leaves served by the certified subspace iteration
        self._busy_lanes = set()

    def _ptr(self, t):
        return ctypes.cast(t.data_ptr(), dbl_p)

    def empty(self, count: int):
        with self.torch.cuda.stream(self.stream):
            return self.torch.empty(max(int(count), 1), dtype=self.torch.float64, device=self.device)[:int(count)]

    def zeros(self, count: int):
        with self.torch.cuda.stream(self.stream):
            return self.torch.zeros(max(int(count), 1), dtype=self.torch.float64, device=self.device)[:int(count)]

    def from_host(self, array: np.ndarray):
        with self.torch.cuda.stream(self.stream):
            return self.torch.from_numpy(np.ascontiguousarray(array, dtype=np.float64).reshape(-1)).to(
                self.device, non_blocking=False)

    def to_host(self, t) -> np.ndarray:
        with self.torch.cuda.stream(self.stream):
            out = t.cpu()
        return out.numpy()

    def ttm_partial(self, x, dims, mode, factor, l_full, l0, k, dest_cuts):
        count = int(np.prod([d if i != mode else k for i, d in enumerate(dims)], dtype=np.int64))
        z = self.empty(count)
        cuts = size_array(dest_cuts)
        check(lib.tp_dev_ttm_partial(self.ctx._h, self._ptr(x), len(dims), size_array(dims), int(mode),
                                     self._ptr(factor), ctypes.c_size_t(l_full), ctypes.c_size_t(l0),
                                     ctypes.c_size_t(k), len(dest_cuts) - 1, cuts, self._ptr(z)))
        return z

    def ttm_scatter(self, x, dims, mode, factor, l_full, l0, k, dest_cuts, targets):
        """Partial product whose chunk d is stored straight into targets[d] (own or peer memory)."""
        ptrs = (dbl_p * len(targets))(*[self._ptr(t) if t is not None and t.numel() else None for t in targets])
        check(lib.tp_dev_ttm_scatter(self.ctx._h, self._ptr(x), len(dims), size_array(dims), int(mode),
                                     self._ptr(factor), ctypes.c_size_t(l_full), ctypes.c_size_t(l0),
                                     ctypes.c_size_t(k), len(dest_cuts) - 1, size_array(dest_cuts), ptrs))

    def reduce_slots(self, slots, count):
        out = self.empty(count)
        ptrs = (dbl_p * len(slots))(*[self._ptr(s) for s in slots])
        check(lib.tp_dev_reduce_slots(self.ctx._h, self._ptr(out), ptrs, len(slots), ctypes.c_size_t(count)))
        return out

    def assemble(self, dst, outer, full_len, inner, src, l0, count):
        check(lib.tp_dev_assemble_mode(self.ctx._h, self._ptr(dst), ctypes.c_size_t(outer), ctypes.c_size_t(full_len),
                                       ctypes.c_size_t(inner), self._ptr(src), ctypes.c_size_t(l0),
                                       ctypes.c_size_t(count)))

    def gram(self, y, outer, rows, inner, out=None):
        g = out if out is not None else self.empty(rows * rows)
        check(lib.tp_dev_gram(self.ctx._h, self._ptr(y), ctypes.c_size_t(outer), ctypes.c_size_t(rows),
                              ctypes.c_size_t(inner), self._ptr(g)))
        return g

    def leaf_solve(self, gram, rows, k, start=None):
        """Top-k eigenvectors of gram; `start` (previous factor) enables the certified subspace iteration."""
        factor = self.empty(rows * k)
        with self.torch.cuda.stream(self.stream):
            status = self.torch.zeros(2, dtype=self.torch.int32, device=self.device)
        flag = ctypes.cast(status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        info = ctypes.cast(status.data_ptr() + 4, ctypes.POINTER(ctypes.c_int))
        used = ctypes.c_int()
        check(lib.tp_dev_leaf_solve_warm(self.ctx._h, self._ptr(gram), ctypes.c_size_t(rows), int(k),
                                         self._ptr(start) if start is not None else None, self._ptr(factor), flag,
                                         info, ctypes.byref(used)))
        self.fast_solves += used.value
        return factor, status

    def leaf_solve_begin(self, gram, rows, k, start, lane):
        """Queues the leaf solve on side stream `lane` and returns a handle for leaf_solve_finish; falls back to the
        synchronous call when that lane is still busy."""
        factor = self.empty(rows * k)
        with self.torch.cuda.stream(self.stream):
            status = self.torch.zeros(2, dtype=self.torch.int32, device=self.device)
        if lane in self._busy_lanes:
            done_factor, done_status = self.leaf_solve(gram, rows, k, start)
            return {"lane": None, "factor": done_factor, "status": done_status}
        flag = ctypes.cast(status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        info = ctypes.cast(status.data_ptr() + 4, ctypes.POINTER(ctypes.c_int))
        check(lib.tp_dev_leaf_solve_begin(self.ctx._h, self._ptr(gram), ctypes.c_size_t(rows), int(k),
                                          self._ptr(start) if start is not None else None, self._ptr(factor), flag,
                                          info, int(lane)))
        self._busy_lanes.add(lane)
        return {"lane": lane, "factor": factor, "status": status, "gram": gram, "start": start}

    def leaf_solve_finish(self, handle):
        if handle["lane"] is None:
            return handle["factor"], handle["status"]
        status = handle["status"]
        flag = ctypes.cast(status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        info = ctypes.cast(status.data_ptr() + 4, ctypes.POINTER(ctypes.c_int))
        used = ctypes.c_int()
        check(lib.tp_dev_leaf_solve_finish(self.ctx._h, int(handle["lane"]), self._ptr(handle["factor"]), flag, info,
                                           ctypes.byref(used)))
        self._busy_lanes.discard(handle["lane"])
        self.fast_solves += used.value
        return handle["factor"], status

    def empty_status(self):
        with self.torch.cuda.stream(self.stream):
            return self.torch.zeros(2, dtype=self.torch.int32, device=self.device)

    def sum_squares(self, x, count):
        out = self.empty(1)
        check(lib.tp_dev_sum_squares(self.ctx._h, self._ptr(x), ctypes.c_size_t(count), self._ptr(out)))
        return out

    def status_to_host(self, status):
        flag, info = (int(v) for v in self.to_host_int(status))
        return flag, info

    def to_host_int(self, t):
        with self.torch.cuda.stream(self.stream):
            return t.cpu().tolist()

    def synchronize(self):
        self.ctx.synchronize()

    def stream_context(self):
        """torch ops issued by the runners (copies, NCCL calls) must queue on the engine's stream."""
        return self.torch.cuda.stream(self.stream)


# ----------------------------------------------------------------------------------------------- rank program
@dataclass
class SweepResult:
    tree_macs: int = 0
    core_macs: int = 0
    peak_live: int = 0
    degenerate: bool = False
    volume_sent: Dict[int, int] = field(default_factory=dict)   # tree node -> elements this rank shipped (TTM)
    regrid_sent: Dict[int, int] = field(default_factory=dict)   # tree node -> elements this rank shipped (regrid)


class DistributedHooi:
    """One rank's share of Jacobi HOOI sweeps (hooi.hpp:189-229) on a static grid, or on a per-node scheme
    (grid_dynamic.hpp: `q` may be a planner.DynamicGridScheme; the tensor and the core live on its root grid, a node
    whose grid differs from its parent's first redistributes its input)."""

    def __init__(self, ops, spec: P.ProblemSpec, tree: P.TtmTree, q, rank: int, async_solve: bool = True):
        self.ops, self.spec, self.tree, self.rank = ops, spec, tree, int(rank)
        scheme = q if isinstance(q, P.DynamicGridScheme) else P.uniform_scheme(tree, q)
        self.scheme = scheme
        self.layout = GridLayout(scheme.root)
        self.n = spec.n_modes()
        P.validate_tree(tree, spec)
        P.scheme_volume(tree, spec, scheme, self.layout.procs)      # validates every grid, missing_assignment
        self.node_layout = {node: (self.layout if list(g) == list(self.layout.q) else GridLayout(g))
                            for node, g in scheme.node_grids.items()}
        if not 0 <= self.rank < self.layout.procs:
            raise ValueError("rank outside the grid")
        self.cost = P.tree_cost(tree, spec)
        self.factors: List[object] = [None] * self.n      # replicated, L_n x K_n column-major flat buffers
        self.core = None                                   # local core block, flat
        self.core_ldims: List[int] = []
        self.tensor = None                                 # local block of T, flat
        self.tensor_ldims = self.layout.local_dims(self.rank, spec.L)
        self.core_order = _cheapest_chain_order(spec)
        self.events: Optional[Callable[[str, int], None]] = None   # timing hook: ("begin"/"end" + phase, node)
        # Carried path (as in the single-GPU plan): the core chain contracts along one root-to-leaf
        # path of the tree with the new factors, on the grids of those nodes; its partial products are the next
        # sweep's intermediates at those nodes and are kept instead of recomputed.
        # Leaf eigen-solves: queued on a side stream right after the Gram all-reduce and collected where the core
        # chain first needs the factor, so they overlap the rest of the tree; with more than one rank each leaf has
        # one owner rank that solves it and broadcasts the factor (replicating every solve on every rank would put
        # P copies of the same latency-bound work on the critical path: at C5 / P = 8 more than the tree itself).
        self.async_solve = async_solve and hasattr(ops, "leaf_solve_begin")
        self.owner_solve = self.layout.procs > 1
        self.peer_scatter = True      # use peer-slot stores for reduce-scatters where the runner offers them
        self.scatter_launches = 0
        self.carry_enabled = self.n >= 2
        self._carry_path, self._carry_leaf_mode = self._first_leaf_path()
        self._carried: Dict[int, tuple] = {}
        self._gram_buf: Dict[int, object] = {}

    # -- state ------------------------------------------------------------------------------------
    def set_local_tensor(self, block: np.ndarray):
        if list(block.shape) != self.tensor_ldims:
            raise ValueError("local block has shape %s, expected %s" % (block.shape, self.tensor_ldims))
        self.tensor = self.ops.from_host(block)
        self._carried = {}

    def set_local_tensor_buffer(self, buf):
        self.tensor = buf
        self._carried = {}

    def set_factors(self, factors: Sequence[np.ndarray]):
        self.factors = [self.ops.from_host(np.asfortranarray(f).reshape(-1, order="F")) for f in factors]
        self._carried = {}

    def invalidate(self):
        """Call after changing the local tensor block in place: drops the products carried from the last sweep."""
        self._carried = {}

    def _first_leaf_path(self):
        """TTM nodes from the root down to the first leaf in execution order, and that leaf's mode."""
        node, path = 0, []
        while True:
            kids = self.tree.children[node]
            leaf = next((c for c in kids if self.tree.kind[c] == P.LEAF), None)
            if leaf is not None:
                return path, self.tree.mode[leaf]
            node = kids[0]
            path.append(node)

    def get_factors(self) -> List[np.ndarray]:
        return [self.ops.to_host(f).reshape((l, k), order="F").copy()
                for f, l, k in zip(self.factors, self.spec.L, self.spec.K)]

    def get_local_core(self) -> np.ndarray:
        return self.ops.to_host(self.core).reshape(self.core_ldims).copy()

    def _mark(self, what: str, node: int = -1):
        if self.events:
            self.events(what, node)

    # -- distributed mode product -------------------------------------------------------------------
    def _ttm(self, x, ext, ldims, mode, factor, node, result: SweepResult, lay: Optional[GridLayout] = None):
        """x: local block with global extents ext / local dims ldims; returns (z, new_ext, new_ldims)."""
        lay = lay or self.layout
        q_n = lay.q[mode]
        k, l_full = self.spec.K[mode], self.spec.L[mode]
        l0, _ = lay.local_range(self.rank, mode, ext[mode])
        new_ext = list(ext)
        new_ext[mode] = k
        new_ldims = list(ldims)
        if q_n == 1:
            z = self.ops.ttm_partial(x, ldims, mode, factor, l_full, l0, k, [0, k])
            new_ldims[mode] = k
            return z, new_ext, new_ldims
        kcuts = lay.cuts(k, mode)
        group = lay.mode_group(self.rank, mode)
        me = lay.coords(self.rank)[mode]
        per_row = int(np.prod(ldims, dtype=np.int64)) // ldims[mode]      # outer_loc * inner_loc
        offs = [per_row * c for c in kcuts]
        mine = offs[me + 1] - offs[me]
        new_ldims[mode] = kcuts[me + 1] - kcuts[me]
        if self.peer_scatter and hasattr(self.ops, "ttm_scatter"):
            # fused form: the kernel's epilogue stores every chunk into its owner's receive slot (peer memory over
            # NVLink); what remains of the reduce-scatter is a barrier and the ordered sum of the local slots
            reply = yield PeerSlots(("ttm", node, mode, tuple(ldims)), group, me, mine,
                                    [offs[d + 1] - offs[d] for d in range(len(group))])
            if reply is not None:
                self.ops.ttm_scatter(x, ldims, mode, factor, l_full, l0, k, kcuts, reply.targets)
                self.scatter_launches += 1
                if node >= 0:
                    result.volume_sent[node] = result.volume_sent.get(node, 0) + (offs[-1] - mine)
                yield GroupBarrier(group)
                return self.ops.reduce_slots(reply.my_slots, mine), new_ext, new_ldims
        part = self.ops.ttm_partial(x, ldims, mode, factor, l_full, l0, k, kcuts)
        slots, sends, recvs = [], [], []
        for d, peer in enumerate(group):
            if d == me:
                slots.append(part[offs[me]:offs[me + 1]])
            else:
                sends.append((peer, part[offs[d]:offs[d + 1]]))
                buf = self.ops.empty(mine)
                recvs.append((peer, buf))
                slots.append(buf)
        if node >= 0:
            result.volume_sent[node] = result.volume_sent.get(node, 0) + (offs[-1] - mine)
        yield Exchange(sends, recvs)
        z = self.ops.reduce_slots(slots, mine)
        new_ldims[mode] = kcuts[me + 1] - kcuts[me]
        return z, new_ext, new_ldims

    # -- leaf: Gram (all ranks) + eigen-solve -------------------------------------------------------
    def _leaf(self, y, ext, ldims, mode, result: SweepResult, statuses: list, lay: Optional[GridLayout] = None):
        lay = lay or self.layout
        q_n = lay.q[mode]
        rows, k = self.spec.L[mode], self.spec.K[mode]
        outer = int(np.prod(ldims[:mode], dtype=np.int64)) if mode else 1
        inner = int(np.prod(ldims[mode + 1:], dtype=np.int64)) if mode + 1 < self.n else 1
        # one Gram buffer per mode for the life of the executor: the leaf solve records its kernel sequence as a
        # CUDA graph on the buffers it first sees
        if mode not in self._gram_buf:
            self._gram_buf[mode] = self.ops.empty(rows * rows)
        gram_out = self._gram_buf[mode]
        if q_n == 1:
            gram = self.ops.gram(y, outer, rows, inner, gram_out)
        else:
            # the unfolding's rows are split over the mode-n group: bring the slices to the group's first rank,
            # which then owns these columns of the unfolding; the other ranks add nothing to the Gram sum
            group = lay.mode_group(self.rank, mode)
            me = lay.coords(self.rank)[mode]
            cuts = lay.cuts(rows, mode)
            if me == 0:
                full = self.ops.empty(outer * rows * inner)
                recvs, pieces = [], []
                for d, peer in enumerate(group):
                    count = cuts[d + 1] - cuts[d]
                    if d == 0:
                        pieces.append((y, cuts[d], count))
                    else:
                        buf = self.ops.empty(outer * count * inner)
                        recvs.append((peer, buf))
                        pieces.append((buf, cuts[d], count))
                yield Exchange([], recvs)
                for buf, lo, count in pieces:
                    self.ops.assemble(full, outer, rows, inner, buf, lo, count)
                gram = self.ops.gram(full, outer, rows, inner, gram_out)
            else:
                yield Exchange([(group[0], y)], [])
                gram = gram_out
                gram.zero_()
        yield AllReduce(gram)
        index = len(self._pending)                       # position of this leaf in the walk
        owner = index % lay.procs if self.owner_solve else None
        entry = {"owner": owner, "rows": rows, "k": k, "handle": None, "done": None}
        if owner is None or owner == self.rank:
            if self.async_solve:
                entry["handle"] = self.ops.leaf_solve_begin(gram, rows, k, self.factors[mode], index % 4)
            else:
                entry["done"] = self.ops.leaf_solve(gram, rows, k, self.factors[mode])
        self._pending[mode] = entry
        return None

    def _collect(self, mode, statuses: list):
        """New factor of `mode`: finish this rank's solve if it has one, then share the owner's result."""
        entry = self._pending.pop(mode)
        if entry["handle"] is not None:
            factor, status = self.ops.leaf_solve_finish(entry["handle"])
        elif entry["done"] is not None:
            factor, status = entry["done"]
        else:
            factor = self.ops.empty(entry["rows"] * entry["k"])
            status = self.ops.empty_status()
        if entry["owner"] is not None:
            yield Broadcast(factor, entry["owner"])
            yield Broadcast(status, entry["owner"])
        statuses.append(status)
        return factor

    # -- one sweep ------------------------------------------------------------------------------------
    def sweep(self) -> Generator:
        """Generator: yields Exchange / AllReduce requests, returns a SweepResult."""
        res = SweepResult(tree_macs=self.cost.total_macs, peak_live=self.cost.depth + 1)
        statuses: list = []
        fresh: List[object] = [None] * self.n
        tree = self.tree
        self._pending = {}

        def walk(node, x, ext, ldims, lay):
            for c in tree.children[node]:
                mode = tree.mode[c]
                if tree.kind[c] == P.LEAF:
                    self._mark("begin_leaf", c)
                    yield from self._leaf(x, ext, ldims, mode, res, statuses, lay)
                    self._mark("end_leaf", c)
                elif c in self._carried:
                    # computed by the previous sweep's core chain with the factors this sweep starts from
                    z, e2, l2, sent, moved = self._carried[c]
                    if sent:
                        res.volume_sent[c] = sent
                    if moved:
                        res.regrid_sent[c] = moved
                    yield from walk(c, z, e2, l2, self.node_layout[c])
                else:
                    xin, lin, target = x, ldims, self.node_layout[c]
                    if target.q != lay.q:
                        # the node runs on its own grid: redistribute its input first (the paper's regrid)
                        self._mark("begin_regrid", c)
                        sends, _ = regrid_plan(ext, lay, target, self.rank)
                        res.regrid_sent[c] = sum(int(np.prod([hi - lo for lo, hi in o], dtype=np.int64))
                                                 for peer, o in sends if peer != self.rank)
                        moved = yield from regrid(x.view(ldims), ext, lay, target, self.rank, self.ops.empty)
                        lin = target.local_dims(self.rank, ext)
                        xin = moved.reshape(-1)
                        self._mark("end_regrid", c)
                    self._mark("begin_ttm", c)
                    z, e2, l2 = yield from self._ttm(xin, ext, lin, mode, self.factors[mode], c, res, target)
                    self._mark("end_ttm", c)
                    yield from walk(c, z, e2, l2, target)

        self._mark("begin_tree")
        yield from walk(0, self.tensor, list(self.spec.L), list(self.tensor_ldims), self.layout)
        self._mark("end_tree")
        # core_from_factors (hooi.hpp:93-100) in the cheapest order, with the new factors
        self._mark("begin_core")
        x, ext, ldims = self.tensor, list(self.spec.L), list(self.tensor_ldims)
        card = int(np.prod(self.spec.L, dtype=object))
        core_macs = 0
        for m in range(self.n):                      # the ledger keeps the reference's mode order
            core_macs += self.spec.K[m] * card
            card = card * self.spec.K[m] // self.spec.L[m]
        if self.carry_enabled and self._carry_path:
            lay, carried = self.layout, {}
            for c in self._carry_path:
                mode, target, ledger = tree.mode[c], self.node_layout[c], SweepResult()
                fresh[mode] = yield from self._collect(mode, statuses)
                if target.q != lay.q:
                    sends, _ = regrid_plan(ext, lay, target, self.rank)
                    ledger.regrid_sent[c] = sum(int(np.prod([hi - lo for lo, hi in o], dtype=np.int64))
                                                for peer, o in sends if peer != self.rank)
                    moved = yield from regrid(x.view(ldims), ext, lay, target, self.rank, self.ops.empty)
                    x, ldims = moved.reshape(-1), target.local_dims(self.rank, ext)
                self._mark("begin_ttm", c)
                x, ext, ldims = yield from self._ttm(x, ext, ldims, mode, fresh[mode], c, ledger, target)
                self._mark("end_ttm", c)
                carried[c] = (x, list(ext), list(ldims), ledger.volume_sent.get(c, 0), ledger.regrid_sent.get(c, 0))
                lay = target
            m = self._carry_leaf_mode
            fresh[m] = yield from self._collect(m, statuses)
            x, ext, ldims = yield from self._ttm(x, ext, ldims, m, fresh[m], -1, res, lay)
            if lay.q != self.layout.q:      # the core lives on the root grid
                moved = yield from regrid(x.view(ldims), ext, lay, self.layout, self.rank, self.ops.empty)
                x, ldims = moved.reshape(-1), self.layout.local_dims(self.rank, ext)
            self._carried = carried
        else:
            self._carried = {}
            for m in self.core_order:
                fresh[m] = yield from self._collect(m, statuses)
                x, ext, ldims = yield from self._ttm(x, ext, ldims, m, fresh[m], -1, res)
        self._mark("end_core")
        self.core, self.core_ldims = x, ldims
        self.factors = fresh
        res.core_macs = core_macs
        for status in statuses:
            flag, info = self.ops.status_to_host(status)
            if info != 0:
                from ._lib import Errc, TuckerplanError
                raise TuckerplanError(int(Errc.too_large), "eigensolver did not converge")
            res.degenerate = res.degenerate or bool(flag)
        return res

    def norm_squared(self, buf, count) -> Generator:
        s = self.ops.sum_squares(buf, count)
        yield AllReduce(s)
        return float(self.ops.to_host(s)[0])

    def fit_from_norms(self) -> Generator:
        """sqrt(||T||^2 - ||G||^2) / ||T|| (orthonormal factors)."""
        t2 = yield from self.norm_squared(self.tensor, int(np.prod(self.tensor_ldims, dtype=np.int64)))
        g2 = yield from self.norm_squared(self.core, int(np.prod(self.core_ldims, dtype=np.int64)))
        return float(np.sqrt(max(t2 - g2, 0.0) / t2)), float(np.sqrt(g2))


def _cheapest_chain_order(spec: P.ProblemSpec) -> List[int]:
    """Same DP as the engine's core chain (engine.cu cheapest_chain_order): fewest MACs, ties to the smaller mode."""
    n = spec.n_modes()
    full = (1 << n) - 1
    best = {0: (0, [])}
    for done in range(full):
        if done not in best:
            continue
        cost, order = best[done]
        card = 1
        for m in range(n):
            card *= spec.K[m] if (done >> m) & 1 else spec.L[m]
        for m in range(n):
            if (done >> m) & 1:
                continue
            nxt = done | (1 << m)
            c = cost + spec.K[m] * card
            if nxt not in best or c < best[nxt][0]:
                best[nxt] = (c, order + [m])
    return best[full][1]


# ----------------------------------------------------------------------------------------------- runners
def _stream_of(ops):
    import contextlib
    return ops.stream_context() if ops is not None and hasattr(ops, "stream_context") else contextlib.nullcontext()


class SymmetricSlots:
    """Receive slots in NVLink-mapped symmetric memory (torch.distributed._symmetric_memory): the runner-side half of
    the fused reduce-scatter.  Rank r keeps, per call site, one symmetric buffer of len(group) slots; slot s is
    written by group member s directly from its TTM kernel's epilogue (tp_dev_ttm_scatter), through the peer view
    `get_buffer(r, ...)` of that buffer.  Buffers are allocated once per call site and reused every sweep; a barrier
    on the symmetric-memory signal pads before the stores (the owners are done reading the previous sweep's slots)
    and one after (all stores have landed) replace the send/recv.

    Opt-in (`bench.py --peer-slots`): only one GPU was available while this was written, so it has run at world size 1
    only (tests/test_distributed.py::test_symmetric_slots_world_size_one)."""

    def __init__(self, dist, device):
        import torch
        import torch.distributed._symmetric_memory as symm
        self.torch, self.symm, self.dist, self.device = torch, symm, dist, device
        self.cache = {}

    def slots(self, req: PeerSlots) -> PeerSlotsReply:
        torch, q = self.torch, len(req.group)
        entry = self.cache.get(req.key)
        if entry is None:
            # symmetric allocations must have one size on every rank: agree on the largest chunk once per call site
            bound = torch.tensor([max(req.counts + [req.count, 1])], dtype=torch.int64, device=self.device)
            self.dist.all_reduce(bound, op=self.dist.ReduceOp.MAX)
            bound = (int(bound.item()) + 1) // 2 * 2            # keep every slot 16-byte aligned
            buf = self.symm.empty(q_max_slots(self.dist) * bound, dtype=torch.float64, device=self.device)
            handle = self.symm.rendezvous(buf, group=self.dist.group.WORLD)
            entry = self.cache[req.key] = (buf, handle, bound)
        buf, handle, bound = entry
        my_slots = [buf[s * bound:s * bound + req.count] for s in range(q)]
        targets = [handle.get_buffer(peer, (req.counts[d],), torch.float64, req.me * bound) if req.counts[d] else None
                   for d, peer in enumerate(req.group)]
        handle.barrier(channel=0)          # nobody is still summing the slots this sweep is about to overwrite
        self.last = handle
        return PeerSlotsReply(my_slots, targets)

    def barrier(self):
        self.last.barrier(channel=0)


def q_max_slots(dist) -> int:
    """Upper bound on a mode group's size: the world size (a grid extent cannot exceed it)."""
    return dist.get_world_size()


def run_rank(gen: Generator, dist, ops=None, to_tensor=lambda b: b, peer_slots: Optional[SymmetricSlots] = None):
    """Drive one rank program with torch.distributed (`dist`); buffers must be torch tensors of the right device.
    Pass the rank's `ops` so that the collectives queue on the engine's stream.  `peer_slots`: a SymmetricSlots
    provider turns the reduce-scatters into direct peer stores; without it they go through send/recv."""
    with _stream_of(ops):
        return _run_rank(gen, dist, to_tensor, peer_slots)


def _run_rank(gen: Generator, dist, to_tensor, peer_slots=None):
    try:
        req = next(gen)
        while True:
            if isinstance(req, Exchange):
                ops = [dist.P2POp(dist.isend, to_tensor(t), peer) for peer, t in req.sends]
                ops += [dist.P2POp(dist.irecv, to_tensor(t), peer) for peer, t in req.recvs]
                if ops:
                    for work in dist.batch_isend_irecv(ops):
                        work.wait()
            elif isinstance(req, AllReduce):
                dist.all_reduce(to_tensor(req.tensor))
            elif isinstance(req, Broadcast):
                dist.broadcast(to_tensor(req.tensor), src=req.root)
            elif isinstance(req, PeerSlots):
                # without a provider the program falls back to packed chunks + send/recv
                req = gen.send(peer_slots.slots(req) if peer_slots is not None else None)
                continue
            elif isinstance(req, GroupBarrier):
                if peer_slots is not None:
                    peer_slots.barrier()
                else:
                    dist.barrier()
            else:
                raise TypeError("unknown request %r" % (req,))
            req = gen.send(None)
    except StopIteration as stop:
        return stop.value


def run_virtual(gens: Sequence[Generator], ops=None, copy=lambda dst, src: dst.copy_(src),
                add=lambda dst, src: dst.add_(src)):
    """Step P rank programs in lock-step inside one process and perform their requests by direct copies.
    Pass the (shared) `ops` so that those copies queue on the engine's stream.

    All ranks must issue the same kind of request at each step (they do: the program is SPMD and data-independent).
    AllReduce sums in rank order into a scratch copy and hands every rank the same bits, as NCCL/gloo would."""
    with _stream_of(ops):
        return _run_virtual(gens, copy, add, ops.empty if ops is not None and hasattr(ops, "empty") else None)


def _run_virtual(gens, copy, add, alloc=None):
    if alloc is None:
        import torch
        alloc = lambda count: torch.empty(int(count), dtype=torch.float64)
    n = len(gens)
    results = [None] * n
    reqs = []
    live = [True] * n
    for r, g in enumerate(gens):
        try:
            reqs.append(next(g))
        except StopIteration as stop:
            reqs.append(None)
            live[r] = False
            results[r] = stop.value
    while any(live):
        kinds = {type(reqs[r]) for r in range(n) if live[r]}
        if len(kinds) != 1 or not all(live):
            raise RuntimeError("rank programs diverged: %s" % kinds)
        kind = kinds.pop()
        if kind is Exchange:
            posted = {}
            for r in range(n):
                for peer, t in reqs[r].sends:
                    posted.setdefault((r, peer), []).append(t)
            for r in range(n):
                for peer, t in reqs[r].recvs:
                    queue = posted.get((peer, r))
                    if not queue:
                        raise RuntimeError("rank %d expects a message from %d that was never sent" % (r, peer))
                    copy(t, queue.pop(0))
            if any(v for v in posted.values()):
                raise RuntimeError("unmatched sends")
        elif kind is AllReduce:
            total = reqs[0].tensor.clone()
            for r in range(1, n):
                add(total, reqs[r].tensor)
            for r in range(n):
                copy(reqs[r].tensor, total)
        elif kind is Broadcast:
            root = reqs[0].root
            for r in range(n):
                if r != root:
                    copy(reqs[r].tensor, reqs[root].tensor)
        elif kind is PeerSlots:
            # one address space: a "peer" slot is simply the other rank program's buffer
            slots = [[alloc(reqs[r].count) for _ in reqs[r].group] for r in range(n)]
            replies = [PeerSlotsReply(slots[r], [slots[peer][reqs[r].me] for peer in reqs[r].group]) for r in range(n)]
        elif kind is GroupBarrier:
            pass                      # lock-step: every rank program has issued its stores
        else:
            raise TypeError("unknown request %r" % (kind,))
        for r, g in enumerate(gens):
            try:
                reqs[r] = g.send(replies[r] if kind is PeerSlots else None)
            except StopIteration as stop:
                live[r] = False
                results[r] = stop.value
    return results


# ----------------------------------------------------------------------------------------------- regrid
def regrid_plan(ext: Sequence[int], src: GridLayout, dst: GridLayout, rank: int):
    """Who sends what when a tensor with extents `ext` moves from layout `src` to layout `dst` (the paper's regrid,
    PAPER.md:767; counted by simulate.hpp:97-113).  Returns (sends, recvs): lists of (peer, global slices)."""
    def overlap(a, b):
        out = []
        for (alo, ahi), (blo, bhi) in zip(a, b):
            lo, hi = max(alo, blo), min(ahi, bhi)
            if lo >= hi:
                return None
            out.append((lo, hi))
        return out

    def box(layout, r):
        return [layout.local_range(r, m, e) for m, e in enumerate(ext)]

    mine_src, mine_dst = box(src, rank), box(dst, rank)
    sends = [(p, o) for p in range(dst.procs) if (o := overlap(mine_src, box(dst, p)))]
    recvs = [(p, o) for p in range(src.procs) if (o := overlap(box(src, p), mine_dst))]
    return sends, recvs


def regrid(block, ext: Sequence[int], src: GridLayout, dst: GridLayout, rank: int, empty) -> Generator:
    """Generator: moves this rank's block (torch tensor shaped like its `src` block) to the `dst` layout."""
    sends, recvs = regrid_plan(ext, src, dst, rank)
    src_lo = [src.local_range(rank, m, e)[0] for m, e in enumerate(ext)]
    dst_lo = [dst.local_range(rank, m, e)[0] for m, e in enumerate(ext)]
    dst_dims = dst.local_dims(rank, ext)
    out = empty(int(np.prod(dst_dims, dtype=np.int64))).view(dst_dims)
    send_list, recv_list, local = [], [], None
    for peer, o in sends:
        piece = block[tuple(slice(lo - s, hi - s) for (lo, hi), s in zip(o, src_lo))]
        if peer == rank:
            local = (o, piece)
        else:
            send_list.append((peer, piece.contiguous().view(-1)))
    pending = []
    for peer, o in recvs:
        if peer == rank:
            continue
        shape = [hi - lo for lo, hi in o]
        buf = empty(int(np.prod(shape, dtype=np.int64)))
        recv_list.append((peer, buf))
        pending.append((o, buf, shape))
    yield Exchange(send_list, recv_list)
    if local is not None:
        o, piece = local
        out[tuple(slice(lo - s, hi - s) for (lo, hi), s in zip(o, dst_lo))].copy_(piece)
    for o, buf, shape in pending:
        out[tuple(slice(lo - s, hi - s) for (lo, hi), s in zip(o, dst_lo))].copy_(buf.view(shape))
    return out


# ----------------------------------------------------------------------------------------------- bench driver
class _DevicePointerView:
    """Zero-copy torch view of a library-owned device buffer (via __cuda_array_interface__)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def build_local_block(ctx, ops, cfg, layout: GridLayout, rank: int, dist, threads: int):
    """This rank's block of T = X + sigma E under `layout`.  Every rank generates a mode-0 slab range of the noise
    (the slab-parallel stream of workloads.py, or its slice of the single stream), assembles the matching rows of X
    on its GPU, and the ranks regrid from that mode-0 layout to the target grid (send/recv)."""
    import torch
    from . import engine as E, hostgen, workloads as W
    world = layout.procs
    gen_q = [world] + [1] * (layout.n - 1)
    if cfg.L[0] < world:
        raise ValueError("mode 0 is shorter than the process count")
    gen = GridLayout(gen_q)
    i0, i1 = gen.local_range(rank, 0, cfg.L[0])
    rest = list(cfg.L[1:])
    noise = np.empty([i1 - i0] + rest, dtype=np.float64)
    seed = 1000 * cfg.index + 3
    if cfg.slab_noise:
        from concurrent.futures import ThreadPoolExecutor
        flat = noise.reshape(i1 - i0, -1)
        with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
            list(pool.map(lambda i: hostgen.random_tensor(rest, seed + i0 + i, flat[i]), range(i1 - i0)))
    else:
        full = hostgen.random_tensor(cfg.L, seed)      # one sequential stream: generate, keep the slab range
        noise[...] = full[i0:i1]
        del full
    block = E.DeviceTensor.upload(ctx, noise)
    del noise
    x = E.DeviceTensor.upload(ctx, W.generating_core(cfg))
    for n, a in enumerate(W.generating_factors(cfg)):
        nxt = x.ttm(a[i0:i1] if n == 0 else a, n)
        x.free()
        x = nxt
    block.axpby(cfg.sigma, 1.0, x)
    x.free()
    ctx.synchronize()
    with torch.cuda.stream(ops.stream):
        view = torch.as_tensor(_DevicePointerView(block.device_ptr, block.size), device=ops.device).view(
            [i1 - i0] + rest)
        gen_dist = regrid(view, cfg.L, gen, layout, rank, ops.empty)
        local = run_rank(gen_dist, dist, ops) if dist is not None else run_virtual([gen_dist], ops)[0]
        local = local.contiguous().view(-1).clone()
    ctx.synchronize()
    block.free()
    return local


class _Clock:
    """Device-time marks on the engine's stream (CUDA events), or host time for the CPU contract test."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream

    def mark(self):
        if self.stream is None:
            return time.perf_counter()
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        return ev

    def ms(self, a, b):
        if self.stream is None:
            return (b - a) * 1e3
        b.synchronize()
        return a.elapsed_time(b)


def _timed_sweeps(dh, run, clock, steps):
    """K sweeps with per-node spans; returns (total_ms, tree_ms, core_ms, {node: ms}, last SweepResult), sums over K."""
    marks = []
    dh.events = lambda what, node: marks.append((what, node, clock.mark()))
    e0 = clock.mark()
    res = None
    for _ in range(steps):
        res = run(dh.sweep())
    e1 = clock.mark()
    dh.events = None
    total_ms = clock.ms(e0, e1)
    open_ev, node_ms, tree_ms, core_ms = {}, {}, 0.0, 0.0
    for what, node, ev in marks:
        if what.startswith("begin_"):
            open_ev[(what[6:], node)] = ev
            continue
        key = (what[4:], node)
        ms = clock.ms(open_ev.pop(key), ev)
        if key[0] in ("ttm", "regrid"):
            node_ms[node] = node_ms.get(node, 0.0) + ms
        elif key[0] == "tree":
            tree_ms += ms
        elif key[0] == "core":
            core_ms += ms
    return total_ms, tree_ms, core_ms, node_ms, res


def run_bench_rank(args, rank: int, world: int, local_rank: int):
    """bench.py for N >= 1 ranks under torchrun: one process per GPU, NCCL over NVLink.  With --backend numpy-test
    (CPU contract test only) the same rank program runs over gloo on the tests' NumPy stand-in for the kernels."""
    import json
    import torch
    import torch.distributed as dist
    from . import workloads as W
    import bench as B

    cuda = getattr(args, "backend", "cuda") == "cuda"
    if cuda:
        from . import engine as E
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group("gloo")
    cfg = W.CONFIGS[args.config]
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    cost = P.tree_cost(tree, spec)
    grid = P.optimal_static_grid(tree, spec, world)
    scheme = None
    if getattr(args, "grid", None) == "dynamic":       # per-node grids (grid_dynamic.hpp): regrid where it pays
        scheme = P.optimal_dynamic_scheme(tree, spec, world).scheme
        q = list(scheme.root)
    else:
        q = list(grid.grid) if not getattr(args, "grid", None) else [int(v) for v in args.grid.split("x")]
    node_q = (lambda node: scheme.node_grids[node]) if scheme else (lambda node: q)
    layout = GridLayout(q)
    hbm_gbs, hbm_src = B.read_peaks()
    cores = max(1, (os.cpu_count() or 1) // world)
    t0 = time.perf_counter()
    if cuda:
        p_fp64, fp64_src = B.measure_fp64_peak(torch)
        ctx = E.Context(local_rank)
        ops = GpuOps(ctx, local_rank)
        local = build_local_block(ctx, ops, cfg, layout, rank, dist, cores)
        clock = _Clock(torch, ops.stream)
        sync = ctx.synchronize
        launch_counts = ctx.launch_counts
        stat_device = ops.device
    else:
        from tests.numpy_ops import NumpyOps
        p_fp64, fp64_src = B.FP64_FALLBACK_TFLOPS, "not measured (numpy-test backend)"
        ctx, ops = None, NumpyOps()
        local = ops.from_host(np.ascontiguousarray(W.build_tensor_host(cfg, cores)[layout.slices(rank, cfg.L)]))
        clock = _Clock(torch, None)
        sync = lambda: None
        launch_counts = lambda: (0, 0)
        stat_device = torch.device("cpu")
    build_s = time.perf_counter() - t0
    dh = DistributedHooi(ops, spec, tree, scheme or q, rank)
    dh.set_local_tensor_buffer(local)
    f0 = W.start_factors(cfg)

    # --peer-slots: reduce-scatters as direct stores into NVLink-mapped peer slots (see SymmetricSlots)
    peer_slots = SymmetricSlots(dist, ops.device) if cuda and getattr(args, "peer_slots", False) else None

    def run(gen):
        return run_rank(gen, dist, ops, peer_slots=peer_slots)

    def measure(executor):
        """W warm-up + K timed sweeps of one HOOI run from the start factors; device time, max over ranks."""
        executor.set_factors(f0)
        for _ in range(max(args.warmup, 0)):
            run(executor.sweep())
        sync()
        dist.barrier()
        if cuda:
            torch.cuda.synchronize()
        total_ms, tree_ms, core_ms, node_ms, res = _timed_sweeps(executor, run, clock, args.steps)
        sync()
        dist.barrier()
        nodes = sorted(node_ms)
        stats = torch.tensor([total_ms, tree_ms, core_ms] + [node_ms[n] for n in nodes], dtype=torch.float64,
                             device=stat_device)
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)       # max over ranks
        stats = (stats / args.steps).tolist()
        return stats[0], stats[1], stats[2], dict(zip(nodes, stats[3:])), res

    k0, _ = launch_counts()
    sampler = B.ClockSampler(local_rank) if rank == 0 and cuda else None
    if sampler:
        sampler.start()
    ms_per_step, tree_phase_ms, core_ms, node_ms, res = measure(dh)
    clocks = sampler.stop() if sampler else None
    k1, lib_calls = launch_counts()
    fit, core_norm = run(dh.fit_from_norms())

    # the optimal grid against the uniform 2 x 2 x 2 grid (north_star, largest config at 8 GPUs): the local blocks are
    # redistributed to the other grid and the same measurement repeated
    comparison, compare_q = None, B.comparison_grid(spec.n_modes(), world, spec.K)
    if compare_q is not None and not scheme and not getattr(args, "no_grid_comparison", False) and compare_q != q:
        other = GridLayout(compare_q)
        with _stream_of(ops):
            moved = run(regrid(local.view(layout.local_dims(rank, cfg.L)), cfg.L, layout, other, rank, ops.empty))
            moved = moved.contiguous().view(-1)
        dh2 = DistributedHooi(ops, spec, tree, compare_q, rank)
        dh2.set_local_tensor_buffer(moved)
        ms2, tree2, core2, node2, res2 = measure(dh2)
        comparison = {"grid": compare_q, "ms_per_step": ms2, "tree_phase_ms": tree2,
                      "grid_volume_elements": P.static_volume(tree, spec, compare_q, world).total,
                      "per_node_ms": {str(k): v for k, v in node2.items()},
                      "optimal": {"grid": list(q), "ms_per_step": ms_per_step,
                                  "grid_volume_elements": P.static_volume(tree, spec, q, world).total}}
        del dh2, moved

    # e2e: per step the local block comes from pinned host memory and the result goes back to the host
    e2e = None
    if not args.no_e2e:
        host_block = torch.empty(local.numel(), dtype=torch.float64, pin_memory=cuda)
        with _stream_of(ops):
            host_block.copy_(local)
        sync()
        dh.set_factors(f0)
        dist.barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            with _stream_of(ops):
                local.copy_(host_block, non_blocking=True)
            dh.invalidate()
            dh.set_factors(dh.get_factors() if dh.core is not None else f0)
            run(dh.sweep())
            dh.get_factors()
            dh.get_local_core()
        sync()
        dist.barrier()
        secs = torch.tensor([(time.perf_counter() - w0) / args.steps], dtype=torch.float64, device=stat_device)
        dist.all_reduce(secs, op=dist.ReduceOp.MAX)
        fbytes = 8 * sum(l * k for l, k in zip(spec.L, spec.K))
        e2e = {"value": float(secs.item()), "unit": "s/iter", "h2d_bytes_per_step": int(local.numel() * 8 + fbytes) * world,
               "d2h_bytes_per_step": int(fbytes * world + 8 * int(np.prod(spec.K))), "host_memory": "pinned" if cuda else "pageable"}

    # CPU baseline + parity: the oracle runs the config's iterations on rank 0's host cores from the start factors; the
    # grid executor runs the same iterations on all ranks and is compared after every one of them
    cpu, parity_ok = None, True
    if not args.no_cpu:
        dh.set_factors(f0)

        def grid_step():
            run(dh.sweep())
            gfit, gnorm = run(dh.fit_from_norms())
            return dh.get_factors(), gnorm, gfit

        # every rank steps the executor exactly `iters` times (each step is a sequence of collectives); only rank 0
        # also runs the oracle, without a time budget so that the count cannot differ between ranks
        iters = cfg.iterations
        if rank == 0:
            host_t = W.build_tensor_host(cfg, os.cpu_count() or 1)
            result = B.oracle_run_with_parity(host_t, spec, tree, f0, iters, grid_step, budget_s=float("inf"))
            parity_ok = result["ok"]
            cpu = {"value": float(np.mean(result["secs"])), "unit": "s/iter", "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": "the %d HOOI iterations of %s from the start factors (NumPy/OpenBLAS oracle port) on "
                             "rank 0's host, mean per iteration" % (iters, cfg.name),
                   "phases_s": result["phases"], "parity_per_iteration": result["rows"], "parity_ok": parity_ok}
        else:
            for _ in range(iters):
                grid_step()
        verdict = torch.tensor([1 if parity_ok else 0], dtype=torch.int64, device=stat_device)
        dist.broadcast(verdict, src=0)          # every rank exits with rank 0's verdict
        parity_ok = bool(verdict.item())

    if rank == 0:
        # per-TTM roofline on P GPUs: flops / P, local bytes 8 (|In| + q_n |Out|) / P, plus the
        # reduce-scatter bytes 8 (q_n - 1) |Out| / P over NVLink when the grid splits the contracted mode
        rows, t_roof, flops_total = [], 0.0, 0
        for node, kind in enumerate(tree.kind):
            if kind != P.MODE:
                continue
            n = tree.mode[node]
            flops = 2 * spec.K[n] * cost.card_in[node]
            qn = node_q(node)[n]
            local_bytes = 8 * (cost.card_in[node] + qn * cost.card_out[node]) / world + 8 * spec.K[n] * spec.L[n]
            link_bytes = 8 * (qn - 1) * cost.card_out[node] / world
            if scheme:
                up = tree.parent[node]
                if list(node_q(node)) != list(q if tree.kind[up] == P.ROOT else node_q(up)):
                    link_bytes += 8 * cost.card_in[node] / world        # regrid: the model ships the whole input
            t = max(flops / world / (p_fp64 * 1e12), local_bytes / (hbm_gbs * 1e9)) + link_bytes / (B.NVLINK_GBS * 1e9)
            t_roof += t
            flops_total += flops
            ms = node_ms.get(node, 0.0)
            rows.append({"node": node, "mode": n, "ms": ms, "roofline_ms": t * 1e3, "frac": t * 1e3 / ms if ms else None,
                         "nvlink_bytes_per_gpu": link_bytes})
        ttm_ms = sum(r["ms"] for r in rows)
        dom = max(rows, key=lambda r: r["ms"])
        dom_flops = 2 * spec.K[dom["mode"]] * cost.card_in[dom["node"]]
        achieved = dom_flops / (dom["ms"] * 1e-3) / 1e12 if dom["ms"] else None
        volume = (P.scheme_volume(tree, spec, scheme, world).total if scheme
                  else P.static_volume(tree, spec, q, world).total)
        line = {
            "metric": "hooi_s_per_iter", "value": ms_per_step * 1e-3, "unit": "s/iter", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": B.shared_config(cfg.name, cfg.iterations, tree.label(), world, q, volume if world > 1 else 0,
                                      "x".join(map(str, compare_q)) if compare_q else None),
            "engine": {"timed_steps": "iterations W+1..W+K of one HOOI run from the random orthonormal start",
                       "core": "chain along a tree path, partial products carried into the next sweep",
                       "node_grids": {str(k): list(v) for k, v in scheme.node_grids.items()} if scheme else None,
                       "l2": "inputs_larger_than_L2", "noise": "slab-parallel" if cfg.slab_noise else "sequential",
                       "evd": "each leaf solved by its owner rank (leaves round-robin in walk order) on a side stream, "
                              "factor + status broadcast" if world > 1 else "solved on a side stream",
                       "reduce_scatter": "peer-slot stores from the TTM epilogue" if peer_slots else
                                         "destination-major partial product + grouped send/recv + ordered sum",
                       "backend": "cuda + nccl" if cuda else "numpy-test + gloo (contract test, not a measurement)"},
            "ttm_tree": {"tflops": flops_total / (ttm_ms * 1e-3) / 1e12 if ttm_ms else None,
                         "roofline_frac": t_roof * 1e3 / ttm_ms if ttm_ms else None, "measured_ms": ttm_ms,
                         "roofline_ms": t_roof * 1e3, "flops": flops_total, "p_fp64_tflops": p_fp64,
                         "p_fp64_source": fp64_src, "hbm_gbs": hbm_gbs, "hbm_source": hbm_src,
                         "nvlink_gbs": B.NVLINK_GBS, "per_node": rows,
                         "note": "per-node time = (regrid +) local kernel + chunk exchange + ordered reduction, max over ranks"},
            "phases_ms": {"tree_phase_incl_leaves": tree_phase_ms, "core_ms": core_ms},
            "grid_comparison": comparison,
            "relative_fit": fit, "core_norm": core_norm, "build_s": build_s,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": p_fp64 * world, "unit": "TFLOP/s",
                         "frac": achieved / (p_fp64 * world) if achieved else None, "traffic": None,
                         "kernel": "ttm_dmma_kernel (tree node %d, mode %d) across %d GPUs" % (dom["node"], dom["mode"] + 1, world),
                         "peak_source": fp64_src},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(k1 - k0), "library_calls": int(lib_calls),
            "clocks": clocks, "degenerate": bool(res.degenerate),
            "volume_sent_rank0": {str(k): v for k, v in res.volume_sent.items()},
            "regrid_sent_rank0": {str(k): v for k, v in res.regrid_sent.items()},
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    if not parity_ok:
        print("bench.py: parity against the oracle FAILED, see cpu_baseline.parity_per_iteration", file=sys.stderr)
        return 3
    return 0
