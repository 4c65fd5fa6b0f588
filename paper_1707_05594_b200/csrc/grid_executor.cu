// HOOI on a Cartesian processor grid inside ONE process: P ranks, one CUDA device each, tensors block-distributed,
// factors replicated.  This is the paper's distribution scheme (PAPER.md:576-593 Cartesian blocks, :582-588 the
// reduce-scatter after a product along a split mode, :628-754 per-node grids with regrids) executed for real behind the
// C ABI (tp_grid_*), so that a C++ caller of the reference API -- or the command line's `hooi --procs P` -- can use
// every GPU of the box.  The reference only simulates this (simulate.hpp) and charges (q_n - 1)|Out_u| elements per
// TTM (grid_volume.hpp:41) and |In_u| per regrid (grid_dynamic.hpp:37-62).
//
// Data plane: peer memory over NVLink, no staging and no collective library on the critical path.
//   * product along a split mode: every rank's TTM kernel writes its partial product destination-major, each chunk
//     straight into the receive slot of the rank that owns those core rows (tp_dev_ttm_scatter: the kernel's epilogue
//     IS the send of the reduce-scatter); an event per rank says "my stores are out", and each owner then adds its
//     q_n slots in group order (fixed order: bit-reproducible);
//   * leaf: local Gram kernels; the leaf's owner rank (leaves round-robin in walk order) adds the partial Gram
//     matrices in rank order reading them from peer memory, runs the certified top-k solve on a side stream
//     (tp_dev_leaf_solve_begin), and copies the new factor into every rank's replica;
//   * regrid between a node's grid and its parent's: every destination rank pulls the boxes its new block overlaps
//     from the peers' old blocks (tp_dev_copy_box reading peer memory);
//   * cross-rank ordering is CUDA events between the ranks' streams; the host only enqueues.
// Ranks may share a device ("virtual ranks": the same code path on one GPU, where a peer pointer is an ordinary
// device pointer) -- that is how the executor is tested on a single-GPU box.
// TP_GRID_NCCL switches the leaf all-reduce and the factor broadcast to NCCL (ncclCommInitAll, loaded at run time);
// it needs one distinct device per rank.
//
// Schedule and carried path follow the single-GPU plan (engine.cu) and paper_1707_05594_b200/distributed.py, which
// stays as the torch.distributed (one process per GPU) harness: Jacobi walk in stored child order, core chain along
// the path to the first leaf with the new factors, its partial products kept as the next sweep's tree nodes.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"
#include "planner.hpp"

using namespace tpb;

namespace {

#define TPG_CUDA(expr)                                                                             \
  do {                                                                                             \
    cudaError_t tpg_e_ = (expr);                                                                   \
    if (tpg_e_ != cudaSuccess) raise(TP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(tpg_e_)); \
  } while (0)

// forwards a C-ABI status of a building block as this call's failure
void ok(int status) {
  if (status != TP_OK) raise(status, tp_last_error(), tp_last_error_mode());
}

using Dims = std::vector<size_t>;

size_t volume(const Dims& d) {
  size_t v = 1;
  for (size_t e : d) v *= e;
  return v;
}

// Block distribution induced by one grid: floor cuts per mode (grid.hpp:114-119), ranks number the blocks row-major
// (simulate.hpp:69-73).
struct Layout {
  Grid q;
  int n = 0;
  int procs = 1;

  explicit Layout(const Grid& grid = {}) : q(grid), n(static_cast<int>(grid.size())) {
    for (u64 v : q) procs *= static_cast<int>(v);
  }
  std::vector<int> coords(int rank) const {
    std::vector<int> c(n, 0);
    for (int m = n - 1; m >= 0; --m) {
      c[m] = rank % static_cast<int>(q[m]);
      rank /= static_cast<int>(q[m]);
    }
    return c;
  }
  int rank_of(const std::vector<int>& c) const {
    int r = 0;
    for (int m = 0; m < n; ++m) r = r * static_cast<int>(q[m]) + c[m];
    return r;
  }
  // [lo, hi) of the rank's block on `mode` of a tensor whose extent there is ext
  std::pair<size_t, size_t> range(int rank, int mode, u64 ext) const {
    const std::vector<u64> cuts = block_bounds(ext, q[mode]);
    const int c = coords(rank)[mode];
    return {static_cast<size_t>(cuts[c]), static_cast<size_t>(cuts[c + 1])};
  }
  Dims local_dims(int rank, const std::vector<u64>& ext) const {
    Dims d(n);
    for (int m = 0; m < n; ++m) {
      const auto r = range(rank, m, ext[m]);
      d[m] = r.second - r.first;
    }
    return d;
  }
  Dims local_origin(int rank, const std::vector<u64>& ext) const {
    Dims d(n);
    for (int m = 0; m < n; ++m) d[m] = range(rank, m, ext[m]).first;
    return d;
  }
  // ranks that share every coordinate but `mode`, ordered by their mode coordinate
  std::vector<int> group(int rank, int mode) const {
    std::vector<int> c = coords(rank), out;
    for (int v = 0; v < static_cast<int>(q[mode]); ++v) {
      c[mode] = v;
      out.push_back(rank_of(c));
    }
    return out;
  }
  bool same(const Layout& o) const { return q == o.q; }
};

// ---- NCCL, loaded at run time (torch ships its own libnccl.so.2; linking a second copy would clash) --------------
struct Nccl {
  using Comm = void*;
  int (*CommInitAll)(Comm*, int, const int*) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  void* handle = nullptr;
  static constexpr int kFloat64 = 8, kSum = 0;  // ncclDataType_t / ncclRedOp_t values (nccl.h)

  bool load() {
    if (handle) return true;
    handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!handle) handle = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!handle) return false;
    auto sym = [&](const char* name) { return dlsym(handle, name); };
    CommInitAll = reinterpret_cast<decltype(CommInitAll)>(sym("ncclCommInitAll"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    Broadcast = reinterpret_cast<decltype(Broadcast)>(sym("ncclBroadcast"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    return CommInitAll && CommDestroy && AllReduce && Broadcast && GroupStart && GroupEnd;
  }
  void check(int status, const char* what) const {
    if (status != 0)
      raise(TP_ERR_NCCL, std::string(what) + ": " + (GetErrorString ? GetErrorString(status) : "nccl error"));
  }
};

struct Rank {
  int device = 0;
  tp_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  double* tensor = nullptr;
  Dims tensor_dims;
  std::vector<double*> cur, fresh;       // replicated factors, L_n x K_n column-major
  std::vector<double*> gram;             // per mode: this rank's partial Gram matrix (L_n x L_n)
  std::vector<double*> gram_sum;         // per mode, on the leaf's owner only: the reduced Gram matrix
  std::vector<int*> status;              // per mode, owner only: {degenerate flag, solver info}
  double* core = nullptr;
  Dims core_dims;
  double* scalar = nullptr;              // one double for norm reductions
  cudaEvent_t walk_done = nullptr;
};

// One tensor of the sweep: a block per rank under a layout.
struct Piece {
  std::vector<double*> ptr;
  std::vector<Dims> ldims;
  std::vector<u64> ext;
  const Layout* lay = nullptr;
  std::vector<cudaEvent_t> ready;        // per rank; nullptr = complete since before the sweep (the input tensor)
};

struct NodeState {
  Layout lay;                            // the node's own grid
  bool regrids = false;                  // its grid differs from its parent's: the input is redistributed first
  Piece moved;                           // the regridded input (buffers owned here)
  Piece out;                             // the node's product (buffers owned here)
  std::vector<std::vector<double*>> slots;  // per rank: q_n receive slots (split mode only)
  std::vector<size_t> mine;              // per rank: elements of its own chunk
  std::vector<cudaEvent_t> scattered;    // per rank: its partial-product stores are out
  std::vector<cudaEvent_t> reduced;      // per rank: its slots have been consumed
  std::vector<cudaEvent_t> begin, end;   // timing
  u64 sent_ttm = 0, sent_regrid = 0;     // elements shipped in the last sweep, all ranks
  u64 pending_ttm = 0, pending_regrid = 0;  // shipped by the last core chain for a product the NEXT sweep consumes
  bool carried = false;                  // `out` already holds this sweep's product (from the previous core chain)
  float ms = 0.f;
};

}  // namespace

struct tp_grid {
  Spec spec;
  Tree tree;
  int n = 0, procs = 1;
  Layout root;
  std::vector<Rank> ranks;
  std::vector<NodeState> nodes;
  std::vector<int> carry_path;           // TTM nodes from the root to the first leaf in walk order
  int carry_leaf_mode = -1;
  Cost cost;
  Cards cards;
  bool use_nccl = false;
  Nccl nccl;
  std::vector<Nccl::Comm> comms;
  // leaves in flight during a sweep
  struct Pending {
    int owner = 0, lane = 0;
    bool begun = false;                  // the solve is in flight on the owner's side stream `lane`
    bool collected = false;              // its factor has been (queued to be) copied to every rank this sweep
  };
  std::vector<Pending> pending;          // per mode
  std::vector<int> lane_mode;            // per owner x 4 lanes: the mode whose solve occupies the lane, -1 if free
  std::vector<int> owner_leaves;         // per owner: leaves assigned this sweep
  std::vector<cudaEvent_t> gram_done;    // per mode x rank
  std::vector<cudaEvent_t> factor_out;   // per mode: the owner's broadcast copies are queued
  int leaves_seen = 0;
  int fast_solves = 0;
  tp_sweep_stats model{};
  float last_total_ms = 0.f;
  cudaEvent_t sweep_begin = nullptr, sweep_end = nullptr;
  bool have_factors = false, have_tensor = false;
  std::vector<std::pair<int, double*>> scratch;  // (rank, buffer) allocated during a sweep, released at its end
};

namespace {

void on(const Rank& r) { TPG_CUDA(cudaSetDevice(r.device)); }

double* device_doubles(const Rank& r, size_t count) {
  on(r);
  double* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(TP_ERR_CUDA, "cudaMalloc of " + std::to_string(count * 8) + " bytes on device " + std::to_string(r.device) +
                           ": " + cudaGetErrorString(e));
  }
  return p;
}

cudaEvent_t new_event(const Rank& r, bool timing = false) {
  on(r);
  cudaEvent_t e = nullptr;
  TPG_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  return e;
}

void record(const Rank& r, cudaEvent_t e) {
  on(r);
  TPG_CUDA(cudaEventRecord(e, r.stream));
}

void wait(const Rank& r, cudaEvent_t e) {
  if (!e) return;
  on(r);
  TPG_CUDA(cudaStreamWaitEvent(r.stream, e, 0));
}

// Products kept from the last core chain are functions of (tensor, factors): forget them when either changes.
void invalidate(tp_grid* g) {
  for (Rank& rk : g->ranks)
    if (rk.ctx) ok(tp_dev_leaf_solve_reset(rk.ctx));  // a new run starts its solves from its own factors
  for (NodeState& st : g->nodes) {
    st.carried = false;
    st.pending_ttm = st.pending_regrid = 0;
  }
}

// The piece a node consumes before any regrid: its parent's product, or the input tensor below the root.
Piece input_piece(tp_grid* g) {
  Piece p;
  p.ext = g->spec.L;
  p.lay = &g->root;
  for (const Rank& r : g->ranks) {
    p.ptr.push_back(r.tensor);
    p.ldims.push_back(r.tensor_dims);
    p.ready.push_back(nullptr);
  }
  return p;
}

// Moves `src` to layout `to` into the preallocated piece `dst`: every rank pulls, box by box, what its new block
// shares with the peers' old blocks.  Returns the elements that crossed ranks.
u64 regrid(tp_grid* g, const Piece& src, Piece& dst, const Layout& to) {
  u64 shipped = 0;
  const int n = g->n;
  for (int r = 0; r < g->procs; ++r) {
    const Dims my_lo = to.local_origin(r, src.ext);
    const Dims& my_dims = dst.ldims[r];
    for (int s = 0; s < g->procs; ++s) {
      const Dims their_lo = src.lay->local_origin(s, src.ext);
      const Dims& their_dims = src.ldims[s];
      Dims box(n), dlo(n), slo(n);
      bool empty = false;
      for (int m = 0; m < n; ++m) {
        const size_t lo = std::max(my_lo[m], their_lo[m]);
        const size_t hi = std::min(my_lo[m] + my_dims[m], their_lo[m] + their_dims[m]);
        if (hi <= lo) {
          empty = true;
          break;
        }
        box[m] = hi - lo;
        dlo[m] = lo - my_lo[m];
        slo[m] = lo - their_lo[m];
      }
      if (empty) continue;
      wait(g->ranks[r], src.ready[s]);
      ok(tp_dev_copy_box(g->ranks[r].ctx, dst.ptr[r], my_dims.data(), dlo.data(), src.ptr[s], their_dims.data(),
                         slo.data(), box.data(), n));
      if (s != r) shipped += volume(box);
    }
    record(g->ranks[r], dst.ready[r]);
  }
  return shipped;
}

// Product of `in` (on the node's layout) with the mode's factor into the node's `out` piece.  `new_factors`: the
// core chain multiplies by the factors this sweep produced.
void product(tp_grid* g, int node, const Piece& in, bool new_factors) {
  NodeState& st = g->nodes[node];
  const int mode = g->tree.mode[node];
  const Layout& lay = st.lay;
  const int qn = static_cast<int>(lay.q[mode]);
  const size_t K = static_cast<size_t>(g->spec.K[mode]), L = static_cast<size_t>(g->spec.L[mode]);
  const std::vector<u64> kcuts64 = block_bounds(g->spec.K[mode], lay.q[mode]);
  const std::vector<size_t> kcuts(kcuts64.begin(), kcuts64.end());
  for (int r = 0; r < g->procs; ++r) {
    Rank& rk = g->ranks[r];
    const double* factor = (new_factors ? rk.fresh : rk.cur)[mode];
    const size_t l0 = lay.range(r, mode, in.ext[mode]).first;
    wait(rk, in.ready[r]);
    record(rk, st.begin[r]);
    if (qn == 1) {
      const size_t whole[2] = {0, K};
      ok(tp_dev_ttm_partial(rk.ctx, in.ptr[r], g->n, in.ldims[r].data(), mode, factor, L, l0, K, 1, whole,
                            st.out.ptr[r]));
      record(rk, st.end[r]);
      record(rk, st.out.ready[r]);
      continue;
    }
    // split mode: chunk d of the partial product goes straight into group member d's slot number `me`
    const std::vector<int> group = lay.group(r, mode);
    const int me = lay.coords(r)[mode];
    std::vector<double*> targets(qn, nullptr);
    for (int d = 0; d < qn; ++d) {
      wait(rk, st.reduced[group[d]]);  // the owner is done with what this slot held before (no-op if never used)
      targets[d] = st.slots[group[d]][me];
    }
    ok(tp_dev_ttm_scatter(rk.ctx, in.ptr[r], g->n, in.ldims[r].data(), mode, factor, L, l0, K, qn, kcuts.data(),
                          targets.data()));
    record(rk, st.scattered[r]);
    const size_t per_row = volume(in.ldims[r]) / in.ldims[r][mode];
    st.sent_ttm += static_cast<u64>(per_row) * (K - (kcuts[me + 1] - kcuts[me]));
  }
  if (qn == 1) return;
  for (int r = 0; r < g->procs; ++r) {
    Rank& rk = g->ranks[r];
    for (int d : lay.group(r, mode)) wait(rk, st.scattered[d]);
    std::vector<const double*> slots(st.slots[r].begin(), st.slots[r].end());
    ok(tp_dev_reduce_slots(rk.ctx, st.out.ptr[r], slots.data(), qn, st.mine[r]));
    record(rk, st.reduced[r]);
    record(rk, st.end[r]);
    record(rk, st.out.ready[r]);
  }
}

// Leaf of `mode` below the piece y: partial Gram matrices, the owner's ordered sum, the solve on its side stream.
void collect(tp_grid* g, int mode);

void leaf(tp_grid* g, int mode, const Piece& y) {
  const Layout& lay = *y.lay;
  const int qn = static_cast<int>(lay.q[mode]);
  const size_t rows = static_cast<size_t>(g->spec.L[mode]);
  const int k = static_cast<int>(g->spec.K[mode]);
  std::vector<int> contributors;
  for (int r = 0; r < g->procs; ++r) {
    Rank& rk = g->ranks[r];
    const Dims& d = y.ldims[r];
    size_t outer = 1, inner = 1;
    for (int m = 0; m < mode; ++m) outer *= d[m];
    for (int m = mode + 1; m < g->n; ++m) inner *= d[m];
    cudaEvent_t done = g->gram_done[mode * g->procs + r];
    if (qn == 1) {
      wait(rk, y.ready[r]);
      ok(tp_dev_gram(rk.ctx, y.ptr[r], outer, rows, inner, rk.gram[mode]));
      record(rk, done);
      contributors.push_back(r);
      continue;
    }
    // the unfolding's rows are split over the mode group: its first rank pulls the slices from the peers and owns
    // these columns of the unfolding; the other members add nothing to the Gram sum
    if (lay.coords(r)[mode] != 0) continue;
    const std::vector<int> group = lay.group(r, mode);
    const std::vector<u64> cuts = block_bounds(g->spec.L[mode], lay.q[mode]);
    double* full = device_doubles(rk, outer * rows * inner);
    for (int dth = 0; dth < qn; ++dth) {
      const int peer = group[dth];
      wait(rk, y.ready[peer]);
      ok(tp_dev_assemble_mode(rk.ctx, full, outer, rows, inner, y.ptr[peer], static_cast<size_t>(cuts[dth]),
                              static_cast<size_t>(cuts[dth + 1] - cuts[dth])));
    }
    ok(tp_dev_gram(rk.ctx, full, outer, rows, inner, rk.gram[mode]));
    record(rk, done);
    g->scratch.emplace_back(r, full);
    contributors.push_back(r);
  }
  tp_grid::Pending& job = g->pending[mode];
  job.owner = g->procs > 1 ? g->leaves_seen % g->procs : 0;
  job.lane = g->owner_leaves[job.owner]++ % 4;
  ++g->leaves_seen;
  // an owner has four side streams: a fifth leaf of the same owner first completes the one that holds its lane
  int& occupant = g->lane_mode[job.owner * 4 + job.lane];
  if (occupant >= 0) collect(g, occupant);
  occupant = mode;
  Rank& owner = g->ranks[job.owner];
  if (g->use_nccl && qn == 1) {
    // all-reduce of the partial Gram matrices over every rank (in place), one group call for the whole process
    g->nccl.check(g->nccl.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < g->procs; ++r)
      g->nccl.check(g->nccl.AllReduce(g->ranks[r].gram[mode], g->ranks[r].gram[mode], rows * rows, Nccl::kFloat64,
                                      Nccl::kSum, g->comms[r], g->ranks[r].stream),
                    "ncclAllReduce");
    g->nccl.check(g->nccl.GroupEnd(), "ncclGroupEnd");
    on(owner);
    TPG_CUDA(cudaMemcpyAsync(owner.gram_sum[mode], owner.gram[mode], sizeof(double) * rows * rows,
                             cudaMemcpyDeviceToDevice, owner.stream));
  } else {
    std::vector<const double*> parts;
    for (int r : contributors) {
      wait(owner, g->gram_done[mode * g->procs + r]);
      parts.push_back(g->ranks[r].gram[mode]);
    }
    ok(tp_dev_reduce_slots(owner.ctx, owner.gram_sum[mode], parts.data(), static_cast<int>(parts.size()), rows * rows));
  }
  // the same leaf lands on the same owner and lane every sweep, so the lane's accepted Ritz vectors start the next one
  ok(tp_dev_leaf_solve_begin_ex(owner.ctx, owner.gram_sum[mode], rows, k, owner.cur[mode], owner.fresh[mode],
                                owner.status[mode], owner.status[mode] + 1, job.lane, TP_LEAF_CONTINUE));
  job.begun = true;
  job.collected = false;
}

// New factor of `mode` on every rank: finish the owner's solve (certificate check, full-solve fallback), then copy.
void collect(tp_grid* g, int mode) {
  tp_grid::Pending& job = g->pending[mode];
  if (job.collected) return;
  if (!job.begun) raise(TP_ERR_INTERNAL, "core chain reached a mode whose leaf has not been visited");
  job.collected = true;
  g->lane_mode[job.owner * 4 + job.lane] = -1;
  Rank& owner = g->ranks[job.owner];
  int used_fast = 0;
  ok(tp_dev_leaf_solve_finish(owner.ctx, job.lane, owner.fresh[mode], owner.status[mode], owner.status[mode] + 1,
                              &used_fast));
  g->fast_solves += used_fast;
  job.begun = false;
  const size_t bytes = sizeof(double) * g->spec.L[mode] * g->spec.K[mode];
  on(owner);
  if (g->use_nccl) {
    g->nccl.check(g->nccl.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < g->procs; ++r)
      g->nccl.check(g->nccl.Broadcast(owner.fresh[mode], g->ranks[r].fresh[mode], bytes / sizeof(double),
                                      Nccl::kFloat64, job.owner, g->comms[r], g->ranks[r].stream),
                    "ncclBroadcast");
    g->nccl.check(g->nccl.GroupEnd(), "ncclGroupEnd");
    return;
  }
  for (int r = 0; r < g->procs; ++r)
    if (r != job.owner)
      TPG_CUDA(cudaMemcpyAsync(g->ranks[r].fresh[mode], owner.fresh[mode], bytes, cudaMemcpyDefault, owner.stream));
  record(owner, g->factor_out[mode]);
  for (int r = 0; r < g->procs; ++r)
    if (r != job.owner) wait(g->ranks[r], g->factor_out[mode]);
}

// The piece node `node` multiplies: its parent's product, redistributed first where the grids differ.
const Piece& node_input(tp_grid* g, int node, const Piece& parent_out) {
  NodeState& st = g->nodes[node];
  if (!st.regrids) return parent_out;
  st.sent_regrid += regrid(g, parent_out, st.moved, st.lay);
  return st.moved;
}

void walk(tp_grid* g, int node, const Piece& here) {
  for (int c : g->tree.kids[node]) {
    if (g->tree.kind[c] == TP_NODE_LEAF) {
      leaf(g, g->tree.mode[c], here);
      continue;
    }
    NodeState& st = g->nodes[c];
    if (!st.carried) product(g, c, node_input(g, c, here), false);
    walk(g, c, st.out);
  }
}

void destroy(tp_grid* g) {
  if (!g) return;
  for (Rank& r : g->ranks) {
    if (r.ctx) {
      cudaSetDevice(r.device);
      tp_ctx_synchronize(r.ctx);
    }
  }
  auto drop_piece = [&](Piece& p) {
    for (size_t r = 0; r < p.ptr.size(); ++r) {
      cudaSetDevice(g->ranks[r].device);
      cudaFree(p.ptr[r]);
      if (p.ready[r]) cudaEventDestroy(p.ready[r]);
    }
  };
  for (NodeState& st : g->nodes) {
    drop_piece(st.moved);
    drop_piece(st.out);
    for (size_t r = 0; r < st.slots.size(); ++r) {
      cudaSetDevice(g->ranks[r].device);
      for (double* s : st.slots[r]) cudaFree(s);
    }
    for (auto* list : {&st.scattered, &st.reduced, &st.begin, &st.end})
      for (cudaEvent_t e : *list)
        if (e) cudaEventDestroy(e);
  }
  for (cudaEvent_t e : g->gram_done)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : g->factor_out)
    if (e) cudaEventDestroy(e);
  if (g->sweep_begin) cudaEventDestroy(g->sweep_begin);
  if (g->sweep_end) cudaEventDestroy(g->sweep_end);
  for (size_t r = 0; r < g->comms.size(); ++r)
    if (g->comms[r]) g->nccl.CommDestroy(g->comms[r]);
  for (Rank& r : g->ranks) {
    cudaSetDevice(r.device);
    cudaFree(r.tensor);
    cudaFree(r.core);
    cudaFree(r.scalar);
    for (auto* list : {&r.cur, &r.fresh, &r.gram, &r.gram_sum})
      for (double* p : *list) cudaFree(p);
    for (int* p : r.status) cudaFree(p);
    if (r.walk_done) cudaEventDestroy(r.walk_done);
    if (r.ctx) tp_ctx_destroy(r.ctx);
  }
  delete g;
}

}  // namespace

extern "C" {

int tp_grid_create(int n_ranks, const int* devices, int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes,
                   const int* kind, const int* mode, const int* parent, const tp_u64* root_grid,
                   const tp_u64* node_grids, unsigned flags, tp_grid** out) {
  return guarded([&] {
    if (!out || !devices || !root_grid) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    if (n_ranks < 1 || n_ranks > kMaxReduceSlots) raise(TP_ERR_BAD_ARGUMENT, "between 1 and 16 ranks");
    tp_grid* g = new tp_grid;
    try {
      g->spec = make_spec(n_modes, L, K);
      validate_spec(g->spec);
      g->n = n_modes;
      g->procs = n_ranks;
      g->tree = tree_from_arrays(n_modes, n_nodes, kind, mode, parent);
      validate_tree(g->tree, g->spec);
      for (int m = 0; m < n_modes; ++m)
        if (g->spec.L[m] > TP_MAX_GRAM_ROWS)
          raise(TP_ERR_TOO_LARGE, "unfolding has too many rows for the Gram route", m);  // hooi.hpp:48-49
      // the scheme: one grid per TTM node (the root grid where none is given); validated as the reference validates
      // a DynamicGridScheme (grid_dynamic.hpp:37-62)
      Scheme scheme;
      scheme.root.assign(root_grid, root_grid + n_modes);
      scheme.node.assign(g->tree.size(), Grid{});
      for (int id = 0; id < g->tree.size(); ++id)
        if (g->tree.internal(id))
          scheme.node[id] = node_grids ? Grid(node_grids + static_cast<size_t>(id) * n_modes,
                                              node_grids + static_cast<size_t>(id + 1) * n_modes)
                                       : scheme.root;
      scheme_volume(g->tree, g->spec, scheme, static_cast<u64>(n_ranks));
      g->root = Layout(scheme.root);
      g->cost = tree_cost(g->tree, g->spec, &g->cards);
      g->model.tree_macs = g->cost.total_macs;
      g->model.peak_live = g->cost.depth + 1;
      {
        u64 card = partial_cardinality(g->spec, 0), macs = 0;
        for (int m = 0; m < n_modes; ++m) {  // the ledger keeps the reference's mode order (hooi.hpp:93-100)
          macs = add_or_throw(macs, mul_or_throw(g->spec.K[m], card));
          card = scale_exact(card, g->spec.K[m], g->spec.L[m]);
        }
        g->model.core_macs = macs;
      }
      g->use_nccl = (flags & TP_GRID_NCCL) != 0;

      // ranks: one context per rank; peers map each other's memory
      g->ranks.resize(n_ranks);
      for (int r = 0; r < n_ranks; ++r) {
        Rank& rk = g->ranks[r];
        rk.device = devices[r];
        ok(tp_ctx_create(rk.device, &rk.ctx));
        void* s = nullptr;
        ok(tp_ctx_stream(rk.ctx, &s));
        rk.stream = static_cast<cudaStream_t>(s);
      }
      for (int a = 0; a < n_ranks; ++a)
        for (int b = 0; b < n_ranks; ++b) {
          if (devices[a] == devices[b]) continue;
          int can = 0;
          TPG_CUDA(cudaDeviceCanAccessPeer(&can, devices[a], devices[b]));
          if (!can)
            raise(TP_ERR_CUDA, "device " + std::to_string(devices[a]) + " cannot map the memory of device " +
                                   std::to_string(devices[b]) + " (no peer access)");
          TPG_CUDA(cudaSetDevice(devices[a]));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled)
            cudaGetLastError();
          else if (e != cudaSuccess)
            raise(TP_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        }
      if (g->use_nccl) {
        for (int a = 0; a < n_ranks; ++a)
          for (int b = a + 1; b < n_ranks; ++b)
            if (devices[a] == devices[b])
              raise(TP_ERR_NCCL, "TP_GRID_NCCL needs one distinct device per rank (NCCL refuses duplicate devices)");
        if (!g->nccl.load()) raise(TP_ERR_NCCL, "libnccl.so.2 could not be loaded");
        g->comms.assign(n_ranks, nullptr);
        g->nccl.check(g->nccl.CommInitAll(g->comms.data(), n_ranks, devices), "ncclCommInitAll");
      }

      // per-rank replicated state
      for (int r = 0; r < n_ranks; ++r) {
        Rank& rk = g->ranks[r];
        rk.tensor_dims = g->root.local_dims(r, g->spec.L);
        rk.tensor = device_doubles(rk, volume(rk.tensor_dims));
        rk.core_dims = g->root.local_dims(r, g->spec.K);
        rk.core = device_doubles(rk, volume(rk.core_dims));
        rk.scalar = device_doubles(rk, 1);
        rk.walk_done = new_event(rk);
        for (int m = 0; m < n_modes; ++m) {
          const size_t lk = static_cast<size_t>(g->spec.L[m] * g->spec.K[m]), ll = static_cast<size_t>(g->spec.L[m] * g->spec.L[m]);
          rk.cur.push_back(device_doubles(rk, lk));
          rk.fresh.push_back(device_doubles(rk, lk));
          rk.gram.push_back(device_doubles(rk, ll));
          rk.gram_sum.push_back(device_doubles(rk, ll));
          int* st = nullptr;
          on(rk);
          TPG_CUDA(cudaMalloc(&st, 2 * sizeof(int)));
          TPG_CUDA(cudaMemset(st, 0, 2 * sizeof(int)));
          rk.status.push_back(st);
        }
      }
      g->pending.assign(n_modes, tp_grid::Pending{});
      for (int m = 0; m < n_modes; ++m) {
        for (int r = 0; r < n_ranks; ++r) g->gram_done.push_back(new_event(g->ranks[r]));
        g->factor_out.push_back(new_event(g->ranks[0]));
      }
      on(g->ranks[0]);
      TPG_CUDA(cudaEventCreate(&g->sweep_begin));
      TPG_CUDA(cudaEventCreate(&g->sweep_end));

      // per-node buffers
      g->nodes.resize(g->tree.size());
      for (int id = 1; id < g->tree.size(); ++id) {
        if (!g->tree.internal(id)) continue;
        NodeState& st = g->nodes[id];
        st.lay = Layout(scheme.node[id]);
        const int md = g->tree.mode[id];
        const Layout& up = g->tree.kind[g->tree.parent[id]] == TP_NODE_ROOT ? g->root : g->nodes[g->tree.parent[id]].lay;
        st.regrids = !st.lay.same(up);
        const std::vector<u64> out_ext = node_extents(g->tree, g->spec, id);
        std::vector<u64> in_ext = out_ext;
        in_ext[md] = g->spec.L[md];
        auto make_piece = [&](Piece& p, const std::vector<u64>& ext) {
          p.ext = ext;
          p.lay = &st.lay;
          for (int r = 0; r < n_ranks; ++r) {
            p.ldims.push_back(st.lay.local_dims(r, ext));
            p.ptr.push_back(device_doubles(g->ranks[r], volume(p.ldims.back())));
            p.ready.push_back(new_event(g->ranks[r]));
          }
        };
        if (st.regrids) make_piece(st.moved, in_ext);
        make_piece(st.out, out_ext);
        const int qn = static_cast<int>(st.lay.q[md]);
        st.slots.assign(n_ranks, {});
        st.mine.assign(n_ranks, 0);
        for (int r = 0; r < n_ranks; ++r) {
          st.mine[r] = volume(st.out.ldims[r]);
          if (qn > 1)
            for (int d = 0; d < qn; ++d) st.slots[r].push_back(device_doubles(g->ranks[r], st.mine[r]));
          st.scattered.push_back(new_event(g->ranks[r]));
          st.reduced.push_back(new_event(g->ranks[r]));
          st.begin.push_back(new_event(g->ranks[r], true));
          st.end.push_back(new_event(g->ranks[r], true));
        }
      }
      // the path the core chain follows: down the first children to the first leaf in walk order
      for (int at = 0;;) {
        int leaf_child = -1;
        for (int c : g->tree.kids[at])
          if (g->tree.kind[c] == TP_NODE_LEAF) {
            leaf_child = c;
            break;
          }
        if (leaf_child >= 0) {
          g->carry_leaf_mode = g->tree.mode[leaf_child];
          break;
        }
        at = g->tree.kids[at][0];
        g->carry_path.push_back(at);
      }
      for (Rank& rk : g->ranks) ok(tp_ctx_synchronize(rk.ctx));
    } catch (...) {
      destroy(g);
      throw;
    }
    *out = g;
  });
}

int tp_grid_destroy(tp_grid* g) {
  return guarded([&] { destroy(g); });
}

int tp_grid_ranks(const tp_grid* g, int* n_ranks) {
  return guarded([&] {
    if (!g || !n_ranks) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    *n_ranks = g->procs;
  });
}

int tp_grid_block(const tp_grid* g, int rank, size_t* lo, size_t* dims) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    if (rank < 0 || rank >= g->procs) raise(TP_ERR_BAD_ARGUMENT, "rank outside the grid");
    const Dims origin = g->root.local_origin(rank, g->spec.L);
    for (int m = 0; m < g->n; ++m) {
      if (lo) lo[m] = origin[m];
      if (dims) dims[m] = g->ranks[rank].tensor_dims[m];
    }
  });
}

int tp_grid_set_block(tp_grid* g, int rank, const double* host_block) {
  return guarded([&] {
    if (!g || !host_block) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    if (rank < 0 || rank >= g->procs) raise(TP_ERR_BAD_ARGUMENT, "rank outside the grid");
    Rank& rk = g->ranks[rank];
    on(rk);
    TPG_CUDA(cudaMemcpyAsync(rk.tensor, host_block, volume(rk.tensor_dims) * sizeof(double), cudaMemcpyHostToDevice,
                             rk.stream));
    TPG_CUDA(cudaStreamSynchronize(rk.stream));
    invalidate(g);
    g->have_tensor = true;
  });
}

int tp_grid_set_tensor(tp_grid* g, const double* host_tensor) {
  return guarded([&] {
    if (!g || !host_tensor) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    // pack each rank's box on the host (runs of the innermost mode are contiguous), then one copy per rank
    const int n = g->n;
    std::vector<size_t> stride(n, 1);
    for (int m = n - 2; m >= 0; --m) stride[m] = stride[m + 1] * static_cast<size_t>(g->spec.L[m + 1]);
    for (int r = 0; r < g->procs; ++r) {
      Rank& rk = g->ranks[r];
      const Dims lo = g->root.local_origin(r, g->spec.L);
      const Dims& d = rk.tensor_dims;
      const size_t total = volume(d), run = d[n - 1];
      std::vector<double> packed(total);
      std::vector<size_t> at(n, 0);
      for (size_t done = 0; done < total; done += run) {
        size_t src = 0;
        for (int m = 0; m < n; ++m) src += (lo[m] + at[m]) * stride[m];
        std::memcpy(packed.data() + done, host_tensor + src, run * sizeof(double));
        for (int m = n - 2; m >= 0; --m) {
          if (++at[m] < d[m]) break;
          at[m] = 0;
        }
      }
      on(rk);
      TPG_CUDA(cudaMemcpyAsync(rk.tensor, packed.data(), total * sizeof(double), cudaMemcpyHostToDevice, rk.stream));
      TPG_CUDA(cudaStreamSynchronize(rk.stream));
    }
    invalidate(g);
    g->have_tensor = true;
  });
}

int tp_grid_set_factors(tp_grid* g, const double* const* factors) {
  return guarded([&] {
    if (!g || !factors) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    for (int m = 0; m < g->n; ++m)
      if (!factors[m]) raise(TP_ERR_SHAPE_MISMATCH, "factor count differs from mode count");
    for (Rank& rk : g->ranks) {
      on(rk);
      for (int m = 0; m < g->n; ++m)
        TPG_CUDA(cudaMemcpyAsync(rk.cur[m], factors[m], sizeof(double) * g->spec.L[m] * g->spec.K[m],
                                 cudaMemcpyHostToDevice, rk.stream));
      TPG_CUDA(cudaStreamSynchronize(rk.stream));
    }
    invalidate(g);
    g->have_factors = true;
  });
}

int tp_grid_get_factors(tp_grid* g, double* const* factors_out) {
  return guarded([&] {
    if (!g || !factors_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    Rank& rk = g->ranks[0];
    on(rk);
    for (int m = 0; m < g->n; ++m)
      TPG_CUDA(cudaMemcpyAsync(factors_out[m], rk.cur[m], sizeof(double) * g->spec.L[m] * g->spec.K[m],
                               cudaMemcpyDeviceToHost, rk.stream));
    TPG_CUDA(cudaStreamSynchronize(rk.stream));
  });
}

int tp_grid_sweep(tp_grid* g, tp_sweep_stats* stats) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    if (stats) *stats = tp_sweep_stats{};  // hooi.hpp:198
    if (!g->have_tensor || !g->have_factors) raise(TP_ERR_BAD_ARGUMENT, "set the tensor blocks and the factors first");
    for (NodeState& st : g->nodes) st.sent_ttm = st.sent_regrid = 0;
    g->leaves_seen = 0;
    g->lane_mode.assign(static_cast<size_t>(g->procs) * 4, -1);
    g->owner_leaves.assign(g->procs, 0);
    for (tp_grid::Pending& job : g->pending) job.begun = job.collected = false;
    record(g->ranks[0], g->sweep_begin);
    const Piece input = input_piece(g);
    walk(g, 0, input);
    // every peer read of a node's product (regrids, leaf gathers) precedes the core chain, which rewrites products
    for (Rank& rk : g->ranks) record(rk, rk.walk_done);
    for (Rank& rk : g->ranks)
      for (Rank& other : g->ranks)
        if (&other != &rk) wait(rk, other.walk_done);
    // core_from_factors (hooi.hpp:93-100) with the new factors along the path to the first leaf: its partial
    // products are the next sweep's tree nodes there (volumes are booked to the sweep that consumes them)
    std::vector<u64> carried_ttm(g->tree.size(), 0), carried_regrid(g->tree.size(), 0);
    const Piece* at = &input;
    for (int c : g->carry_path) {
      NodeState& st = g->nodes[c];
      collect(g, g->tree.mode[c]);
      const u64 t0 = st.sent_ttm, r0 = st.sent_regrid;
      product(g, c, node_input(g, c, *at), true);
      carried_ttm[c] = st.sent_ttm - t0;
      carried_regrid[c] = st.sent_regrid - r0;
      st.sent_ttm = t0;
      st.sent_regrid = r0;
      at = &st.out;
    }
    // the last product of the chain lands in the core; it runs on the grid of the path's last node (the root grid
    // for a one-node path) and the core lives on the root grid
    {
      const int md = g->carry_leaf_mode;
      collect(g, md);
      const Layout& lay = *at->lay;
      const int qn = static_cast<int>(lay.q[md]);
      const size_t K = static_cast<size_t>(g->spec.K[md]), L = static_cast<size_t>(g->spec.L[md]);
      std::vector<u64> core_ext = at->ext;
      core_ext[md] = g->spec.K[md];
      const std::vector<u64> kc64 = block_bounds(g->spec.K[md], lay.q[md]);
      const std::vector<size_t> kcuts(kc64.begin(), kc64.end());
      // scratch for this product: partial chunks land in per-rank slot buffers allocated for the call
      std::vector<std::vector<double*>> slots(g->procs);
      std::vector<double*> local(g->procs, nullptr);
      std::vector<Dims> ldims(g->procs);
      std::vector<cudaEvent_t> scattered(g->procs, nullptr), done(g->procs, nullptr);
      for (int r = 0; r < g->procs; ++r) {
        ldims[r] = lay.local_dims(r, core_ext);
        const bool direct = lay.same(g->root);  // the chain's last grid is the core's: write it in place
        local[r] = direct ? g->ranks[r].core : device_doubles(g->ranks[r], volume(ldims[r]));
        if (qn > 1)
          for (int d = 0; d < qn; ++d) slots[r].push_back(device_doubles(g->ranks[r], volume(ldims[r])));
        scattered[r] = new_event(g->ranks[r]);
        done[r] = new_event(g->ranks[r]);
      }
      for (int r = 0; r < g->procs; ++r) {
        Rank& rk = g->ranks[r];
        const size_t l0 = lay.range(r, md, at->ext[md]).first;
        wait(rk, at->ready[r]);
        if (qn == 1) {
          const size_t whole[2] = {0, K};
          ok(tp_dev_ttm_partial(rk.ctx, at->ptr[r], g->n, at->ldims[r].data(), md, rk.fresh[md], L, l0, K, 1, whole,
                                local[r]));
        } else {
          const std::vector<int> group = lay.group(r, md);
          const int me = lay.coords(r)[md];
          std::vector<double*> targets(qn);
          for (int d = 0; d < qn; ++d) targets[d] = slots[group[d]][me];
          ok(tp_dev_ttm_scatter(rk.ctx, at->ptr[r], g->n, at->ldims[r].data(), md, rk.fresh[md], L, l0, K, qn,
                                kcuts.data(), targets.data()));
        }
        record(rk, scattered[r]);
      }
      for (int r = 0; r < g->procs; ++r) {
        Rank& rk = g->ranks[r];
        if (qn > 1) {
          for (int d : lay.group(r, md)) wait(rk, scattered[d]);
          std::vector<const double*> src(slots[r].begin(), slots[r].end());
          ok(tp_dev_reduce_slots(rk.ctx, local[r], src.data(), qn, volume(ldims[r])));
        }
        record(rk, done[r]);
      }
      if (!lay.same(g->root)) {  // bring the core home to the root grid
        Piece from, to;
        from.ext = to.ext = core_ext;
        from.lay = &lay;
        to.lay = &g->root;
        for (int r = 0; r < g->procs; ++r) {
          from.ptr.push_back(local[r]);
          from.ldims.push_back(ldims[r]);
          from.ready.push_back(done[r]);
          to.ptr.push_back(g->ranks[r].core);
          to.ldims.push_back(g->ranks[r].core_dims);
          to.ready.push_back(new_event(g->ranks[r]));
        }
        regrid(g, from, to, g->root);
        for (cudaEvent_t e : to.ready) cudaEventDestroy(e);
      }
      // host: wait for everything, then release the scratch
      for (Rank& rk : g->ranks) ok(tp_ctx_synchronize(rk.ctx));
      for (int r = 0; r < g->procs; ++r) {
        cudaSetDevice(g->ranks[r].device);
        if (local[r] != g->ranks[r].core) cudaFree(local[r]);
        for (double* s : slots[r]) cudaFree(s);
        cudaEventDestroy(scattered[r]);
        cudaEventDestroy(done[r]);
      }
    }
    record(g->ranks[0], g->sweep_end);
    for (Rank& rk : g->ranks) ok(tp_ctx_synchronize(rk.ctx));
    for (const auto& item : g->scratch) {
      cudaSetDevice(g->ranks[item.first].device);
      cudaFree(item.second);
    }
    g->scratch.clear();
    // bookkeeping: this sweep consumed what the previous chain carried; what this chain shipped belongs to the next
    for (NodeState& st : g->nodes) st.carried = false;
    for (int c : g->carry_path) {
      NodeState& st = g->nodes[c];
      st.carried = true;
      st.sent_ttm += st.pending_ttm;
      st.sent_regrid += st.pending_regrid;
      st.pending_ttm = carried_ttm[c];
      st.pending_regrid = carried_regrid[c];
    }
    // timing, status, new factors become the current ones
    on(g->ranks[0]);
    TPG_CUDA(cudaEventElapsedTime(&g->last_total_ms, g->sweep_begin, g->sweep_end));
    int degenerate = 0;
    for (int m = 0; m < g->n; ++m) {
      Rank& owner = g->ranks[g->pending[m].owner];
      int host[2] = {0, 0};
      on(owner);
      TPG_CUDA(cudaMemcpy(host, owner.status[m], sizeof(host), cudaMemcpyDeviceToHost));
      TPG_CUDA(cudaMemset(owner.status[m], 0, sizeof(host)));
      if (host[1] != 0) raise(TP_ERR_TOO_LARGE, "eigensolver did not converge");  // hooi.hpp:56-57
      degenerate |= host[0];
    }
    for (NodeState& st : g->nodes) {
      st.ms = 0.f;
      for (size_t r = 0; r < st.begin.size(); ++r) {
        float ms = 0.f;
        cudaSetDevice(g->ranks[r].device);
        if (cudaEventElapsedTime(&ms, st.begin[r], st.end[r]) == cudaSuccess)
          st.ms = std::max(st.ms, ms);
        else
          cudaGetLastError();  // not recorded this sweep (a carried node)
      }
    }
    for (Rank& rk : g->ranks) std::swap(rk.cur, rk.fresh);
    if (stats) {
      *stats = g->model;
      stats->degenerate = degenerate;
    }
  });
}

int tp_grid_get_core(tp_grid* g, double* core_out) {
  return guarded([&] {
    if (!g || !core_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    const int n = g->n;
    std::vector<size_t> stride(n, 1);
    for (int m = n - 2; m >= 0; --m) stride[m] = stride[m + 1] * static_cast<size_t>(g->spec.K[m + 1]);
    for (int r = 0; r < g->procs; ++r) {
      Rank& rk = g->ranks[r];
      const Dims lo = g->root.local_origin(r, g->spec.K);
      const Dims& d = rk.core_dims;
      const size_t total = volume(d), run = d[n - 1];
      std::vector<double> packed(total);
      on(rk);
      TPG_CUDA(cudaMemcpy(packed.data(), rk.core, total * sizeof(double), cudaMemcpyDeviceToHost));
      std::vector<size_t> at(n, 0);
      for (size_t done = 0; done < total; done += run) {
        size_t dst = 0;
        for (int m = 0; m < n; ++m) dst += (lo[m] + at[m]) * stride[m];
        std::memcpy(core_out + dst, packed.data() + done, run * sizeof(double));
        for (int m = n - 2; m >= 0; --m) {
          if (++at[m] < d[m]) break;
          at[m] = 0;
        }
      }
    }
  });
}

int tp_grid_norms(tp_grid* g, double* tensor_norm, double* core_norm) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    double t2 = 0.0, c2 = 0.0;
    for (Rank& rk : g->ranks) {
      double part[2] = {0.0, 0.0};
      on(rk);
      ok(tp_dev_sum_squares(rk.ctx, rk.tensor, volume(rk.tensor_dims), rk.scalar));
      TPG_CUDA(cudaMemcpyAsync(&part[0], rk.scalar, sizeof(double), cudaMemcpyDeviceToHost, rk.stream));
      TPG_CUDA(cudaStreamSynchronize(rk.stream));
      ok(tp_dev_sum_squares(rk.ctx, rk.core, volume(rk.core_dims), rk.scalar));
      TPG_CUDA(cudaMemcpyAsync(&part[1], rk.scalar, sizeof(double), cudaMemcpyDeviceToHost, rk.stream));
      TPG_CUDA(cudaStreamSynchronize(rk.stream));
      t2 += part[0];  // rank order: deterministic
      c2 += part[1];
    }
    if (tensor_norm) *tensor_norm = std::sqrt(t2);
    if (core_norm) *core_norm = std::sqrt(c2);
  });
}

int tp_grid_fit_from_norms(tp_grid* g, double* out) {
  return guarded([&] {
    if (!g || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    double t = 0.0, c = 0.0;
    ok(tp_grid_norms(g, &t, &c));
    if (t == 0.0) raise(TP_ERR_ZERO_TENSOR, "relative error undefined at zero");  // hooi.hpp:233-234
    *out = std::sqrt(std::max(t * t - c * c, 0.0)) / t;
  });
}

int tp_grid_last_volumes(const tp_grid* g, int n_nodes, tp_u64* ttm_elements, tp_u64* regrid_elements) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    if (n_nodes != g->tree.size()) raise(TP_ERR_SHAPE_MISMATCH, "node count differs from the grid's tree");
    for (int i = 0; i < n_nodes; ++i) {
      if (ttm_elements) ttm_elements[i] = g->nodes[i].sent_ttm;
      if (regrid_elements) regrid_elements[i] = g->nodes[i].sent_regrid;
    }
  });
}

int tp_grid_last_timing(const tp_grid* g, float* total_ms, int n_nodes, float* node_ms, int* fast_solves) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    if (total_ms) *total_ms = g->last_total_ms;
    if (node_ms) {
      if (n_nodes != g->tree.size()) raise(TP_ERR_SHAPE_MISMATCH, "node count differs from the grid's tree");
      for (int i = 0; i < n_nodes; ++i) node_ms[i] = g->nodes[i].ms;
    }
    if (fast_solves) *fast_solves = g->fast_solves;
  });
}

int tp_grid_launch_counts(const tp_grid* g, tp_u64* own_kernels, tp_u64* library_calls) {
  return guarded([&] {
    if (!g) raise(TP_ERR_BAD_ARGUMENT, "null grid");
    tp_u64 own = 0, lib = 0;
    for (const Rank& rk : g->ranks) {
      tp_u64 a = 0, b = 0;
      ok(tp_ctx_launch_counts(rk.ctx, &a, &b));
      own += a;
      lib += b;
    }
    if (own_kernels) *own_kernels = own;
    if (library_calls) *library_calls = lib;
  });
}

}  // extern "C"
