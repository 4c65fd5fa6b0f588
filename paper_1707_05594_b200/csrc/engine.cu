// Device engine behind the C ABI: context, HBM-resident tensors, the TTM-tree
// executor (hooi_sweep), Gram + eigen-solve leaf updates, core and fit.
//
// Reference behaviour followed (proj/include/tuckerplan): ttm.hpp:73-96,
// hooi.hpp:45-76 (leaf update), :93-100 (core), :136-159 (Jacobi walk),
// :163-229 (Gauss-Seidel + sweep driver), :232-245 (reconstruction error).
//
// HBM layout: tensors are row-major FP64, exactly the reference's
// DenseTensor::data order; factors are L_n x K_n column-major (Eigen::MatrixXd
// order), which read as row-major is the K_n x L_n matrix F^T a tree TTM needs.
// A sweep never allocates: intermediates live in one buffer per tree depth
// (depth-first execution frees in tree order, so depth d has one live tensor),
// sized from the planner's node cardinalities.
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"
#include "planner.hpp"

namespace tpb {

[[noreturn]] static void cuda_fail(cudaError_t e, const char* what) {
  raise(TP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define TPB_CUDA(expr)                               \
  do {                                               \
    cudaError_t tpb_e_ = (expr);                     \
    if (tpb_e_ != cudaSuccess) cuda_fail(tpb_e_, #expr); \
  } while (0)
#define TPB_BLAS(expr)                                                                          \
  do {                                                                                          \
    cublasStatus_t tpb_b_ = (expr);                                                             \
    if (tpb_b_ != CUBLAS_STATUS_SUCCESS)                                                        \
      raise(TP_ERR_CUDA, std::string(#expr) + ": cublas status " + std::to_string(static_cast<int>(tpb_b_))); \
  } while (0)
#define TPB_SOLVER(expr)                                                                        \
  do {                                                                                          \
    cusolverStatus_t tpb_s_ = (expr);                                                           \
    if (tpb_s_ != CUSOLVER_STATUS_SUCCESS)                                                      \
      raise(TP_ERR_CUDA, std::string(#expr) + ": cusolver status " + std::to_string(static_cast<int>(tpb_s_))); \
  } while (0)

}  // namespace tpb

using namespace tpb;

struct tp_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  u64 own_kernels = 0;
  u64 library_calls = 0;
  double* reduce_scratch = nullptr;  // reduce_scratch_doubles() + 1 result slot
  double* frag_scratch = nullptr;    // fragment buffer for one-off TTMs
  size_t frag_capacity = 0;
  // side streams for the eigen-solves of a Jacobi sweep: the leaves are independent of each other and of the
  // remaining tree TTMs, and an eigen-solve is latency-bound, so it runs beside the TTM kernels
  void* dev_scratch = nullptr;       // LeafScratch of the tp_dev_* entry points
  // asynchronous leaf solves of the grid executor (tp_dev_leaf_solve_begin / _finish): one lane per side stream
  struct Lane {
    void* scratch = nullptr;         // LeafScratch
    cudaEvent_t ready = nullptr, done = nullptr;
    bool busy = false, fast = false;
    bool keep = false;               // TP_LEAF_CONTINUE: an accepted solve leaves its Ritz vectors as the next start
    bool accepted = false;           // the lane's last solve was accepted with its certificate
    double* gram = nullptr;
    size_t rows = 0;
    int k = 0;
  };
  Lane lanes[4];
  // by-value hooi_sweep calls in a loop (the reference CLI's pattern) keep their device tensor and plan between
  // calls as long as shape, ranks, tree and schedule repeat; only the tensor and factor bytes move again
  std::vector<long long> host_call_key;
  tp_plan* host_call_plan = nullptr;
  tp_tensor* host_call_tensor = nullptr;
  static constexpr int kAux = 4;
  cudaStream_t aux[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cusolverDnHandle_t aux_solver[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cublasHandle_t blas = nullptr;     // small dense products inside the eigen-solve (off the hot path)
  cublasHandle_t aux_blas[kAux] = {nullptr, nullptr, nullptr, nullptr};
  // by-value calls upload the tensor in slabs on their own stream so that the root products can start on the
  // slabs that have arrived (tp_hooi_sweep_host)
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> arrival_events;
  // fixed cuBLAS workspaces (one per handle): recorded CUDA graphs must not depend on cuBLAS' own pool
  static constexpr size_t kBlasWorkspaceBytes = 32u << 20;
  void* blas_ws[kAux + 1] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // tp_ctx_set_option
  size_t streamed_upload_min_bytes = size_t{256} << 20;  // by-value calls: below this the upload is one copy
  bool trace_evd = false;                                // print every leaf's certificate margins to stderr
  bool dump_sweep_graph = false;                         // write a recorded sweep's graph to /tmp/tpb_sweep_graph.dot
  // by-value calls with TP_HOST_TENSOR_UNCHANGED: what the cached device tensor was uploaded from, and the factors the
  // last call returned (a caller that feeds them back continues the resident run: warm solves, carried products)
  bool host_call_busy = false;                           // a by-value call is using the cache right now
  const double* host_call_source = nullptr;
  std::vector<std::vector<double>> host_call_last_factors;
};

struct tp_tensor {
  std::vector<size_t> dims;
  size_t size = 0;
  double* data = nullptr;
  // changes whenever the contents may have changed (creation, tp_tensor_axpby, a by-value re-upload, handing out
  // the raw pointer); plans compare it before reusing products of this tensor kept from the previous sweep
  tp_u64 stamp = 0;
  // the raw device pointer has been handed out: writes through it are invisible to the stamp, so plans stop carrying
  // products of this tensor until tp_tensor_mark_modified re-establishes the contract
  bool pointer_escaped = false;
};

static tp_u64 next_tensor_stamp() {
  static std::atomic<tp_u64> counter{0};  // contexts on different host threads create tensors concurrently
  return counter.fetch_add(1, std::memory_order_relaxed) + 1;
}

static void release_host_call_cache(tp_ctx* ctx);

// Plans created from now on visit the carried subtree first: 0 never, 1 always, 2 (default) in short sweeps.
static std::atomic<int>& carry_first_mode() {
  static std::atomic<int> mode{2};
  return mode;
}

namespace tpb {
namespace {

thread_local tp_ctx* bound_ctx = nullptr;  // the context of the entry point running on this thread

void bind(const tp_ctx* ctx) {
  if (!ctx) raise(TP_ERR_BAD_ARGUMENT, "null context");
  TPB_CUDA(cudaSetDevice(ctx->device));
  bound_ctx = const_cast<tp_ctx*>(ctx);
}

// Device allocation.  When the device is out of memory the by-value call cache of the bound context (a whole device
// copy of the last tensor plus its plan's buffers, kept so that loops of by-value calls do not reallocate) is given
// up and the allocation retried once: the reference's usual sequence hooi_sweep -> reconstruction_error -> ttm, each
// uploading its own copy, must fit whenever each call fits on its own.
double* device_alloc(size_t doubles) {
  double* p = nullptr;
  const size_t bytes = std::max<size_t>(doubles, 1) * sizeof(double);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation && bound_ctx && (bound_ctx->host_call_plan || bound_ctx->host_call_tensor) &&
      !bound_ctx->host_call_busy) {
    cudaGetLastError();
    release_host_call_cache(bound_ctx);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(TP_ERR_CUDA, std::string("cudaMalloc of ") + std::to_string(doubles * 8) + " bytes: " + cudaGetErrorString(e));
  }
  return p;
}

size_t checked_size(int n_modes, const size_t* dims) {
  if (n_modes <= 0 || n_modes > kMaxModes || !dims) raise(TP_ERR_BAD_DIMS, "tensor needs 1..16 modes");
  u64 total = 1;
  for (int m = 0; m < n_modes; ++m) {
    if (dims[m] == 0) raise(TP_ERR_BAD_DIMS, "zero extent", m);  // zeros(), dense_tensor.hpp:35-36
    total = mul_or_throw(total, dims[m]);
  }
  return static_cast<size_t>(total);
}

tp_tensor* new_tensor(const std::vector<size_t>& dims) {
  tp_tensor* t = new tp_tensor;
  t->dims = dims;
  t->size = checked_size(static_cast<int>(dims.size()), dims.data());
  t->stamp = next_tensor_stamp();
  try {
    t->data = device_alloc(t->size);
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

void mode_extents(const std::vector<size_t>& dims, int mode, long long& outer, long long& inner) {
  if (mode < 0 || mode >= static_cast<int>(dims.size())) raise(TP_ERR_BAD_MODE, "mode out of range", mode);
  outer = inner = 1;
  for (int m = 0; m < mode; ++m) outer *= static_cast<long long>(dims[m]);
  for (int m = mode + 1; m < static_cast<int>(dims.size()); ++m) inner *= static_cast<long long>(dims[m]);
}

double* ensure_frag_scratch(tp_ctx* ctx, size_t doubles) {
  if (doubles > ctx->frag_capacity) {
    if (ctx->frag_scratch) {
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
      TPB_CUDA(cudaFree(ctx->frag_scratch));
      ctx->frag_scratch = nullptr;
      ctx->frag_capacity = 0;
    }
    ctx->frag_scratch = device_alloc(doubles);
    ctx->frag_capacity = doubles;
  }
  return ctx->frag_scratch;
}

// One TTM with an arbitrary-stride device matrix (prep + contraction), out preallocated.
void run_ttm(tp_ctx* ctx, const double* x, const std::vector<size_t>& dims, int mode, const double* m_dev,
             long long row_stride, long long col_stride, long long new_len, double* frag, double* out) {
  long long outer, inner;
  mode_extents(dims, mode, outer, inner);
  const long long len = static_cast<long long>(dims[mode]);
  const TtmFragmentLayout f = ttm_fragment_layout(new_len, len);
  if (!frag) frag = ensure_frag_scratch(ctx, f.doubles);
  TPB_CUDA(prep_factor_fragments(ctx->stream, m_dev, row_stride, col_stride, new_len, len, f, frag));
  TPB_CUDA(launch_ttm(ctx->stream, x, outer, len, inner, frag, f, new_len, out, ctx->sm_count));
  ctx->own_kernels += 2;
}

double device_scalar(tp_ctx* ctx, const double* dev) {
  double v = 0.0;
  TPB_CUDA(cudaMemcpyAsync(&v, dev, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}

double sum_squares(tp_ctx* ctx, const double* x, size_t n) {
  double* result = ctx->reduce_scratch + reduce_scratch_doubles();
  TPB_CUDA(launch_sum_squares(ctx->stream, x, n, ctx->reduce_scratch, result));
  ctx->own_kernels += 2;
  return device_scalar(ctx, result);
}

double diff_sum_squares(tp_ctx* ctx, const double* x, const double* y, size_t n) {
  double* result = ctx->reduce_scratch + reduce_scratch_doubles();
  TPB_CUDA(launch_diff_sum_squares(ctx->stream, x, y, n, ctx->reduce_scratch, result));
  ctx->own_kernels += 2;
  return device_scalar(ctx, result);
}

// Eigen-solve scratch shared by every leaf update of a plan / one-off call.
struct LeafScratch {
  long long max_rows = 0;
  double* gram = nullptr;      // rows x rows, overwritten with eigenvectors
  double* gram_ws = nullptr;   // split-k partials
  size_t gram_ws_doubles = 0;
  double* w = nullptr;         // eigenvalues
  double* work = nullptr;
  int lwork = 0;
  int* info = nullptr;
  int* flag = nullptr;         // degenerate flag, OR-ed by leaves
  // warm-started subspace iteration (top-k only): block basis / products, small Rayleigh-Ritz problem
  int block = 0;               // columns of the iteration block (k + oversampling), 0 = fast path not set up
  double* q = nullptr;         // rows x block
  double* z = nullptr;         // rows x block
  double* x = nullptr;         // rows x block (Ritz vectors, ascending)
  double* h = nullptr;         // block x block
  double* theta = nullptr;     // block
  double* chol = nullptr;      // block x block Cholesky factor
  double* ritz = nullptr;      // block x block Ritz rotation
  double* small_work = nullptr;
  int small_lwork = 0;
  int* verdict = nullptr;      // [0] |= 1: a kept Ritz pair missed the residual bound, |= 4: the gap / angle criterion
                               // failed; [1]: a factorisation failed (1 Cholesky pivot, 2 Jacobi not converged,
                               // else cuSOLVER info); [2]: Jacobi sweeps used; [3]: power steps (one-launch solve)
  double* diag = nullptr;      // certificate margins: worst kept residual / bound, angle bound, tau / theta_k, rounds
  bool use_graph = true;       // replay the multi-launch iteration as a CUDA graph from its third run on
  bool use_fused = true;       // small leaves: the whole solve in one launch (leaf_solve_kernels.cu)
  // the iteration is a fixed kernel sequence on fixed buffers: recorded once, replayed as a CUDA graph afterwards
  cudaGraphExec_t graph = nullptr;
  const double* graph_gram = nullptr;
  long long graph_rows = 0;
  int graph_k = 0;
  const double* graph_result = nullptr;  // where the recorded sequence leaves the Ritz vectors
  // all `block` Ritz vectors of the previous accepted solve on the same (gram, rows, k): the next start block.  With
  // them the Rayleigh-Ritz matrix starts out nearly diagonal and the Jacobi solver needs few sweeps.
  const double* last_ritz = nullptr;
  int graph_state = 0;         // 0: not run yet (first run is eager), 1: eager run done, 2: graph ready, -1: disabled
  int graph_aux = -2;          // side stream (cuBLAS handle and workspace with it) the graph belongs to: a replay
                               // anywhere else could share that workspace with another leaf's concurrent solve
  long long fast_rows = 0;     // rows the iteration buffers were sized for (tp_dev_leaf_solve_warm only)
  int failures = 0;            // consecutive warm sweeps in which the fast path was rejected
  // Launch-sequence solves (leaves too large for the one-launch kernel): power steps of the next solve.  A cold solve
  // takes kSubspacePowerSteps; each certified warm solve that beat the residual bound by two orders of magnitude
  // gives two steps back, a rejected one restores the count and raises the floor (so the count settles).
  int power_steps = 0, power_steps_floor = 1;
  int graph_steps = 0;         // step count the leaf's recorded graph was built with
  bool launch_sequence = false;  // the last solve ran as a launch sequence (not the one-launch kernel)
  bool refinable = false;      // last rejection was a missed residual bound only (no failed factorisation / gap)
  bool was_cold = false;       // this sweep's solve started from the caller's factors
  bool cold_rejected = false;  // a cold start missed its certificate before: later cold starts take the full solve
  bool fast_used = false;      // this sweep's factor came from the fast path (verdict still to be checked)

  void release() {
    if (graph) cudaGraphExecDestroy(graph);
    cudaFree(chol);
    cudaFree(ritz);
    cudaFree(q);
    cudaFree(z);
    cudaFree(x);
    cudaFree(h);
    cudaFree(theta);
    cudaFree(small_work);
    cudaFree(verdict);
    cudaFree(diag);
    cudaFree(gram);
    cudaFree(gram_ws);
    cudaFree(w);
    cudaFree(work);
    cudaFree(info);
    cudaFree(flag);
    *this = LeafScratch{};
  }
};

// The iteration buffers are about to change: the recorded graph and the kept Ritz vectors point into them.
void forget_recorded_solve(LeafScratch& s) {
  if (s.graph) cudaGraphExecDestroy(s.graph);
  s.graph = nullptr;
  if (s.graph_state > 0) s.graph_state = 0;
  s.graph_gram = nullptr;
  s.last_ritz = nullptr;
}

void leaf_scratch_reserve(tp_ctx* ctx, LeafScratch& s, long long rows, size_t gram_ws_doubles) {
  if (rows > s.max_rows) {
    cudaFree(s.gram);
    cudaFree(s.w);
    cudaFree(s.work);
    s.gram = device_alloc(static_cast<size_t>(rows) * rows);
    s.w = device_alloc(static_cast<size_t>(rows));
    int lwork = 0;
    TPB_SOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                           static_cast<int>(rows), s.gram, static_cast<int>(rows), s.w, &lwork));
    s.work = device_alloc(static_cast<size_t>(lwork));
    s.lwork = lwork;
    s.max_rows = rows;
  }
  if (gram_ws_doubles > s.gram_ws_doubles) {
    cudaFree(s.gram_ws);
    s.gram_ws = device_alloc(gram_ws_doubles);
    s.gram_ws_doubles = gram_ws_doubles;
  }
  if (!s.info) {
    TPB_CUDA(cudaMalloc(&s.info, sizeof(int)));
    TPB_CUDA(cudaMalloc(&s.flag, sizeof(int)));
    // synchronous: the first writers may sit on a side stream that is not ordered after ctx->stream
    TPB_CUDA(cudaMemset(s.flag, 0, sizeof(int)));
    TPB_CUDA(cudaMemset(s.info, 0, sizeof(int)));
  }
}

void check_leaf_args(long long rows, long long cols, int k) {  // hooi.hpp:46-51
  if (rows == 0 || cols == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
  if (rows > TP_MAX_GRAM_ROWS) raise(TP_ERR_TOO_LARGE, "unfolding has too many rows for the Gram route");
  if (k < 1 || k > rows) raise(TP_ERR_BAD_ARGUMENT, "need 1 <= k <= rows");
}

// Gram of the mode-`mode` unfolding of y into s.gram (hooi.hpp:53-54 without the unfold copy of :148-149).
// `spare_sms`: SMs a persistent (wide) Gram grid leaves to eigen-solve kernels in flight on the side streams.
long long leaf_gram(tp_ctx* ctx, LeafScratch& s, const double* y, const std::vector<size_t>& dims, int mode, int k,
                    int spare_sms = 0) {
  long long outer, inner;
  mode_extents(dims, mode, outer, inner);
  const long long rows = static_cast<long long>(dims[mode]);
  check_leaf_args(rows, outer * inner, k);
  const GramLayout g = gram_layout(outer, rows, inner, std::max(1, ctx->sm_count - spare_sms));
  leaf_scratch_reserve(ctx, s, rows, g.workspace_doubles);
  TPB_CUDA(launch_gram(ctx->stream, y, outer, rows, inner, g, s.gram_ws, s.gram));
  ctx->own_kernels += 2;
  return rows;
}

// Top-k eigenvectors of s.gram into factor_out (rows x k column-major): full symmetric eigen-solve (hooi.hpp:55),
// then the sign / gap rules (hooi.hpp:60-74).  The eigen-solve is cuSOLVER's (off the hot path per the spec).
void leaf_solve(tp_ctx* ctx, LeafScratch& s, long long rows, int k, double* factor_out, int aux = -1) {
  cusolverDnHandle_t solver = aux < 0 ? ctx->solver : ctx->aux_solver[aux];
  cudaStream_t stream = aux < 0 ? ctx->stream : ctx->aux[aux];
  TPB_SOLVER(cusolverDnDsyevd(solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(rows),
                              s.gram, static_cast<int>(rows), s.w, s.work, s.lwork, s.info));
  ctx->library_calls += 1;
  TPB_CUDA(launch_select_basis(stream, s.gram, s.w, static_cast<int>(rows), static_cast<int>(rows), k, factor_out,
                               s.flag));
  ctx->own_kernels += 1;
}

// ---- top-k eigen-solve by warm-started block subspace iteration --------------------------------------------
// The leaves only need the K_n leading eigenvectors of an L_n x L_n Gram matrix whose spectrum, for the tensors
// HOOI is run on, drops sharply after K_n, and the previous factor is an excellent start.  Orthogonal iteration
// on a block of K_n + p columns (p = oversampling) converges like (lambda_{K+p+1} / lambda_K)^steps.  The schedule
// is fixed (no host decisions inside the sweep): kSubspacePowerSteps x [Z = G Q; Q = CholQR(Z)] -- one Cholesky-QR
// pass keeps the block well conditioned, which is all the iteration needs since only span(Q) matters; the last
// step repeats the pass so that Q is orthonormal to rounding -- then one Rayleigh-Ritz step.  A device flag records
// whether every kept Ritz pair satisfies ||G x - theta x|| <= 1e-13 theta_max and whether the gap estimate is
// safe.  The sweep checks the flags once at its end; a rejected leaf is redone with the full eigen-solve (the Gram
// matrix is left intact here), so the result is always the reference's: eigenvectors of the Gram matrix to
// rounding (hooi.hpp:55-69).
constexpr int kSubspaceOversample = 8;
constexpr int kSubspacePowerSteps = 6;
constexpr double kSubspaceTol = 1e-13;
// Davis-Kahan bound on the sine of the angle between the kept Ritz space and the leading invariant subspace that the
// certificate accepts: a decade inside the 1e-9 projector tolerance of the reference's own tests (tolerances.hpp:17).
// Leaves whose spectral gap is too small for it go to the full eigen-solve.
constexpr double kSubspaceAngleTol = 1e-10;

// `cols`: columns of the unfolding whose Gram matrix is solved (its rank bound); the iteration block must not exceed
// it or Z = G Q is rank deficient and the Cholesky-QR breaks down.
bool subspace_eligible(long long rows, int k, double cols = 1e300) {
  const long long b = k + kSubspaceOversample;
  if (2 * b > rows || static_cast<double>(b) > cols) return false;
  // with the single-launch small steps (evd_kernels.cu) and graph replay the iteration wins at every size; wider
  // blocks go through cuSOLVER's potrf / syevd, ~70 launches, which only pays against a large full eigen-solve
  return static_cast<size_t>(b) <= small_evd_max_block() || rows >= 704;
}

void subspace_reserve(tp_ctx* ctx, LeafScratch& s, long long rows, int k) {
  const int b = k + kSubspaceOversample;
  if (s.block == b) return;
  const size_t nb = static_cast<size_t>(rows) * b;
  s.q = device_alloc(nb);
  s.z = device_alloc(nb);
  s.x = device_alloc(nb);
  s.h = device_alloc(static_cast<size_t>(b) * b);
  s.theta = device_alloc(static_cast<size_t>(b));
  s.chol = device_alloc(static_cast<size_t>(b) * b);
  s.ritz = device_alloc(static_cast<size_t>(b) * b);
  int l1 = 0, l2 = 0;
  TPB_SOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, b, s.h, b,
                                         s.theta, &l1));
  TPB_SOLVER(cusolverDnDpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, b, s.h, b, &l2));
  s.small_lwork = std::max(l1, l2);
  s.small_work = device_alloc(static_cast<size_t>(s.small_lwork));
  TPB_CUDA(cudaMalloc(&s.verdict, 4 * sizeof(int)));
  TPB_CUDA(cudaMemset(s.verdict, 0, 4 * sizeof(int)));
  s.diag = device_alloc(16);
  TPB_CUDA(cudaMemset(s.diag, 0, 16 * sizeof(double)));
  s.block = b;
}

struct SubspaceIo {
  cublasHandle_t blas;
  cusolverDnHandle_t solver;
  cudaStream_t stream;
  bool own_small;  // block fits the single-CTA kernels of evd_kernels.cu (else cuSOLVER potrf / syevd)
};

// Z (rows x b, column-major) <- Z L^{-T} with L L^T = Z^T Z, `passes` times (2 = orthonormal to rounding).
void cholqr(tp_ctx* ctx, const SubspaceIo& io, LeafScratch& s, int rows, int b, double* zbuf, int passes) {
  const double one = 1.0, zero = 0.0;
  for (int pass = 0; pass < passes; ++pass) {
    TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_T, CUBLAS_OP_N, b, b, rows, &one, zbuf, rows, zbuf, rows, &zero, s.h, b));
    if (io.own_small) {
      TPB_CUDA(launch_cholesky(io.stream, s.h, b, s.chol, s.verdict + 1));
      TPB_CUDA(launch_trsm_right_lt(io.stream, zbuf, rows, b, s.chol));
      ctx->own_kernels += 2;
      ctx->library_calls += 1;
    } else {
      TPB_SOLVER(cusolverDnDpotrf(io.solver, CUBLAS_FILL_MODE_LOWER, b, s.h, b, s.small_work, s.small_lwork,
                                  s.verdict + 1));
      TPB_BLAS(cublasDtrsm(io.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, rows,
                           b, &one, s.h, b, zbuf, rows));
      ctx->library_calls += 3;
    }
  }
}

// The iteration proper: from the start block in s.q (filled by the caller; it needs no orthonormalisation of its
// own, only its span matters) to Ritz vectors
// (ascending) and values in the returned buffer / s.theta, and the certificate in s.verdict.  Touches only device
// memory owned by `s` plus `gram` (read), with no host decision inside -- it is what the CUDA graph records.
const double* subspace_body(tp_ctx* ctx, const SubspaceIo& io, LeafScratch& s, const double* gram, int rows, int k,
                            int power_steps = kSubspacePowerSteps) {
  const int b = s.block;
  const double one = 1.0, zero = 0.0;
  double *q = s.q, *z = s.z, *x = s.x;
  TPB_CUDA(cudaMemsetAsync(s.verdict, 0, 4 * sizeof(int), io.stream));
  for (int step = 0; step < power_steps; ++step) {
    TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, b, rows, &one, gram, rows, q, rows, &zero, z, rows));
    std::swap(q, z);
    cholqr(ctx, io, s, rows, b, q, step + 1 == power_steps ? 2 : 1);
  }
  // Rayleigh-Ritz on span(Q): H = Q^T G Q, H = V Theta V^T (ascending), X = Q V
  TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, b, rows, &one, gram, rows, q, rows, &zero, z, rows));
  TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_T, CUBLAS_OP_N, b, b, rows, &one, q, rows, z, rows, &zero, s.h, b));
  const double* v = s.h;
  if (io.own_small) {
    TPB_CUDA(launch_jacobi_eig(io.stream, s.h, b, s.theta, s.ritz, s.verdict + 1));
    ctx->own_kernels += 1;
    v = s.ritz;
  } else {
    TPB_SOLVER(cusolverDnDsyevd(io.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, b, s.h, b, s.theta,
                                s.small_work, s.small_lwork, s.verdict + 1));
    ctx->library_calls += 1;
  }
  TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, b, b, &one, q, rows, v, b, &zero, x, rows));
  // residuals of the kept pairs: (Z V)_j - theta_j X_j with Z = G Q
  TPB_BLAS(cublasDgemm(io.blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, b, b, &one, z, rows, v, b, &zero, q, rows));
  TPB_CUDA(launch_ritz_certificate(io.stream, gram, q, x, s.theta, rows, b, k, kSubspaceTol, kSubspaceAngleTol,
                                   s.verdict, s.diag));
  ctx->own_kernels += 1;
  ctx->library_calls += power_steps + 4;
  return x;
}

// Enqueues the whole fast solve on the leaf's stream; the verdict is read by the caller at the end of the sweep.
// `recording`: the caller is recording the whole sweep into a CUDA graph; the iteration's launches then go straight
// into that recording instead of through the leaf's own graph.
void leaf_solve_subspace(tp_ctx* ctx, LeafScratch& s, const double* gram, long long rows_ll, int k,
                         const double* start, double* factor_out, int aux, bool recording = false) {
  SubspaceIo io;
  io.solver = aux < 0 ? ctx->solver : ctx->aux_solver[aux];
  io.blas = aux < 0 ? ctx->blas : ctx->aux_blas[aux];
  io.stream = aux < 0 ? ctx->stream : ctx->aux[aux];
  io.own_small = static_cast<size_t>(s.block) <= small_evd_max_block();
  const int rows = static_cast<int>(rows_ll), b = s.block;
  if (s.use_fused && leaf_solve_fused_eligible(rows_ll, k, b)) {
    // small leaf: start block, power steps, Rayleigh-Ritz, certificate (rounds repeat on the device until it holds)
    // and the reference's selection in ONE launch.  Warm: from all Ritz vectors of the previous solve, one power step
    // in the first round; cold: from the caller's factor + filler columns, three.
    const bool warm = s.last_ritz != nullptr;
    TPB_CUDA(launch_leaf_solve_fused(io.stream, gram, rows, k, b, warm ? s.last_ritz : start, warm ? 0 : 1,
                                     warm ? 1 : 3, 4, kSubspaceTol, kSubspaceAngleTol, s.x, s.theta, factor_out,
                                     s.flag, s.verdict, s.diag));
    ctx->own_kernels += 1;
    s.fast_used = true;
    s.last_ritz = s.x;
    s.launch_sequence = false;
    return;
  }
  const bool graphs_off = !s.use_graph || recording;
  // a cold start (the caller's factors plus filler columns) always takes the full count
  if (s.power_steps < 1 || !s.last_ritz) s.power_steps = kSubspacePowerSteps;
  const int steps = s.power_steps;
  s.launch_sequence = true;
  const bool key_ok = s.graph_gram == gram && s.graph_rows == rows_ll && s.graph_k == k && s.graph_steps == steps;
  if (!key_ok && !recording) {  // the slot is being reused for another problem, or the step count moved: start over
    if (s.graph) cudaGraphExecDestroy(s.graph);
    s.graph = nullptr;
    if (s.graph_state > 0) s.graph_state = 0;
    if (s.graph_gram != gram || s.graph_rows != rows_ll || s.graph_k != k) s.last_ritz = nullptr;
  }
  if (s.last_ritz) {
    // start block: the previous solve's Ritz vectors, dominant first (Cholesky QR orthogonalises in column order)
    TPB_CUDA(launch_reverse_columns(io.stream, s.q, s.last_ritz, rows, b));
    ctx->own_kernels += 1;
  } else {
    // start block: previous factor + deterministic filler for the oversampling columns
    TPB_CUDA(cudaMemcpyAsync(s.q, start, sizeof(double) * rows * k, cudaMemcpyDeviceToDevice, io.stream));
    TPB_CUDA(launch_fill_pseudo_random(io.stream, s.q + static_cast<size_t>(rows) * k,
                                       static_cast<size_t>(rows) * (b - k), 0x7461636bull));
    ctx->own_kernels += 1;
  }
  const double* ritz_vectors = nullptr;
  if (io.own_small && !graphs_off && s.graph_state == 1 && aux == s.graph_aux) {
    // second run on the same buffers: record the sequence.  Lazy initialisation (kernel attributes, cuBLAS
    // heuristics) happened during the eager first run.
    const unsigned long long own0 = ctx->own_kernels, lib0 = ctx->library_calls;
    cudaGraph_t recorded = nullptr;
    bool ok = cudaStreamBeginCapture(io.stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      try {
        ritz_vectors = subspace_body(ctx, io, s, gram, rows, k, steps);
      } catch (const Failure&) {
        ok = false;
      }
      if (cudaStreamEndCapture(io.stream, &recorded) != cudaSuccess) ok = false;
      if (ok && cudaGraphInstantiate(&s.graph, recorded, 0) != cudaSuccess) ok = false;
      if (recorded) cudaGraphDestroy(recorded);
    }
    if (ok) {
      s.graph_state = 2;
      s.graph_result = ritz_vectors;
    } else {
      cudaGetLastError();  // recording is an optimisation: fall back to plain launches for this slot
      s.graph = nullptr;
      s.graph_state = -1;
    }
    ctx->own_kernels = own0;
    ctx->library_calls = lib0;
  }
  if (s.graph_state == 2 && !recording && aux == s.graph_aux) {
    ritz_vectors = s.graph_result;
    TPB_CUDA(cudaGraphLaunch(s.graph, io.stream));
    // same work as the eager body, for the launch accounting
    ctx->own_kernels += 2 * (steps + 1) + 2;
    ctx->library_calls += (steps + 1) + steps + 4;
  } else {
    ritz_vectors = subspace_body(ctx, io, s, gram, rows, k, steps);
    if (io.own_small && !graphs_off && s.graph_state == 0) {
      s.graph_state = 1;
      s.graph_aux = aux;
    }
  }
  if (!recording) {  // what the buffers (and a recorded graph) now belong to
    s.graph_steps = steps;
    s.graph_gram = gram;
    s.graph_rows = rows_ll;
    s.graph_k = k;
  }
  TPB_CUDA(launch_select_basis(io.stream, ritz_vectors, s.theta, rows, b, k, factor_out, s.flag));
  ctx->own_kernels += 1;
  s.fast_used = true;
  s.last_ritz = ritz_vectors;  // dropped again by whoever finds the certificate violated
}

void leaf_update(tp_ctx* ctx, LeafScratch& s, const double* y, const std::vector<size_t>& dims, int mode, int k,
                 double* factor_out) {
  const long long rows = leaf_gram(ctx, s, y, dims, mode, k);
  leaf_solve(ctx, s, rows, k, factor_out);
}

int read_and_clear_flag(tp_ctx* ctx, LeafScratch& s) {
  int host[2] = {0, 0};
  TPB_CUDA(cudaMemcpyAsync(&host[0], s.flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TPB_CUDA(cudaMemcpyAsync(&host[1], s.info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TPB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), ctx->stream));
  TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (host[1] != 0) raise(TP_ERR_TOO_LARGE, "eigensolver did not converge");  // hooi.hpp:56-57
  return host[0];
}

// Reads the certificates of the leaves that took the fast path this sweep; returns the modes to redo.
std::vector<int> verify_fast_leaves(tp_ctx* ctx, tp_plan* p);

int read_and_clear_flags(tp_ctx* ctx, std::vector<LeafScratch>& slots) {
  std::vector<int> host(2 * slots.size(), 0);
  for (size_t i = 0; i < slots.size(); ++i) {
    if (!slots[i].flag) continue;
    TPB_CUDA(cudaMemcpyAsync(&host[2 * i], slots[i].flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaMemcpyAsync(&host[2 * i + 1], slots[i].info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaMemsetAsync(slots[i].flag, 0, sizeof(int), ctx->stream));
  }
  TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  int flag = 0;
  for (size_t i = 0; i < slots.size(); ++i) {
    if (host[2 * i + 1] != 0) raise(TP_ERR_TOO_LARGE, "eigensolver did not converge");  // hooi.hpp:56-57
    flag |= host[2 * i];
  }
  return flag;
}

}  // namespace
}  // namespace tpb

// ------------------------------------------------------------------------ plan
struct tp_plan {
  Spec spec;
  Tree tree;
  int sweep_kind = TP_SWEEP_JACOBI;
  int n = 0;
  std::vector<std::vector<int>> gs_paths;
  std::vector<double*> cur, fresh;            // device factors, L_n x K_n column-major
  std::vector<TtmFragmentLayout> frag_layout; // for F_n^T (K_n x L_n) as the TTM matrix
  std::vector<double*> frag;                  // fragment-ordered copies, rebuilt when a factor changes
  std::vector<double*> depth_buf;             // one intermediate per tree depth
  std::vector<size_t> depth_cap;
  // Forked walk (TP_OPT_FORK_SUBTREES; auto = short sweeps).  The subtrees below a node are independent: every child
  // but the last visited runs on a stream of its own, so the short, latency-bound products and Gram kernels of small
  // tensors overlap instead of queueing behind one another.  Siblings then need an output buffer each.
  int fork_mode = 2;                          // 0 off, 1 on, 2 auto
  bool forking = false;                       // this sweep's walk forks
  std::vector<size_t> node_cap;               // per node: elements of its product (0 for leaves)
  std::vector<double*> node_buf;              // allocated on first use
  std::vector<cudaStream_t> branch;           // branch streams, created on first use
  std::vector<cudaEvent_t> fork_events;
  size_t branches_used = 0, fork_events_used = 0;
  std::vector<cudaEvent_t> branch_done;       // recorded at the end of every branch of this sweep: the join list
  double* core = nullptr;
  double* core_tmp[2] = {nullptr, nullptr};
  size_t core_size = 0, core_tmp_cap = 0;
  std::vector<int> core_order;                // cheapest contraction order of the core chain
  tp_u64 core_macs_executed = 0;
  std::vector<LeafScratch> leaf;              // one Gram / eigen-solve scratch per mode (leaves run concurrently)
  std::vector<cudaEvent_t> gram_ready, factor_ready;
  bool overlap_evd = true;                    // Jacobi: eigen-solves on side streams beside the tree TTMs
  bool fast_evd = true;                       // top-k subspace iteration where eligible, verified, full solve otherwise
  bool leaf_steps_changed = false;            // a leaf's power-step count moved: the recorded sweep is stale
  int fast_rejected = 0;
  std::vector<std::vector<int>> visit_order;  // per node: children in execution order (see plan_visit_order)
  std::vector<int> leaf_rank;                 // per mode: position of its leaf in the execution order
  // Carried path (Jacobi): the core chain T x F_new... may contract the modes in any order; run along a root-to-leaf
  // path of the TTM tree it produces, with the new factors, exactly the intermediates the NEXT sweep's walk needs at
  // those nodes.  They are kept (own buffers) and the next walk starts from them, so per sweep every tree node is
  // computed once and the core costs one small extra product instead of a second pass over the tensor.
  // Streamed first pass (by-value calls): the tensor is still arriving from the host in slabs of its first mode.
  // issue(c) queues the upload of slab c (idempotent), ready[c] fires when it is on the device.
  struct Arrival {
    std::vector<size_t> row_end;               // slab c = rows [row_end[c-1], row_end[c]) of mode 0
    std::vector<cudaEvent_t> ready;
    std::function<void(int)> issue;
  };
  Arrival* arrival = nullptr;                  // set for the duration of one sweep
  std::vector<double*> arrival_slots;          // per-slab partial products of the root node that contracts mode 0
  size_t arrival_slot_doubles = 0;
  std::vector<double*> arrival_frag;           // fragment-ordered row slices of F_0, one per slab
  std::vector<size_t> arrival_frag_doubles;
  bool factors_from_caller = true;            // no sweep has run since the factors were set
  bool frags_match_cur = false;               // frag[m] holds the fragments of cur[m] for every mode (the core chain of
                                              // a Jacobi sweep prepares them from the new factors it then copies to cur)
  bool carry_enabled = true;
  std::vector<int> carry_nodes;               // TTM nodes of the path, root child first (empty: no carrying)
  int carry_leaf_mode = -1;                   // mode of the leaf the path ends in = last product of the core chain
  std::vector<char> on_carry;                 // per node
  std::vector<double*> carry_buf;             // one per path node
  bool carry_valid = false;                   // carry_buf holds products of (carry_tensor @ carry_stamp, cur factors)
  const tp_tensor* carry_tensor = nullptr;
  tp_u64 carry_stamp = 0;
  bool carry_live = false;                    // this sweep's walk starts from the carried products
  int spare_sms_short = 16;                   // ... by products shorter than short_product_flops (tuning knobs;
                                              // measured on C5: 2 -> 58.2, 16 -> 57.6, 32 -> 58.1, 48 -> 58.4 ms/iter)
  double short_product_flops = 2e11;
  int spare_sms = 2;                          // SMs left to the side streams while eigen-solves are in flight
                                              // (measured on C5: 0-2 -> 58.4 ms/iter, 6 -> 58.9, 12 -> 60.0)
  int leaves_in_flight = 0;
  int one_launch_leaves = 0;                  // leaves whose solve is the single-CTA kernel (leaf_solve_kernels.cu)
  struct PendingLeaf {
    int mode, node;
  };
  std::vector<PendingLeaf> pending;           // leaves whose eigen-solve still has to be queued                      // leaves of the last sweep that had to be redone with the full solve
  // Whole-sweep CUDA graph (Jacobi).  Once a run is in its steady state -- factors produced by the previous sweep,
  // carried products valid, every leaf on a capturable fast path -- a sweep is a fixed launch sequence on fixed buffers
  // (tree products, Gram kernels, the leaf solves forked onto the side streams, the core chain, the status read-back):
  // it is captured once and replayed, so the short sweeps of small tensors are not paced by ~100 host launches.
  int sweep_graph_mode = 2;                   // 0 off, 1 on, 2 auto: only sweeps whose tree is short (see short_sweep)
  bool short_sweep = false;                   // tree + core flops small enough for launch latency to matter
  bool carry_first = false;                   // visit the carried subtree first (short sweeps), else last
  cudaGraphExec_t sweep_graph = nullptr;
  const double* sweep_graph_tensor = nullptr;
  tp_u64 sweep_graph_stamp = 0;
  std::vector<char> sweep_graph_fast;         // per mode: the leaf's solve inside the graph is a certified fast solve
  bool last_sweep_replayed = false;
  bool capturing = false;                     // the launch sequence is being recorded, not run: no timing events
  u64 sweep_graph_kernels = 0, sweep_graph_library_calls = 0;  // launches of one steady-state sweep (accounting)
  int warm_sweeps = 0;                        // sweeps since the caller last set the factors
  cudaEvent_t graph_begin = nullptr, graph_end = nullptr;
  // pinned read-back of every leaf's status, 8 ints per mode: verdict[0..3], degenerate flag, solver info, 2 unused;
  // and of the certificate margins, 4 doubles per mode
  int* host_status = nullptr;    // one pinned block: 8 n ints, then (host_diag) 4 n doubles
  double* host_diag = nullptr;
  void* dev_status = nullptr;    // the same layout on the device, written by finish_sweep_kernel
  tp_sweep_stats model{};   // analytic SweepStats (tree_macs, core_macs, peak_live)
  tp_sweep_timing timing{};
  // event pool for phase timing: triples (phase, begin, end)
  std::vector<cudaEvent_t> events;
  std::vector<int> event_phase;
  std::vector<int> event_node;   // tree node a span belongs to, -1 if none
  size_t events_used = 0;
  std::vector<float> node_ms, node_evd_ms;
};

namespace tpb {
namespace {

enum Phase { kTree = 0, kGram = 1, kEvd = 2, kCore = 3 };

cudaEvent_t next_event(tp_plan* p) {
  if (p->events_used == p->events.size()) {
    cudaEvent_t e;
    TPB_CUDA(cudaEventCreate(&e));
    p->events.push_back(e);
  }
  return p->events[p->events_used++];
}

struct Span {
  tp_plan* plan;
  cudaStream_t stream;
  cudaEvent_t end;
  // both events are reserved up front so that spans may nest (an eigen-solve queued inside the core span)
  Span(tp_ctx* c, tp_plan* p, int phase, int node = -1, int aux = -1)
      : plan(p), stream(aux < 0 ? c->stream : c->aux[aux]), end(nullptr) {
    if (plan->capturing) return;  // timing events do not belong in a recorded sweep
    plan->event_phase.push_back(phase);
    plan->event_node.push_back(node);
    cudaEvent_t begin = next_event(plan);
    end = next_event(plan);
    TPB_CUDA(cudaEventRecord(begin, stream));
  }
  void close() {
    if (end) TPB_CUDA(cudaEventRecord(end, stream));
  }
};

void plan_refresh_fragments(tp_ctx* ctx, tp_plan* p, int mode, const double* factor) {
  // F (L x K col-major) read as M = F^T: M(k, l) = F[k * L + l]
  const long long L = static_cast<long long>(p->spec.L[mode]), K = static_cast<long long>(p->spec.K[mode]);
  TPB_CUDA(prep_factor_fragments(ctx->stream, factor, L, 1, K, L, p->frag_layout[mode], p->frag[mode]));
  ctx->own_kernels += 1;
}

// `spare_sms`: SMs the persistent TTM grid leaves free so that eigen-solve kernels queued on the side streams can
// run beside it (the TTM CTAs are register-heavy and would otherwise hold every SM until the kernel ends).
void plan_ttm(tp_ctx* ctx, tp_plan* p, const double* x, const std::vector<size_t>& dims, int mode, double* out,
              int spare_sms = 0) {
  long long outer, inner;
  mode_extents(dims, mode, outer, inner);
  // a short product beside running eigen-solves gives them a real share of the machine (it costs little: the product
  // is short); a long one only leaves the few SMs their latency-bound kernels need
  if (spare_sms > 0) {
    const double flops = 2.0 * static_cast<double>(p->spec.K[mode]) * static_cast<double>(outer) *
                         static_cast<double>(dims[mode]) * static_cast<double>(inner);
    if (p->one_launch_leaves == p->n)
      spare_sms = std::max(spare_sms, p->n);  // every solve in flight is one CTA that needs a whole SM to itself
    else if (flops < p->short_product_flops)
      spare_sms = std::max(spare_sms, p->spare_sms_short);
  }
  TPB_CUDA(launch_ttm(ctx->stream, x, outer, static_cast<long long>(dims[mode]), inner, p->frag[mode],
                      p->frag_layout[mode], static_cast<long long>(p->spec.K[mode]), out,
                      std::max(1, ctx->sm_count - spare_sms)));
  ctx->own_kernels += 1;
}

// Columns of the unfolding a leaf's Gram matrix comes from: every other mode is already at its core extent.
double plan_leaf_columns(const tp_plan* p, int mode) {
  double cols = 1.0;
  for (int m = 0; m < p->n; ++m)
    if (m != mode) cols *= static_cast<double>(p->spec.K[m]);
  return cols;
}

// Leaf update.  The Gram kernels stay on the main stream (the intermediate they read lives in a per-depth buffer the
// next sibling TTM overwrites); with `overlap` the eigen-solve moves to a side stream and the main stream carries on
// with the tree, joining again before the core chain needs the new factors.
void plan_leaf_solve(tp_ctx* ctx, tp_plan* p, int mode, int node, double* dst, bool overlap) {
  const int k = static_cast<int>(p->spec.K[mode]);
  const long long rows = static_cast<long long>(p->spec.L[mode]);
  const int aux = overlap ? mode % tp_ctx::kAux : -1;
  if (overlap) TPB_CUDA(cudaStreamWaitEvent(ctx->aux[aux], p->gram_ready[mode], 0));
  Span evd(ctx, p, kEvd, node, aux);
  LeafScratch& slot = p->leaf[mode];
  slot.fast_used = false;
  // cold: the start factors are the caller's (plan creation / tp_plan_set_factors), not a previous sweep's result
  const bool cold = p->factors_from_caller;
  if (p->fast_evd && slot.failures < 2 && !(cold && slot.cold_rejected) &&
      subspace_eligible(rows, k, plan_leaf_columns(p, mode))) {
    subspace_reserve(ctx, slot, rows, k);
    slot.was_cold = cold;
    leaf_solve_subspace(ctx, slot, slot.gram, rows, k, p->cur[mode], dst, aux, p->capturing);
  } else {
    leaf_solve(ctx, slot, rows, k, dst, aux);
  }
  evd.close();
  if (overlap) TPB_CUDA(cudaEventRecord(p->factor_ready[mode], ctx->aux[aux]));
}

// Eigen-solves whose Gram matrix is queued but whose own (many, partly host-blocking) library calls are not yet:
// they are issued right after the NEXT product has been queued on the main stream, so the GPU is never left
// without work while the host walks through a solver's call sequence.
void plan_flush_pending(tp_ctx* ctx, tp_plan* p) {
  for (const tp_plan::PendingLeaf& job : p->pending) plan_leaf_solve(ctx, p, job.mode, job.node, p->fresh[job.mode], true);
  p->pending.clear();
}

void plan_leaf(tp_ctx* ctx, tp_plan* p, const double* y, const std::vector<size_t>& dims, int mode, double* dst,
               int node, bool overlap) {
  const int k = static_cast<int>(p->spec.K[mode]);
  Span gram(ctx, p, kGram, node);
  leaf_gram(ctx, p->leaf[mode], y, dims, mode, k,
            (overlap && p->leaves_in_flight > 0) ? gram_wide_spare_sms().load(std::memory_order_relaxed) : 0);
  gram.close();
  if (overlap) {
    TPB_CUDA(cudaEventRecord(p->gram_ready[mode], ctx->stream));
    p->pending.push_back(tp_plan::PendingLeaf{mode, node});
    ++p->leaves_in_flight;
  } else {
    plan_leaf_solve(ctx, p, mode, node, dst, false);
  }
}

// Status read-back of a sweep, on the main stream: the certificate of every leaf that took a fast path this sweep,
// every leaf's degenerate flag and solver info (the flags are cleared for the next sweep).  All copies land in the
// plan's pinned buffers, so the same sequence can be part of a recorded sweep.
void queue_status_readback(tp_ctx* ctx, tp_plan* p, bool with_flags) {
  for (int m = 0; m < p->n; ++m) {
    LeafScratch& s = p->leaf[m];
    int* const host = p->host_status + 8 * m;
    if (s.fast_used) {
      TPB_CUDA(cudaMemcpyAsync(host, s.verdict, 4 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaMemcpyAsync(p->host_diag + 4 * m, s.diag, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (!s.flag) continue;
    if (with_flags || s.fast_used)
      TPB_CUDA(cudaMemcpyAsync(host + 4, s.flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (with_flags) {
      TPB_CUDA(cudaMemcpyAsync(host + 5, s.info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), ctx->stream));
    }
  }
}

// After the stream has been synchronised: which of the fast leaves missed their certificate (-> to be redone).
std::vector<int> evaluate_fast_leaves(tp_ctx* ctx, tp_plan* p) {
  std::vector<int> rejected;
  for (int m = 0; m < p->n; ++m) {
    LeafScratch& s = p->leaf[m];
    if (!s.fast_used) continue;
    const int* const host = p->host_status + 8 * m;
    // residual bound / gap criterion missed, a factorisation inside failed, or the gap estimate says "degenerate"
    // (then the exact spectrum decides)
    const bool bad = host[0] != 0 || host[1] != 0 || host[4] != 0;
    if (ctx->trace_evd)
      std::fprintf(stderr,
                   "[tpb evd] mode %d block %d: miss=%d factorisation=%d jacobi_sweeps=%d power_steps=%d degenerate=%d "
                   "graph=%d residual/bound=%.3g angle_bound=%.3g tau/theta_k=%.3g rounds=%g\n",
                   m, s.block, host[0], host[1], host[2], host[3], host[4], s.graph_state, p->host_diag[4 * m],
                   p->host_diag[4 * m + 1], p->host_diag[4 * m + 2], p->host_diag[4 * m + 3]);
    if (bad) {
      rejected.push_back(m);
      // only the residual bound missed: the block is sound and simply has not converged yet -> worth iterating on
      // (not when the tail bound already exceeds theta_k -- a flat spectrum, e.g. a start from random factors -- no
      // amount of iterating certifies that)
      s.refinable = (host[0] & 1) != 0 && host[1] == 0 && host[4] == 0 && p->host_diag[4 * m + 2] < 0.5;
      if (!s.refinable) s.last_ritz = nullptr;
      if (s.launch_sequence && s.power_steps < kSubspacePowerSteps) {
        s.power_steps_floor = std::min(kSubspacePowerSteps, s.power_steps + 2);
        s.power_steps = kSubspacePowerSteps;
        p->leaf_steps_changed = true;
      }
      TPB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), ctx->stream));
    } else {
      s.failures = 0;
      if (s.launch_sequence && p->host_diag[4 * m] < 1e-2 && s.power_steps > s.power_steps_floor) {
        s.power_steps = std::max(s.power_steps_floor, s.power_steps - 2);
        p->leaf_steps_changed = true;
      }
    }
    s.fast_used = false;
  }
  return rejected;
}

std::vector<int> verify_fast_leaves(tp_ctx* ctx, tp_plan* p) {
  bool any = false;
  for (int m = 0; m < p->n; ++m) any = any || p->leaf[m].fast_used;
  if (!any) return {};
  queue_status_readback(ctx, p, false);
  TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  return evaluate_fast_leaves(ctx, p);
}

// A leaf whose certified solve was rejected: if only the residual bound was missed, repeat the iteration from the
// Ritz vectors it reached (each round is six more power steps, a fraction of a full eigen-solve); otherwise, or if
// that does not converge either, take the full solve on the intact Gram matrix.  Main stream.
// Returns true if the full solve had to take over.
bool redo_rejected_leaf(tp_ctx* ctx, tp_plan* p, int mode, double* dst) {
  LeafScratch& s = p->leaf[mode];
  const long long rows = static_cast<long long>(p->spec.L[mode]);
  const int k = static_cast<int>(p->spec.K[mode]);
  Span evd(ctx, p, kEvd, -1);
  bool ok = false;
  for (int round = 0; s.refinable && s.last_ritz && round < 3 && !ok; ++round) {
    leaf_solve_subspace(ctx, s, s.gram, rows, k, p->cur[mode], dst, -1);
    ok = verify_fast_leaves(ctx, p).empty();
  }
  if (!ok) {
    if (s.was_cold)
      s.cold_rejected = true;  // arbitrary start factors need more than a few rounds on this problem
    else
      ++s.failures;
    s.last_ritz = nullptr;
    leaf_solve(ctx, s, rows, k, dst, -1);
  }
  evd.close();
  return !ok;
}

// Execution order of siblings.  A Jacobi sweep gives the same factors in any order (every product uses the
// start-of-sweep factors, hooi.hpp:9-12), so children are visited leaves-first and then by descending leaf count of
// their subtrees (stable): eigen-solves start as early as possible and the remaining big products hide them.
void plan_visit_order(tp_plan* p) {
  const Tree& t = p->tree;
  std::vector<int> leaves(t.size(), 0);
  for (int id = t.size() - 1; id >= 0; --id) {
    if (t.leaf(id)) leaves[id] = 1;
    if (t.parent[id] >= 0) leaves[t.parent[id]] += leaves[id];
  }
  p->visit_order.assign(t.size(), {});
  for (int id = 0; id < t.size(); ++id) {
    std::vector<int> order = t.kids[id];
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const bool ca = !p->on_carry.empty() && p->on_carry[a], cb = !p->on_carry.empty() && p->on_carry[b];
      // the carried path ends in the mode the core chain contracts last: its leaves are needed last, so they go last
      // and their eigen-solves overlap the chain's large products.  In a short sweep (forked walk) it is the other
      // way round: the carried subtree's inputs exist when the sweep starts, the leaf solve at its end is the longest
      // dependent chain of the whole sweep (C3: 0.64 ms of 1.04) and the core waits for it -- so it is issued first
      // and everything else fills the machine beside it.
      if (ca != cb) return p->carry_first ? ca : cb;
      if (t.leaf(a) != t.leaf(b)) return t.leaf(a);
      return leaves[a] > leaves[b];
    });
    p->visit_order[id] = std::move(order);
  }
  p->leaf_rank.assign(p->n, 0);
  int next = 0;
  std::vector<int> stack{0};
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    if (t.leaf(id)) p->leaf_rank[t.mode[id]] = next++;
    for (auto it = p->visit_order[id].rbegin(); it != p->visit_order[id].rend(); ++it) stack.push_back(*it);
  }
}

cudaEvent_t next_fork_event(tp_plan* p) {
  if (p->fork_events_used == p->fork_events.size()) {
    cudaEvent_t e;
    TPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->fork_events.push_back(e);
  }
  return p->fork_events[p->fork_events_used++];
}

cudaStream_t next_branch_stream(tp_plan* p) {
  if (p->branches_used == p->branch.size()) {
    int least = 0, greatest = 0;
    TPB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    cudaStream_t st;
    TPB_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, least));  // the tree's priority
    p->branch.push_back(st);
  }
  return p->branch[p->branches_used++];
}

// Whether this sweep's walk forks, and the per-node buffers it then needs.
void plan_begin_walk(tp_plan* p) {
  p->forking = p->sweep_kind == TP_SWEEP_JACOBI && !p->arrival && p->overlap_evd &&
               (p->fork_mode == 1 || (p->fork_mode == 2 && p->short_sweep));
  p->branches_used = 0;
  p->fork_events_used = 0;
  p->branch_done.clear();
  if (!p->forking) return;
  if (p->node_buf.empty()) p->node_buf.assign(p->tree.size(), nullptr);
  for (int id = 1; id < p->tree.size(); ++id)
    if (p->node_cap[id] > 0 && !p->node_buf[id]) p->node_buf[id] = device_alloc(p->node_cap[id]);
}

// The main stream waits for every branch of the walk (before the core chain rewrites the carried products the
// branches read, and so that a recorded sweep's capture forest joins its origin stream).
void plan_join_branches(tp_ctx* ctx, tp_plan* p) {
  for (cudaEvent_t e : p->branch_done) TPB_CUDA(cudaStreamWaitEvent(ctx->stream, e, 0));
  p->branch_done.clear();
}

void jacobi_walk(tp_ctx* ctx, tp_plan* p, int node, const double* tensor, std::vector<size_t>& dims, int depth) {
  const std::vector<int>& order = p->visit_order[node];
  const bool fork = p->forking && order.size() > 1;
  cudaStream_t const home = ctx->stream;
  cudaEvent_t input_ready = nullptr;
  if (fork) {
    input_ready = next_fork_event(p);
    TPB_CUDA(cudaEventRecord(input_ready, home));
  }
  for (size_t i = 0; i < order.size(); ++i) {
    const int c = order[i];
    const int mode = p->tree.mode[c];
    // every child but the last visited gets a stream of its own; launches go to ctx->stream, which is switched for
    // the duration of the child's subtree
    struct OnBranch {
      tp_ctx* ctx;
      tp_plan* plan;
      cudaStream_t home;
      bool active;
      ~OnBranch() {
        if (!active) return;
        cudaEvent_t done = nullptr;
        try {
          done = next_fork_event(plan);
        } catch (...) {
        }
        if (done && cudaEventRecord(done, ctx->stream) == cudaSuccess) plan->branch_done.push_back(done);
        ctx->stream = home;
      }
    } on_branch{ctx, p, home, fork && i + 1 < order.size()};
    if (on_branch.active) {
      cudaStream_t st = next_branch_stream(p);
      TPB_CUDA(cudaStreamWaitEvent(st, input_ready, 0));
      ctx->stream = st;
    }
    if (p->tree.kind[c] == TP_NODE_LEAF) {
      plan_leaf(ctx, p, tensor, dims, mode, p->fresh[mode], c, p->overlap_evd);
    } else {
      double* out = p->forking ? p->node_buf[c] : p->depth_buf[depth];
      if (p->carry_live && p->on_carry[c]) {
        out = p->carry_buf[depth];  // computed by the previous sweep's core chain (path depth == tree depth)
      } else {
        Span s(ctx, p, kTree, c);
        plan_ttm(ctx, p, tensor, dims, mode, out, (p->overlap_evd && p->leaves_in_flight > 0) ? p->spare_sms : 0);
        s.close();
        plan_flush_pending(ctx, p);
      }
      const size_t saved = dims[mode];
      dims[mode] = static_cast<size_t>(p->spec.K[mode]);
      jacobi_walk(ctx, p, c, out, dims, depth + 1);
      dims[mode] = saved;
    }
  }
}

// Root level of a Jacobi walk while the tensor is still arriving (plan->arrival): slab by slab, the first root
// child that contracts a mode other than 0 multiplies its slab (slabs of mode 0 are independent there), and the
// root child that contracts mode 0 forms the slab's partial product into its own slot; the slots are summed in slab
// order once all have arrived.  Everything below the root, and any further root children, run as usual afterwards.
void jacobi_walk_streamed_root(tp_ctx* ctx, tp_plan* p, const double* tensor, std::vector<size_t>& dims) {
  tp_plan::Arrival& arr = *p->arrival;
  const Tree& t = p->tree;
  const int chunks = static_cast<int>(arr.row_end.size());
  int slab_child = -1, sum_child = -1;
  for (int c : p->visit_order[0]) {
    if (!t.internal(c)) continue;
    if (t.mode[c] == 0 && sum_child < 0) sum_child = c;
    if (t.mode[c] != 0 && slab_child < 0) slab_child = c;
  }
  const long long L0 = static_cast<long long>(dims[0]);
  long long per_row = 1;  // elements of one mode-0 row of the tensor
  for (size_t m = 1; m < dims.size(); ++m) per_row *= static_cast<long long>(dims[m]);
  // the mode-0 child needs one slot per slab; give up on streaming it when that would not fit comfortably
  size_t sum_out = 0;
  if (sum_child >= 0) {
    sum_out = static_cast<size_t>(p->spec.K[0]) * static_cast<size_t>(per_row);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const bool have = p->arrival_slot_doubles >= sum_out && static_cast<int>(p->arrival_slots.size()) >= chunks;
    if (!have && static_cast<double>(sum_out) * 8.0 * chunks > 0.5 * static_cast<double>(free_b)) {
      sum_child = -1;
    } else if (!have) {
      for (double* d : p->arrival_slots) cudaFree(d);
      p->arrival_slots.assign(chunks, nullptr);
      for (int c = 0; c < chunks; ++c) p->arrival_slots[c] = device_alloc(sum_out);
      p->arrival_slot_doubles = sum_out;
    }
  }
  if (sum_child >= 0 && static_cast<int>(p->arrival_frag.size()) < chunks) {
    p->arrival_frag.resize(chunks, nullptr);
    p->arrival_frag_doubles.resize(chunks, 0);
  }
  double* const slab_out = p->depth_buf[0];
  cudaEvent_t slab_begin = nullptr, slab_end = nullptr, sum_begin = nullptr, sum_end = nullptr;
  for (int c = 0; c < chunks; ++c) {
    arr.issue(c);
    if (c + 1 < chunks) arr.issue(c + 1);  // keep the link busy while this slab is multiplied
    TPB_CUDA(cudaStreamWaitEvent(ctx->stream, arr.ready[c], 0));
    const long long r0 = c ? static_cast<long long>(arr.row_end[c - 1]) : 0, r1 = static_cast<long long>(arr.row_end[c]);
    if (slab_child >= 0) {
      const int mode = t.mode[slab_child];
      long long outer, inner;
      mode_extents(dims, mode, outer, inner);
      const long long rest = outer / L0;  // product of the extents between mode 0 and `mode`
      const long long len = static_cast<long long>(dims[mode]), K = static_cast<long long>(p->spec.K[mode]);
      if (c == 0) {
        p->event_phase.push_back(kTree);
        p->event_node.push_back(slab_child);
        slab_begin = next_event(p);
        slab_end = next_event(p);
        TPB_CUDA(cudaEventRecord(slab_begin, ctx->stream));
      }
      TPB_CUDA(launch_ttm(ctx->stream, tensor + r0 * rest * len * inner, (r1 - r0) * rest, len, inner, p->frag[mode],
                          p->frag_layout[mode], K, slab_out + r0 * rest * K * inner, ctx->sm_count));
      ctx->own_kernels += 1;
      if (c + 1 == chunks) TPB_CUDA(cudaEventRecord(slab_end, ctx->stream));
    }
    if (sum_child >= 0) {
      const long long K = static_cast<long long>(p->spec.K[0]);
      const TtmFragmentLayout f = ttm_fragment_layout(K, r1 - r0);
      if (p->arrival_frag_doubles[c] < f.doubles) {
        cudaFree(p->arrival_frag[c]);
        p->arrival_frag[c] = device_alloc(f.doubles);
        p->arrival_frag_doubles[c] = f.doubles;
      }
      if (c == 0) {
        p->event_phase.push_back(kTree);
        p->event_node.push_back(sum_child);
        sum_begin = next_event(p);
        sum_end = next_event(p);
        TPB_CUDA(cudaEventRecord(sum_begin, ctx->stream));
      }
      // M = F_0^T restricted to the slab's rows: M(k, l) = F_0[k * L_0 + r0 + l]
      TPB_CUDA(prep_factor_fragments(ctx->stream, p->cur[0] + r0, L0, 1, K, r1 - r0, f, p->arrival_frag[c]));
      TPB_CUDA(launch_ttm(ctx->stream, tensor + r0 * per_row, 1, r1 - r0, per_row, p->arrival_frag[c], f, K,
                          p->arrival_slots[c], ctx->sm_count));
      ctx->own_kernels += 2;
    }
  }
  // main stream is now ordered after every slab: the rest of the sweep may read the whole tensor
  auto descend = [&](int c, double* out) {
    const int mode = t.mode[c];
    const size_t saved = dims[mode];
    dims[mode] = static_cast<size_t>(p->spec.K[mode]);
    jacobi_walk(ctx, p, c, out, dims, 1);
    dims[mode] = saved;
  };
  // the slab child first: its product sits in the depth-0 buffer the other root children reuse
  std::vector<int> order;
  if (slab_child >= 0) order.push_back(slab_child);
  for (int c : p->visit_order[0])
    if (c != slab_child) order.push_back(c);
  for (int c : order) {
    const int mode = t.mode[c];
    if (t.kind[c] == TP_NODE_LEAF) {
      plan_leaf(ctx, p, tensor, dims, mode, p->fresh[mode], c, p->overlap_evd);
    } else if (c == slab_child) {
      descend(c, slab_out);
    } else if (c == sum_child) {
      std::vector<const double*> slots(p->arrival_slots.begin(), p->arrival_slots.begin() + chunks);
      TPB_CUDA(launch_reduce_slots(ctx->stream, p->depth_buf[0], slots.data(), chunks, sum_out));
      TPB_CUDA(cudaEventRecord(sum_end, ctx->stream));
      ctx->own_kernels += 1;
      plan_flush_pending(ctx, p);
      descend(c, p->depth_buf[0]);
    } else {
      double* out = p->depth_buf[0];
      Span s(ctx, p, kTree, c);
      plan_ttm(ctx, p, tensor, dims, mode, out, (p->overlap_evd && p->leaves_in_flight > 0) ? p->spare_sms : 0);
      s.close();
      plan_flush_pending(ctx, p);
      descend(c, out);
    }
  }
}

// core_from_factors (hooi.hpp:93-100): T x_0 F_0^T ... x_{N-1} F_{N-1}^T.  Mode products along different modes
// commute, so the chain runs in the cheapest order (plan->core_order) instead of the reference's fixed 0..N-1; the
// result differs from the reference's only by rounding.  Ping-pong buffers, the last product lands in `core`.
void plan_core(tp_ctx* ctx, tp_plan* p, const double* tensor, const std::vector<double*>& factors,
               bool wait_for_leaves = false) {
  const bool carry = p->carry_enabled && !p->carry_nodes.empty();
  std::vector<size_t> dims(p->spec.L.begin(), p->spec.L.end());
  const double* src = tensor;
  // Short sweeps: each new factor is put into fragment order on its solve's side stream, right behind the solve
  // (once the walk, which still reads the old fragments, is through), instead of in front of every chain product on
  // the main stream -- all but the first-needed factor's preparation then hides behind the chain.
  const bool side_prep = wait_for_leaves && p->forking;
  if (side_prep) {
    plan_flush_pending(ctx, p);
    cudaEvent_t walk_done = next_fork_event(p);
    TPB_CUDA(cudaEventRecord(walk_done, ctx->stream));
    cudaStream_t const home = ctx->stream;
    for (int i = 0; i < p->n; ++i) {
      const int m = p->core_order[i];
      cudaStream_t const side = ctx->aux[m % tp_ctx::kAux];
      TPB_CUDA(cudaStreamWaitEvent(side, walk_done, 0));
      ctx->stream = side;
      try {
        plan_refresh_fragments(ctx, p, m, factors[m]);
      } catch (...) {
        ctx->stream = home;
        throw;
      }
      ctx->stream = home;
      TPB_CUDA(cudaEventRecord(p->factor_ready[m], side));
    }
  }
  bool solves_covered = false;
  for (int i = 0; i < p->n; ++i) {
    const int m = p->core_order[i];
    if (wait_for_leaves) {
      // a factor whose eigen-solve is still unqueued must be queued before the chain can wait for it
      for (const tp_plan::PendingLeaf& job : p->pending)
        if (job.mode == m) {
          plan_flush_pending(ctx, p);
          break;
        }
      TPB_CUDA(cudaStreamWaitEvent(ctx->stream, p->factor_ready[m], 0));
    }
    const bool last = i == p->n - 1;
    // along a carried path the partial products are next sweep's tree nodes: timed as such, kept in their buffers
    Span s = (carry && !last) ? Span(ctx, p, kTree, p->carry_nodes[i]) : Span(ctx, p, kCore);
    if (!side_prep) plan_refresh_fragments(ctx, p, m, factors[m]);
    double* dst = last ? p->core : (carry ? p->carry_buf[i] : p->core_tmp[i & 1]);
    // solves of the modes the chain has not waited for yet may still be running on the side streams: the persistent
    // product grid must leave them SMs (its CTAs would otherwise hold every SM until the product ends, and a solve
    // queued meanwhile would start only then -- exposed on the critical path of short sweeps)
    // ...unless a long product has been queued since the last solve was: a solve is a few milliseconds of small
    // kernels, so those still in flight then are over long before a later chain product starts, and sparing SMs for
    // them would only idle those SMs for the whole product (C5: 57.02 -> 56.85 ms/iter).  (Measured and rejected:
    // the long product itself as two launches, an eighth beside the solves and the rest on the whole machine -- the
    // solves take longer than that eighth under contention and then starve behind the second launch, 62.7 ms/iter.)
    const bool solves_running =
        wait_for_leaves && !last && !solves_covered && (p->leaves_in_flight > 0 || !p->pending.empty());
    long long outer_m, inner_m;
    mode_extents(dims, m, outer_m, inner_m);
    const double flops = 2.0 * static_cast<double>(p->spec.K[m]) * static_cast<double>(outer_m) *
                         static_cast<double>(dims[m]) * static_cast<double>(inner_m);
    const bool long_product = flops >= 2.5 * p->short_product_flops;
    plan_ttm(ctx, p, src, dims, m, dst, solves_running ? p->spare_sms : 0);
    if (long_product) solves_covered = true;
    s.close();
    if (wait_for_leaves) plan_flush_pending(ctx, p);
    dims[m] = static_cast<size_t>(p->spec.K[m]);
    src = dst;
  }
}

// Picks the path the core chain follows (see tp_plan::carry_nodes) and fixes the order of the chain accordingly.
// Any root-to-leaf path works and all cost the same in steady state (tree + one product onto the core), so the choice
// goes by scheduling: the chain's first product needs the new factor of the path's first mode, whose leaf lies in
// another subtree -- take the path for which that leaf (then the second mode's, ...) comes earliest in the walk.
void plan_choose_carry(tp_plan* p) {
  const Tree& t = p->tree;
  p->carry_nodes.clear();
  p->carry_leaf_mode = -1;
  p->on_carry.assign(t.size(), 0);
  if (p->n < 2) {
    plan_visit_order(p);
    return;
  }
  if (p->sweep_kind != TP_SWEEP_JACOBI) {
    // Gauss-Seidel (chain trees): the first chain of a sweep multiplies by F_1 .. F_{N-1} as they stand at the end
    // of the previous sweep -- the factors the core chain uses.  Carry that chain; the core closes it with F_0.
    for (int leaf = 0; leaf < t.size(); ++leaf) {
      if (!t.leaf(leaf) || t.mode[leaf] != 0) continue;
      for (int id = t.parent[leaf]; id > 0; id = t.parent[id]) p->carry_nodes.push_back(id);
      std::reverse(p->carry_nodes.begin(), p->carry_nodes.end());
      for (int id : p->carry_nodes) p->on_carry[id] = 1;
      p->carry_leaf_mode = 0;
      break;
    }
    plan_visit_order(p);
    return;
  }
  std::vector<int> best_nodes, best_key;
  int best_leaf = -1;
  for (int leaf = 0; leaf < t.size(); ++leaf) {
    if (!t.leaf(leaf)) continue;
    std::vector<int> nodes;
    for (int id = t.parent[leaf]; id > 0; id = t.parent[id]) nodes.push_back(id);
    std::reverse(nodes.begin(), nodes.end());
    if (static_cast<int>(nodes.size()) != p->n - 1) continue;  // (always n - 1 TTM nodes above a leaf)
    p->on_carry.assign(t.size(), 0);
    for (int id : nodes) p->on_carry[id] = 1;
    plan_visit_order(p);
    std::vector<int> key;
    if (p->carry_first) {
      // the carried subtree goes first so that the leaf solve at its end starts at once: take the path that ends in
      // the dearest solve (rows x block^2; the chain's needs decide among equals)
      const int lm = t.mode[leaf];
      const double block = static_cast<double>(p->spec.K[lm]) + 8.0;
      const double cost = static_cast<double>(p->spec.L[lm]) * block * block;
      key.push_back(-static_cast<int>(std::min(cost / 64.0, 2e9)));
    }
    for (int id : nodes) key.push_back(p->leaf_rank[t.mode[id]]);
    if (best_leaf < 0 || key < best_key) {
      best_key = key;
      best_nodes = nodes;
      best_leaf = leaf;
    }
  }
  p->on_carry.assign(t.size(), 0);
  if (best_leaf >= 0) {
    for (int id : best_nodes) p->on_carry[id] = 1;
    p->carry_nodes = best_nodes;
    p->carry_leaf_mode = t.mode[best_leaf];
  }
  plan_visit_order(p);
}

// Cheapest order of the core chain: forward DP over the set of already-multiplied modes; ties keep the smaller mode
// first (strict improvement only, modes scanned ascending), so the reference order wins whenever it is optimal.
// Among equally cheap orders the mode whose new factor is finished first (`rank`, smaller = earlier) goes first, so
// the chain's first — largest — product can start while later eigen-solves are still running.
std::vector<int> cheapest_chain_order(const Spec& s, const std::vector<int>& rank, u64* macs_out) {
  const int n = s.n();
  const std::uint32_t full = (n >= 32) ? ~0u : ((1u << n) - 1);
  auto card_of = [&](std::uint32_t done) {
    u64 card = 1;
    for (int m = 0; m < n; ++m) card = mul_sat(card, ((done >> m) & 1u) ? s.K[m] : s.L[m]);
    return card;
  };
  // togo[S] = fewest MACs to finish from the state where the modes of S are already multiplied
  std::vector<u64> togo(static_cast<size_t>(full) + 1, kSat);
  togo[full] = 0;
  for (std::uint32_t done = full; done-- > 0;) {
    const u64 card = card_of(done);
    for (int m = 0; m < n; ++m) {
      if ((done >> m) & 1u) continue;
      const u64 c = add_sat(mul_sat(s.K[m], card), togo[done | (1u << m)]);
      if (c < togo[done]) togo[done] = c;
    }
  }
  std::vector<int> order;
  std::uint32_t done = 0;
  while (done != full) {
    const u64 card = card_of(done);
    int pick = -1;
    for (int m = 0; m < n; ++m) {
      if ((done >> m) & 1u) continue;
      if (add_sat(mul_sat(s.K[m], card), togo[done | (1u << m)]) != togo[done]) continue;
      if (pick < 0 || rank[m] < rank[pick]) pick = m;
    }
    order.push_back(pick);
    done |= 1u << pick;
  }
  if (macs_out) *macs_out = togo[0];
  return order;
}

// The chain just run left the path products of (t, current factors) in the carry buffers.
void plan_mark_carried(tp_plan* p, const tp_tensor* t) {
  if (!p->carry_enabled || p->carry_nodes.empty()) return;
  p->carry_valid = true;
  p->carry_tensor = t;
  p->carry_stamp = t->stamp;
}

void check_tensor_matches(const tp_plan* p, const tp_tensor* t) {  // hooi.hpp:85-91
  if (!t) raise(TP_ERR_BAD_ARGUMENT, "null tensor");
  if (static_cast<int>(t->dims.size()) != p->n) raise(TP_ERR_SHAPE_MISMATCH, "tensor and spec mode counts differ");
  for (int m = 0; m < p->n; ++m)
    if (t->dims[m] != p->spec.L[m]) raise(TP_ERR_SHAPE_MISMATCH, "tensor extent differs from L", m);
}

void plan_collect_timing(tp_ctx* ctx, tp_plan* p) {
  TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int a = 0; a < tp_ctx::kAux; ++a) TPB_CUDA(cudaStreamSynchronize(ctx->aux[a]));
  tp_sweep_timing t{};
  float* slot[4] = {&t.tree_ms, &t.gram_ms, &t.evd_ms, &t.core_ms};
  p->node_ms.assign(p->tree.size(), 0.f);
  p->node_evd_ms.assign(p->tree.size(), 0.f);
  for (size_t i = 0; i < p->event_phase.size(); ++i) {
    float ms = 0.f;
    TPB_CUDA(cudaEventElapsedTime(&ms, p->events[2 * i], p->events[2 * i + 1]));
    *slot[p->event_phase[i]] += ms;
    const int node = p->event_node[i];
    if (node >= 0) (p->event_phase[i] == kEvd ? p->node_evd_ms : p->node_ms)[node] += ms;
  }
  if (!p->event_phase.empty()) {
    // first span's begin to the end of the last main-stream span (the core chain closes every sweep)
    size_t last = 0;
    for (size_t i = 0; i < p->event_phase.size(); ++i)
      if (p->event_phase[i] != kEvd) last = i;
    float ms = 0.f;
    TPB_CUDA(cudaEventElapsedTime(&ms, p->events[0], p->events[2 * last + 1]));
    t.total_ms = ms;
  }
  p->timing = t;
}

}  // namespace
}  // namespace tpb

static void release_host_call_cache(tp_ctx* ctx) {
  if (ctx->host_call_plan) tp_plan_destroy(ctx, ctx->host_call_plan);
  if (ctx->host_call_tensor) tp_tensor_free(ctx, ctx->host_call_tensor);
  ctx->host_call_plan = nullptr;
  ctx->host_call_tensor = nullptr;
  ctx->host_call_key.clear();
  ctx->host_call_source = nullptr;
  ctx->host_call_last_factors.clear();
}

extern "C" {

int tp_device_count(int* out) {
  return guarded([&] {
    if (!out) raise(TP_ERR_BAD_ARGUMENT, "null output");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
      cudaGetLastError();
      count = 0;
    }
    *out = count;
  });
}

int tp_ctx_create(int device, tp_ctx** out) { return tp_ctx_create_ex(device, 0, out); }

int tp_ctx_create_ex(int device, unsigned flags, tp_ctx** out) {
  return guarded([&] {
    if (!out) raise(TP_ERR_BAD_ARGUMENT, "null output");
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      raise(TP_ERR_CUDA, std::string("no CUDA device available (this engine has no CPU fallback): ") +
                             cudaGetErrorString(e));
    if (device < 0 || device >= count) raise(TP_ERR_BAD_ARGUMENT, "device index out of range");
    cudaDeviceProp prop;
    TPB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      raise(TP_ERR_CUDA, std::string("device '") + prop.name + "' is not sm_100: this library carries sm_100a code only");
    tp_ctx* ctx = new tp_ctx;
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    try {
      TPB_CUDA(cudaSetDevice(device));
      int least = 0, greatest = 0;  // numerically: greatest priority = smallest value
      TPB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      // The eigen-solve side streams outrank the tree's stream: their kernels are short and latency-bound, and a
      // leaf's factor is needed by the core chain soon after its Gram matrix is done, so they should not queue
      // behind the thousands of CTAs of a Gram or TTM launch (measured on C5: 58.4 -> 57.8 ms/iter together with
      // the wider SM share short products leave them).  TP_CTX_SIDE_STREAMS_* flags: same priority / below the tree.
      int main_prio = least, side_prio = greatest;
      if (flags & TP_CTX_SIDE_STREAMS_SAME_PRIORITY) side_prio = main_prio;
      if (flags & TP_CTX_SIDE_STREAMS_LOW_PRIORITY) std::swap(main_prio, side_prio);
      TPB_CUDA(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, main_prio));
      TPB_SOLVER(cusolverDnCreate(&ctx->solver));
      TPB_SOLVER(cusolverDnSetStream(ctx->solver, ctx->stream));
      ctx->reduce_scratch = device_alloc(reduce_scratch_doubles() + 1);
      TPB_BLAS(cublasCreate(&ctx->blas));
      TPB_BLAS(cublasSetStream(ctx->blas, ctx->stream));
      TPB_CUDA(cudaMalloc(&ctx->blas_ws[tp_ctx::kAux], tp_ctx::kBlasWorkspaceBytes));
      TPB_BLAS(cublasSetWorkspace(ctx->blas, ctx->blas_ws[tp_ctx::kAux], tp_ctx::kBlasWorkspaceBytes));
      for (int a = 0; a < tp_ctx::kAux; ++a) {
        TPB_CUDA(cudaStreamCreateWithPriority(&ctx->aux[a], cudaStreamNonBlocking, side_prio));
        TPB_SOLVER(cusolverDnCreate(&ctx->aux_solver[a]));
        TPB_SOLVER(cusolverDnSetStream(ctx->aux_solver[a], ctx->aux[a]));
        TPB_BLAS(cublasCreate(&ctx->aux_blas[a]));
        TPB_BLAS(cublasSetStream(ctx->aux_blas[a], ctx->aux[a]));
        TPB_CUDA(cudaMalloc(&ctx->blas_ws[a], tp_ctx::kBlasWorkspaceBytes));
        TPB_BLAS(cublasSetWorkspace(ctx->aux_blas[a], ctx->blas_ws[a], tp_ctx::kBlasWorkspaceBytes));
      }
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int tp_ctx_destroy(tp_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->solver) cusolverDnDestroy(ctx->solver);
    if (ctx->blas) cublasDestroy(ctx->blas);
    for (int a = 0; a < tp_ctx::kAux; ++a) {
      if (ctx->aux[a]) cudaStreamSynchronize(ctx->aux[a]);
      if (ctx->aux_solver[a]) cusolverDnDestroy(ctx->aux_solver[a]);
      if (ctx->aux_blas[a]) cublasDestroy(ctx->aux_blas[a]);
      if (ctx->aux[a]) cudaStreamDestroy(ctx->aux[a]);
    }
    cudaFree(ctx->reduce_scratch);
    cudaFree(ctx->frag_scratch);
    for (cudaEvent_t e : ctx->arrival_events) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (void* ws : ctx->blas_ws) cudaFree(ws);
    release_host_call_cache(ctx);
    for (tp_ctx::Lane& lane : ctx->lanes) {
      if (lane.scratch) {
        static_cast<LeafScratch*>(lane.scratch)->release();
        delete static_cast<LeafScratch*>(lane.scratch);
      }
      if (lane.ready) cudaEventDestroy(lane.ready);
      if (lane.done) cudaEventDestroy(lane.done);
    }
    if (ctx->dev_scratch) {
      static_cast<LeafScratch*>(ctx->dev_scratch)->release();
      delete static_cast<LeafScratch*>(ctx->dev_scratch);
    }
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int tp_ctx_set_option(tp_ctx* ctx, int option, long long value) {
  return guarded([&] {
    if (!ctx) raise(TP_ERR_BAD_ARGUMENT, "null context");
    if (option == TP_CTX_OPT_STREAMED_UPLOAD_MIN_BYTES) {
      if (value < 0) raise(TP_ERR_BAD_ARGUMENT, "negative size");
      ctx->streamed_upload_min_bytes = static_cast<size_t>(value);
    } else if (option == TP_CTX_OPT_TRACE_EVD) {
      ctx->trace_evd = value != 0;
    } else if (option == TP_CTX_OPT_DUMP_SWEEP_GRAPH) {
      ctx->dump_sweep_graph = value != 0;
    } else {
      raise(TP_ERR_BAD_ARGUMENT, "unknown context option");
    }
  });
}

int tp_set_global_option(int option, long long value) {
  return guarded([&] {
    if (option == TP_GLOBAL_OPT_TTM_TMA)
      ttm_tma_enabled().store(value != 0, std::memory_order_relaxed);
    else if (option == TP_GLOBAL_OPT_TTM_PACKED)
      ttm_packed_enabled().store(value != 0, std::memory_order_relaxed);
    else if (option == TP_GLOBAL_OPT_TTM_SPLITK)
      ttm_splitk_enabled().store(value != 0, std::memory_order_relaxed);
    else if (option == TP_GLOBAL_OPT_CARRY_FIRST)
      carry_first_mode().store(static_cast<int>(std::max(0LL, std::min(value, 2LL))), std::memory_order_relaxed);
    else if (option == TP_GLOBAL_OPT_GRAM_WIDE)
      gram_wide_enabled().store(value != 0, std::memory_order_relaxed);
    else if (option == TP_GLOBAL_OPT_GRAM_WIDE_SPARE_SMS)
      gram_wide_spare_sms().store(static_cast<int>(std::max(0LL, std::min(value, 64LL))), std::memory_order_relaxed);
    else
      raise(TP_ERR_BAD_ARGUMENT, "unknown global option");
  });
}

int tp_ctx_synchronize(tp_ctx* ctx) {
  return guarded([&] {
    bind(ctx);
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tp_ctx_stream(tp_ctx* ctx, void** stream_out) {
  return guarded([&] {
    bind(ctx);
    *stream_out = static_cast<void*>(ctx->stream);
  });
}

int tp_ctx_launch_counts(tp_ctx* ctx, tp_u64* own_kernels, tp_u64* library_calls) {
  return guarded([&] {
    if (!ctx) raise(TP_ERR_BAD_ARGUMENT, "null context");
    if (own_kernels) *own_kernels = ctx->own_kernels;
    if (library_calls) *library_calls = ctx->library_calls;
  });
}

int tp_host_alloc(size_t bytes, void** out) {
  return guarded([&] { TPB_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocDefault)); });
}

int tp_host_free(void* p) {
  return guarded([&] {
    if (p) TPB_CUDA(cudaFreeHost(p));
  });
}

int tp_tensor_upload(tp_ctx* ctx, int n_modes, const size_t* dims, const double* host, tp_tensor** out) {
  return guarded([&] {
    bind(ctx);
    if (!host || !out) raise(TP_ERR_BAD_ARGUMENT, "null buffer");
    checked_size(n_modes, dims);
    tp_tensor* t = new_tensor(std::vector<size_t>(dims, dims + n_modes));
    const cudaError_t e = cudaMemcpyAsync(t->data, host, t->size * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) {
      cudaFree(t->data);
      delete t;
      cuda_fail(e, "tensor upload");
    }
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = t;
  });
}

int tp_tensor_alloc(tp_ctx* ctx, int n_modes, const size_t* dims, tp_tensor** out) {
  return guarded([&] {
    bind(ctx);
    if (!out) raise(TP_ERR_BAD_ARGUMENT, "null output");
    checked_size(n_modes, dims);
    tp_tensor* t = new_tensor(std::vector<size_t>(dims, dims + n_modes));
    TPB_CUDA(cudaMemsetAsync(t->data, 0, t->size * sizeof(double), ctx->stream));
    *out = t;
  });
}

int tp_tensor_download(tp_ctx* ctx, const tp_tensor* t, double* host) {
  return guarded([&] {
    bind(ctx);
    if (!t || !host) raise(TP_ERR_BAD_ARGUMENT, "null buffer");
    TPB_CUDA(cudaMemcpyAsync(host, t->data, t->size * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tp_tensor_free(tp_ctx* ctx, tp_tensor* t) {
  return guarded([&] {
    if (!t) return;
    bind(ctx);
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(t->data);
    delete t;
  });
}

int tp_tensor_dims(const tp_tensor* t, int* n_modes, size_t* dims) {
  return guarded([&] {
    if (!t) raise(TP_ERR_BAD_ARGUMENT, "null tensor");
    if (n_modes) *n_modes = static_cast<int>(t->dims.size());
    if (dims) std::copy(t->dims.begin(), t->dims.end(), dims);
  });
}

void* tp_tensor_device_ptr(const tp_tensor* t) {
  if (!t) return nullptr;
  // the caller may write through the pointer at any later time: no product of this tensor is carried between sweeps
  // until tp_tensor_mark_modified puts the caller in charge of announcing writes
  const_cast<tp_tensor*>(t)->stamp = next_tensor_stamp();
  const_cast<tp_tensor*>(t)->pointer_escaped = true;
  return t->data;
}

int tp_tensor_mark_modified(tp_ctx* ctx, tp_tensor* t) {
  return guarded([&] {
    (void)ctx;
    if (!t) raise(TP_ERR_BAD_ARGUMENT, "null tensor");
    t->stamp = next_tensor_stamp();
    t->pointer_escaped = false;  // from here on the caller announces every write with this call
  });
}

int tp_tensor_norm(tp_ctx* ctx, const tp_tensor* t, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!t || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    *out = std::sqrt(sum_squares(ctx, t->data, t->size));
  });
}

static void ttm_common(tp_ctx* ctx, const tp_tensor* t, const double* m_dev, long long row_stride,
                       long long col_stride, size_t m_rows, size_t m_cols, int mode, tp_u64* macs, tp_tensor** out) {
  if (!t || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
  long long outer, inner;
  mode_extents(t->dims, mode, outer, inner);  // bad_mode, ttm.hpp:26-27
  if (m_cols != t->dims[mode]) raise(TP_ERR_SHAPE_MISMATCH, "matrix columns must match the mode extent");
  if (m_rows == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
  std::vector<size_t> out_dims = t->dims;
  out_dims[mode] = m_rows;
  tp_tensor* z = new_tensor(out_dims);
  try {
    run_ttm(ctx, t->data, t->dims, mode, m_dev, row_stride, col_stride, static_cast<long long>(m_rows), nullptr,
            z->data);
    if (macs) *macs = add_or_throw(*macs, mul_or_throw(m_rows, t->size));  // ttm.hpp:92-94
  } catch (...) {
    cudaFree(z->data);
    delete z;
    throw;
  }
  *out = z;
}

int tp_ttm(tp_ctx* ctx, const tp_tensor* t, const double* m, size_t m_rows, size_t m_cols, int mode, tp_u64* macs,
           tp_tensor** out) {
  return guarded([&] {
    bind(ctx);
    if (!m || !t) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    {  // argument errors in the reference's order (ttm.hpp:75-80) before any device work
      long long o, i;
      mode_extents(t->dims, mode, o, i);
      if (m_cols != t->dims[mode]) raise(TP_ERR_SHAPE_MISMATCH, "matrix columns must match the mode extent");
      if (m_rows == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
    }
    double* m_dev = device_alloc(m_rows * m_cols);
    try {
      TPB_CUDA(cudaMemcpyAsync(m_dev, m, m_rows * m_cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      // column-major host matrix: M(k, l) at m[l * m_rows + k]
      ttm_common(ctx, t, m_dev, 1, static_cast<long long>(m_rows), m_rows, m_cols, mode, macs, out);
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(m_dev);
      throw;
    }
    cudaFree(m_dev);
  });
}

int tp_ttm_device(tp_ctx* ctx, const tp_tensor* t, const double* m_dev_rowmajor, size_t m_rows, size_t m_cols,
                  int mode, tp_u64* macs, tp_tensor** out) {
  return guarded([&] {
    bind(ctx);
    if (!m_dev_rowmajor) raise(TP_ERR_BAD_ARGUMENT, "null matrix");
    ttm_common(ctx, t, m_dev_rowmajor, static_cast<long long>(m_cols), 1, m_rows, m_cols, mode, macs, out);
  });
}

int tp_gram(tp_ctx* ctx, const tp_tensor* t, int mode, double* gram_out) {
  return guarded([&] {
    bind(ctx);
    if (!t || !gram_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    long long outer, inner;
    mode_extents(t->dims, mode, outer, inner);
    const long long rows = static_cast<long long>(t->dims[mode]);
    const GramLayout g = gram_layout(outer, rows, inner, ctx->sm_count);
    double* ws = device_alloc(g.workspace_doubles);
    double* gram = device_alloc(static_cast<size_t>(rows) * rows);
    cudaError_t e = launch_gram(ctx->stream, t->data, outer, rows, inner, g, ws, gram);
    ctx->own_kernels += 2;
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(gram_out, gram, sizeof(double) * rows * rows, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(ws);
    cudaFree(gram);
    if (e != cudaSuccess) cuda_fail(e, "gram");
  });
}

int tp_leaf_factor(tp_ctx* ctx, const tp_tensor* t, int mode, int k, double* vectors_out, int* degenerate) {
  return guarded([&] {
    bind(ctx);
    if (!t || !vectors_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    long long outer, inner;
    mode_extents(t->dims, mode, outer, inner);
    const long long rows = static_cast<long long>(t->dims[mode]);
    check_leaf_args(rows, outer * inner, k);
    LeafScratch s;
    double* factor = nullptr;
    try {
      factor = device_alloc(static_cast<size_t>(rows) * k);
      leaf_update(ctx, s, t->data, t->dims, mode, k, factor);
      TPB_CUDA(cudaMemcpyAsync(vectors_out, factor, sizeof(double) * rows * k, cudaMemcpyDeviceToHost, ctx->stream));
      const int flag = read_and_clear_flag(ctx, s);
      if (degenerate) *degenerate = flag;
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(factor);
      s.release();
      throw;
    }
    cudaFree(factor);
    s.release();
  });
}

int tp_leading_left_factors(tp_ctx* ctx, const double* m, size_t rows, size_t cols, int k, double* vectors_out,
                            int* degenerate) {
  return guarded([&] {
    bind(ctx);
    check_leaf_args(static_cast<long long>(rows), static_cast<long long>(cols), k);
    if (!m || !vectors_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    // a column-major rows x cols matrix is, in memory, the row-major tensor (cols, rows); its mode-1 Gram is m m^T
    const size_t dims[2] = {cols, rows};
    tp_tensor* t = nullptr;
    int status = tp_tensor_upload(ctx, 2, dims, m, &t);
    if (status != TP_OK) raise(status, tp_last_error(), tp_last_error_mode());
    status = tp_leaf_factor(ctx, t, 1, k, vectors_out, degenerate);
    const std::string msg = status != TP_OK ? tp_last_error() : "";
    const int bad_mode = tp_last_error_mode();
    tp_tensor_free(ctx, t);
    if (status != TP_OK) raise(status, msg, bad_mode);
  });
}

// Sequentially truncated HOSVD (Vannieuwenhoven, Vandebril, Meerbergen 2012): for each mode in `order`, the leading
// K_n left singular vectors of the mode-n unfolding of the CURRENT tensor become F_n (Gram + eigen-solve + the
// reference's sign rule, exactly as a HOOI leaf, hooi.hpp:45-76), and the tensor is truncated, X <- X x_n F_n^T,
// before the next mode.  The last X is the core of those factors.  What real users start HOOI from;
// the reference itself only offers the random start.  Factors stay on the device in `factors_dev`.
static tp_tensor* sthosvd_device(tp_ctx* ctx, const tp_tensor* t, const std::vector<u64>& K, const std::vector<int>& order,
                                 const std::vector<double*>& factors_dev, int* degenerate, tp_u64* macs) {
  const int n = static_cast<int>(t->dims.size());
  const double* src = t->data;
  std::vector<size_t> dims = t->dims;
  tp_tensor* current = nullptr;
  LeafScratch scratch;
  try {
    for (int step = 0; step < n; ++step) {
      const int m = order[step];
      const int k = static_cast<int>(K[m]);
      leaf_update(ctx, scratch, src, dims, m, k, factors_dev[m]);
      if (macs) {
        size_t count = 1;
        for (size_t d : dims) count *= d;
        *macs = add_or_throw(*macs, mul_or_throw(static_cast<u64>(k), static_cast<u64>(count)));
      }
      std::vector<size_t> out_dims = dims;
      out_dims[m] = static_cast<size_t>(k);
      tp_tensor* next = new_tensor(out_dims);
      try {
        // M = F^T: M(k, l) = F[k * L + l]
        run_ttm(ctx, src, dims, m, factors_dev[m], static_cast<long long>(dims[m]), 1, k, nullptr, next->data);
        TPB_CUDA(cudaStreamSynchronize(ctx->stream));
      } catch (...) {
        cudaFree(next->data);
        delete next;
        throw;
      }
      if (current) {
        cudaFree(current->data);
        delete current;
      }
      current = next;
      src = current->data;
      dims = out_dims;
    }
    const int flag = read_and_clear_flag(ctx, scratch);
    if (degenerate) *degenerate = flag;
  } catch (...) {
    cudaStreamSynchronize(ctx->stream);
    if (current) {
      cudaFree(current->data);
      delete current;
    }
    scratch.release();
    throw;
  }
  scratch.release();
  return current;
}

static std::vector<int> sthosvd_order(int n, const int* order) {
  std::vector<int> out(n);
  std::vector<char> seen(n, 0);
  for (int i = 0; i < n; ++i) {
    out[i] = order ? order[i] : i;
    if (out[i] < 0 || out[i] >= n || seen[out[i]]) raise(TP_ERR_BAD_ARGUMENT, "order must be a permutation of the modes");
    seen[out[i]] = 1;
  }
  return out;
}

int tp_sthosvd(tp_ctx* ctx, const tp_tensor* t, const tp_u64* K, const int* order, double* const* factors_out,
               double* core_out, int* degenerate, tp_u64* macs) {
  return guarded([&] {
    bind(ctx);
    if (!t || !K) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    const int n = static_cast<int>(t->dims.size());
    std::vector<u64> L(t->dims.begin(), t->dims.end()), ks(K, K + n);
    validate_spec(make_spec(n, L.data(), ks.data()));
    for (int m = 0; m < n; ++m)
      if (L[m] > TP_MAX_GRAM_ROWS) raise(TP_ERR_TOO_LARGE, "unfolding has too many rows for the Gram route", m);
    const std::vector<int> ord = sthosvd_order(n, order);
    std::vector<double*> factors(n, nullptr);
    tp_tensor* core = nullptr;
    auto cleanup = [&] {
      cudaStreamSynchronize(ctx->stream);
      for (double* f : factors) cudaFree(f);
      if (core) {
        cudaFree(core->data);
        delete core;
      }
    };
    try {
      for (int m = 0; m < n; ++m) factors[m] = device_alloc(static_cast<size_t>(L[m] * ks[m]));
      core = sthosvd_device(ctx, t, ks, ord, factors, degenerate, macs);
      for (int m = 0; m < n && factors_out; ++m)
        TPB_CUDA(cudaMemcpyAsync(factors_out[m], factors[m], sizeof(double) * L[m] * ks[m], cudaMemcpyDeviceToHost,
                                 ctx->stream));
      if (core_out)
        TPB_CUDA(cudaMemcpyAsync(core_out, core->data, sizeof(double) * core->size, cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int tp_plan_init_sthosvd(tp_ctx* ctx, tp_plan* p, const tp_tensor* t, const int* order) {
  return guarded([&] {
    bind(ctx);
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    check_tensor_matches(p, t);
    const std::vector<int> ord = sthosvd_order(p->n, order);
    tp_tensor* core = sthosvd_device(ctx, t, p->spec.K, ord, p->cur, nullptr, nullptr);
    // the plan's core is the core of its current factors (as after tp_plan_compute_core)
    const cudaError_t e = cudaMemcpyAsync(p->core, core->data, sizeof(double) * p->core_size, cudaMemcpyDeviceToDevice,
                                          ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(core->data);
    delete core;
    if (e != cudaSuccess) cuda_fail(e, "copy of the truncated core");
    p->carry_valid = false;
    p->factors_from_caller = true;   // a start like any other: the first sweep's solves are cold
    p->frags_match_cur = false;
    p->warm_sweeps = 0;
    for (LeafScratch& slot : p->leaf) slot.last_ritz = nullptr;
  });
}

int tp_plan_create(tp_ctx* ctx, int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind,
                   const int* mode, const int* parent, int sweep_kind, tp_plan** out) {
  return guarded([&] {
    bind(ctx);
    if (!out) raise(TP_ERR_BAD_ARGUMENT, "null output");
    if (sweep_kind != TP_SWEEP_JACOBI && sweep_kind != TP_SWEEP_GAUSS_SEIDEL)
      raise(TP_ERR_BAD_ARGUMENT, "unknown sweep kind");
    tp_plan* p = new tp_plan;
    try {
      p->spec = make_spec(n_modes, L, K);
      validate_spec(p->spec);
      p->n = n_modes;
      p->tree = tree_from_arrays(n_modes, n_nodes, kind, mode, parent);
      validate_tree(p->tree, p->spec);
      p->sweep_kind = sweep_kind;
      Cards cards;
      const Cost cost = tree_cost(p->tree, p->spec, &cards);
      for (int m = 0; m < n_modes; ++m)
        if (p->spec.L[m] > TP_MAX_GRAM_ROWS)
          raise(TP_ERR_TOO_LARGE, "unfolding has too many rows for the Gram route", m);  // hooi.hpp:48-49

      // SweepStats are properties of (spec, tree, kind): tree_macs == tree_cost, core_macs in mode order
      p->model.tree_macs = cost.total_macs;
      u64 card = partial_cardinality(p->spec, 0), core_macs = 0;
      for (int m = 0; m < n_modes; ++m) {
        core_macs = add_or_throw(core_macs, mul_or_throw(p->spec.K[m], card));
        card = scale_exact(card, p->spec.K[m], p->spec.L[m]);
      }
      p->model.core_macs = core_macs;
      p->core_size = static_cast<size_t>(card);
      if (sweep_kind == TP_SWEEP_JACOBI) {
        p->model.peak_live = cost.depth + 1;  // hooi.hpp:143-144: live grows by one per mode node on the path
      } else {
        p->gs_paths = chain_paths(p->tree);  // needs_chain_tree
        u64 macs = 0;
        int peak = 1;
        for (int leaf = 0; leaf < n_modes; ++leaf) {
          u64 c = partial_cardinality(p->spec, 0);
          for (size_t i = 0; i < p->gs_paths[leaf].size(); ++i) {
            const int m = p->gs_paths[leaf][i];
            macs = add_or_throw(macs, mul_or_throw(p->spec.K[m], c));
            c = scale_exact(c, p->spec.K[m], p->spec.L[m]);
            peak = std::max(peak, (i == 0 ? 1 : 2) + 1);  // hooi.hpp:213-214
          }
        }
        p->model.tree_macs = macs;
        p->model.peak_live = peak;
      }

      // one intermediate buffer per depth
      std::vector<int> depth(p->tree.size(), 0);
      for (int id = 1; id < p->tree.size(); ++id) {
        depth[id] = depth[p->tree.parent[id]] + (p->tree.internal(id) ? 1 : 0);
        if (!p->tree.internal(id)) continue;
        const size_t d = depth[id] - 1;
        if (p->depth_cap.size() <= d) p->depth_cap.resize(d + 1, 0);
        p->depth_cap[d] = std::max(p->depth_cap[d], static_cast<size_t>(cards.out[id]));
      }
      p->depth_buf.assign(p->depth_cap.size(), nullptr);
      for (size_t d = 0; d < p->depth_cap.size(); ++d) p->depth_buf[d] = device_alloc(p->depth_cap[d]);
      p->node_cap.assign(p->tree.size(), 0);
      for (int id = 1; id < p->tree.size(); ++id)
        if (p->tree.internal(id)) p->node_cap[id] = static_cast<size_t>(cards.out[id]);

      // core chain in its cheapest order; ping-pong buffers hold its largest partial product
      {
        const int mode = carry_first_mode().load(std::memory_order_relaxed);
        p->carry_first = p->sweep_kind == TP_SWEEP_JACOBI &&
                         (mode == 1 || (mode == 2 && 2.0 * static_cast<double>(cost.total_macs) < 5e10));
      }
      plan_choose_carry(p);
      if (p->carry_nodes.empty()) {
        p->core_order = cheapest_chain_order(p->spec, p->leaf_rank, &p->core_macs_executed);
      } else {
        p->core_order.clear();
        p->core_macs_executed = 0;
        u64 at = partial_cardinality(p->spec, 0);
        for (int id : p->carry_nodes) {
          const int m = p->tree.mode[id];
          p->core_order.push_back(m);
          p->core_macs_executed = add_or_throw(p->core_macs_executed, mul_or_throw(p->spec.K[m], at));
          at = scale_exact(at, p->spec.K[m], p->spec.L[m]);
          p->carry_buf.push_back(device_alloc(static_cast<size_t>(cards.out[id])));
        }
        p->core_order.push_back(p->carry_leaf_mode);
        p->core_macs_executed =
            add_or_throw(p->core_macs_executed, mul_or_throw(p->spec.K[p->carry_leaf_mode], at));
      }
      card = partial_cardinality(p->spec, 0);
      for (int i = 0; i + 1 < n_modes; ++i) {
        const int m = p->core_order[i];
        card = scale_exact(card, p->spec.K[m], p->spec.L[m]);
        p->core_tmp_cap = std::max(p->core_tmp_cap, static_cast<size_t>(card));
      }
      p->core = device_alloc(p->core_size);
      if (n_modes > 1) p->core_tmp[0] = device_alloc(p->core_tmp_cap);
      if (n_modes > 2) p->core_tmp[1] = device_alloc(p->core_tmp_cap);

      p->cur.assign(n_modes, nullptr);
      p->fresh.assign(n_modes, nullptr);
      p->frag.assign(n_modes, nullptr);
      p->frag_layout.resize(n_modes);
      long long max_rows = 0;
      for (int m = 0; m < n_modes; ++m) {
        const size_t elems = static_cast<size_t>(p->spec.L[m] * p->spec.K[m]);
        p->cur[m] = device_alloc(elems);
        p->fresh[m] = device_alloc(elems);
        TPB_CUDA(cudaMemsetAsync(p->cur[m], 0, elems * sizeof(double), ctx->stream));
        p->frag_layout[m] = ttm_fragment_layout(static_cast<long long>(p->spec.K[m]), static_cast<long long>(p->spec.L[m]));
        p->frag[m] = device_alloc(p->frag_layout[m].doubles);
        max_rows = std::max(max_rows, static_cast<long long>(p->spec.L[m]));
      }
      // Gram split workspace of each mode's leaf
      std::vector<size_t> leaf_ws(n_modes, 0);
      for (int id = 0; id < p->tree.size(); ++id) {
        if (!p->tree.leaf(id)) continue;
        const std::vector<u64> ext = node_extents(p->tree, p->spec, id);
        const int m = p->tree.mode[id];
        long long outer = 1, inner = 1;
        for (int i = 0; i < m; ++i) outer *= static_cast<long long>(ext[i]);
        for (int i = m + 1; i < n_modes; ++i) inner *= static_cast<long long>(ext[i]);
        leaf_ws[m] = std::max(leaf_ws[m],
                              gram_layout(outer, static_cast<long long>(ext[m]), inner, ctx->sm_count).workspace_doubles);
      }
      (void)max_rows;
      p->leaf.resize(n_modes);
      p->gram_ready.assign(n_modes, nullptr);
      p->factor_ready.assign(n_modes, nullptr);
      for (int m = 0; m < n_modes; ++m) {
        leaf_scratch_reserve(ctx, p->leaf[m], static_cast<long long>(p->spec.L[m]), leaf_ws[m]);
        TPB_CUDA(cudaEventCreateWithFlags(&p->gram_ready[m], cudaEventDisableTiming));
        TPB_CUDA(cudaEventCreateWithFlags(&p->factor_ready[m], cudaEventDisableTiming));
      }
      TPB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p->host_status), 64 * static_cast<size_t>(n_modes),
                             cudaHostAllocDefault));
      p->host_diag = reinterpret_cast<double*>(p->host_status + 8 * n_modes);
      std::memset(p->host_status, 0, 64 * static_cast<size_t>(n_modes));
      TPB_CUDA(cudaMalloc(&p->dev_status, 64 * static_cast<size_t>(n_modes)));
      TPB_CUDA(cudaMemset(p->dev_status, 0, 64 * static_cast<size_t>(n_modes)));
      TPB_CUDA(cudaEventCreate(&p->graph_begin));
      TPB_CUDA(cudaEventCreate(&p->graph_end));
      // below ~2e10 flops a sweep's kernels take a millisecond or two in total and ~100 host launches pace it
      p->short_sweep = 2.0 * (static_cast<double>(cost.total_macs) + static_cast<double>(p->core_macs_executed)) < 5e10;
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      tp_plan_destroy(ctx, p);
      throw;
    }
    *out = p;
  });
}

int tp_plan_destroy(tp_ctx* ctx, tp_plan* p) {
  return guarded([&] {
    if (!p) return;
    if (ctx) {
      cudaSetDevice(ctx->device);
      cudaStreamSynchronize(ctx->stream);
    }
    for (double* d : p->cur) cudaFree(d);
    for (double* d : p->fresh) cudaFree(d);
    for (double* d : p->frag) cudaFree(d);
    for (double* d : p->depth_buf) cudaFree(d);
    for (double* d : p->node_buf) cudaFree(d);
    for (cudaStream_t st : p->branch) cudaStreamDestroy(st);
    for (cudaEvent_t e : p->fork_events) cudaEventDestroy(e);
    for (double* d : p->carry_buf) cudaFree(d);
    for (double* d : p->arrival_slots) cudaFree(d);
    for (double* d : p->arrival_frag) cudaFree(d);
    cudaFree(p->core);
    cudaFree(p->core_tmp[0]);
    cudaFree(p->core_tmp[1]);
    for (LeafScratch& slot : p->leaf) slot.release();
    for (cudaEvent_t e : p->gram_ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->factor_ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->events)
      if (e) cudaEventDestroy(e);
    if (p->sweep_graph) cudaGraphExecDestroy(p->sweep_graph);
    if (p->graph_begin) cudaEventDestroy(p->graph_begin);
    if (p->graph_end) cudaEventDestroy(p->graph_end);
    if (p->host_status) cudaFreeHost(p->host_status);
    cudaFree(p->dev_status);
    delete p;
  });
}

int tp_plan_set_factors(tp_ctx* ctx, tp_plan* p, const double* const* factors) {
  return guarded([&] {
    bind(ctx);
    if (!p || !factors) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    for (int m = 0; m < p->n; ++m) {
      if (!factors[m]) raise(TP_ERR_SHAPE_MISMATCH, "factor count differs from mode count");
      TPB_CUDA(cudaMemcpyAsync(p->cur[m], factors[m], sizeof(double) * p->spec.L[m] * p->spec.K[m],
                               cudaMemcpyHostToDevice, ctx->stream));
    }
    p->carry_valid = false;
    p->factors_from_caller = true;
    p->frags_match_cur = false;
    p->warm_sweeps = 0;
    for (LeafScratch& slot : p->leaf) slot.last_ritz = nullptr;  // the caller's factors are the start, not ours
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tp_plan_get_factors(tp_ctx* ctx, tp_plan* p, double* const* factors_out) {
  return guarded([&] {
    bind(ctx);
    if (!p || !factors_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    for (int m = 0; m < p->n; ++m)
      TPB_CUDA(cudaMemcpyAsync(factors_out[m], p->cur[m], sizeof(double) * p->spec.L[m] * p->spec.K[m],
                               cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tp_plan_get_core(tp_ctx* ctx, tp_plan* p, double* core_out) {
  return guarded([&] {
    bind(ctx);
    if (!p || !core_out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    TPB_CUDA(cudaMemcpyAsync(core_out, p->core, sizeof(double) * p->core_size, cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tp_plan_core_norm(tp_ctx* ctx, tp_plan* p, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!p || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    *out = std::sqrt(sum_squares(ctx, p->core, p->core_size));
  });
}

int tp_plan_compute_core(tp_ctx* ctx, tp_plan* p, const tp_tensor* t) {
  return guarded([&] {
    bind(ctx);
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    check_tensor_matches(p, t);
    p->events_used = 0;
    p->event_phase.clear();
    p->event_node.clear();
    p->carry_valid = false;
    plan_core(ctx, p, t->data, p->cur);
    plan_mark_carried(p, t);
    plan_collect_timing(ctx, p);
  });
}

}  // extern "C"

namespace tpb {
namespace {

// The launch sequence of one Jacobi sweep, everything up to the host's look at the status: start-of-sweep factors to
// fragment order, the tree walk (leaf solves forked onto the side streams), the core chain with the new factors
// (joins the side streams), the status read-back, and the new factors copied over the current ones (the buffers
// never swap, so the sequence is the same every sweep and can be recorded).
void jacobi_sequence(tp_ctx* ctx, tp_plan* p, const tp_tensor* t) {
  std::vector<size_t> dims(p->spec.L.begin(), p->spec.L.end());
  if (!p->frags_match_cur) {
    Span s(ctx, p, kTree);  // start-of-sweep factors -> fragment order, once per mode
    for (int m = 0; m < p->n; ++m) plan_refresh_fragments(ctx, p, m, p->cur[m]);
    s.close();
  }
  p->frags_match_cur = false;
  p->leaves_in_flight = 0;
  p->pending.clear();
  p->one_launch_leaves = 0;
  for (int m = 0; m < p->n; ++m) {
    const long long rows = static_cast<long long>(p->spec.L[m]);
    const int k = static_cast<int>(p->spec.K[m]);
    if (p->fast_evd && p->leaf[m].use_fused && p->leaf[m].failures < 2 &&
        subspace_eligible(rows, k, plan_leaf_columns(p, m)) && leaf_solve_fused_eligible(rows, k, k + kSubspaceOversample))
      ++p->one_launch_leaves;
  }
  plan_begin_walk(p);
  if (p->arrival && p->arrival->row_end.size() > 1 && p->n > 1)
    jacobi_walk_streamed_root(ctx, p, t->data, dims);
  else
    jacobi_walk(ctx, p, 0, t->data, dims, 0);
  plan_join_branches(ctx, p);
  plan_core(ctx, p, t->data, p->fresh, p->overlap_evd);  // waits for each new factor just before using it
  // one launch copies the new factors over the current ones and gathers every leaf's status words, one copy brings
  // them to the host (instead of a copy per word and per factor: ~6 graph nodes per mode at the end of every sweep)
  FinishSweepArgs fin;
  fin.n_modes = p->n;
  for (int m = 0; m < p->n; ++m) {
    const LeafScratch& s = p->leaf[m];
    fin.cur[m] = p->cur[m];
    fin.fresh[m] = p->fresh[m];
    fin.elems[m] = static_cast<size_t>(p->spec.L[m] * p->spec.K[m]);
    fin.verdict[m] = s.fast_used ? s.verdict : nullptr;
    fin.diag[m] = s.fast_used ? s.diag : nullptr;
    fin.flag[m] = s.flag;
    fin.info[m] = s.info;
  }
  fin.status_ints = static_cast<int*>(p->dev_status);
  fin.status_doubles = reinterpret_cast<double*>(static_cast<int*>(p->dev_status) + 8 * p->n);
  TPB_CUDA(launch_finish_sweep(ctx->stream, fin));
  ctx->own_kernels += 1;
  TPB_CUDA(cudaMemcpyAsync(p->host_status, p->dev_status, 64 * static_cast<size_t>(p->n), cudaMemcpyDeviceToHost,
                           ctx->stream));
  p->frags_match_cur = true;  // plan_core prepared every mode's fragments from fresh[m], now also cur[m]
}

// May this sweep run as (or be recorded into) the whole-sweep graph?
bool sweep_graph_usable(const tp_ctx* ctx, const tp_plan* p, const tp_tensor* t) {
  (void)ctx;
  if (p->sweep_graph_mode == 0 || (p->sweep_graph_mode == 2 && !p->short_sweep)) return false;
  if (p->sweep_kind != TP_SWEEP_JACOBI || p->arrival || !p->overlap_evd || !p->fast_evd) return false;
  if (p->factors_from_caller || p->warm_sweeps < 1 || p->fast_rejected != 0 || t->pointer_escaped) return false;
  if (p->carry_enabled && !p->carry_nodes.empty() && !p->carry_live) return false;
  // The second sweep of a run is already the steady-state launch sequence when every leaf takes the one-launch solve
  // AND starts it from the previous sweep's Ritz vectors (the first sweep's solves were certified); otherwise the
  // sequence settles one sweep later (a leaf's own recording, the start block of a leaf that fell back).
  const bool second_sweep = p->warm_sweeps < 2;
  for (int m = 0; m < p->n; ++m) {
    const LeafScratch& s = p->leaf[m];
    const long long rows = static_cast<long long>(p->spec.L[m]);
    const int k = static_cast<int>(p->spec.K[m]);
    if (s.failures >= 2 || !subspace_eligible(rows, k, plan_leaf_columns(p, m))) return false;  // full solve: cuSOLVER
    const int b = k + kSubspaceOversample;
    if (s.use_fused && leaf_solve_fused_eligible(rows, k, b)) {
      if (second_sweep && !s.last_ritz) return false;
      continue;
    }
    if (second_sweep) return false;
    if (static_cast<size_t>(b) > small_evd_max_block()) return false;        // cuSOLVER steps inside the iteration
    if (s.use_graph && s.graph_state != 2 && s.graph_state != -1) return false;  // its own recording comes first
    if (!s.last_ritz) return false;
  }
  return true;
}

void drop_sweep_graph(tp_plan* p) {
  if (p->sweep_graph) cudaGraphExecDestroy(p->sweep_graph);
  p->sweep_graph = nullptr;
  p->sweep_graph_tensor = nullptr;
}

}  // namespace
}  // namespace tpb

extern "C" {

int tp_plan_sweep(tp_ctx* ctx, tp_plan* p, const tp_tensor* t, tp_sweep_stats* stats) {
  return guarded([&] {
    bind(ctx);
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    check_tensor_matches(p, t);
    if (stats) *stats = tp_sweep_stats{};  // hooi.hpp:198
    p->events_used = 0;
    p->event_phase.clear();
    p->event_node.clear();
    std::vector<size_t> dims(p->spec.L.begin(), p->spec.L.end());
    int flag = 0;
    if (p->sweep_kind == TP_SWEEP_JACOBI) {
      p->carry_live = p->carry_enabled && p->carry_valid && p->carry_tensor == t && p->carry_stamp == t->stamp &&
                      !t->pointer_escaped;
      p->carry_valid = false;  // the chain at the end of this sweep overwrites the carried products
      bool replayed = false;
      if (sweep_graph_usable(ctx, p, t)) {
        if (p->sweep_graph && (p->sweep_graph_tensor != t->data || p->sweep_graph_stamp != t->stamp)) drop_sweep_graph(p);
        if (!p->sweep_graph) {
          // record: the same code path as an eager sweep, with the main stream (and, through its event waits, the
          // side streams) in capture mode
          cudaGraph_t recorded = nullptr;
          bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
          if (ok) {
            p->capturing = true;
            const u64 own0 = ctx->own_kernels, lib0 = ctx->library_calls;
            try {
              jacobi_sequence(ctx, p, t);
            } catch (const Failure&) {
              ok = false;
            }
            p->capturing = false;
            ctx->own_kernels = own0;
            ctx->library_calls = lib0;
            if (cudaStreamEndCapture(ctx->stream, &recorded) != cudaSuccess) ok = false;
            if (ok && ctx->dump_sweep_graph && recorded)
              cudaGraphDebugDotPrint(recorded, "/tmp/tpb_sweep_graph.dot", 0);  // TP_CTX_OPT_DUMP_SWEEP_GRAPH
            if (ok && cudaGraphInstantiate(&p->sweep_graph, recorded, 0) != cudaSuccess) ok = false;
            if (recorded) cudaGraphDestroy(recorded);
          }
          if (ok) {
            p->sweep_graph_tensor = t->data;
            p->sweep_graph_stamp = t->stamp;
            p->sweep_graph_fast.assign(p->n, 0);
            for (int m = 0; m < p->n; ++m) p->sweep_graph_fast[m] = p->leaf[m].fast_used ? 1 : 0;
          } else {
            const cudaError_t why = cudaGetLastError();  // recording is an optimisation: carry on with plain launches
            if (ctx->trace_evd)
              std::fprintf(stderr, "[tpb graph] recording the sweep failed (%s); plain launches from here on\n",
                           cudaGetErrorString(why));
            p->sweep_graph = nullptr;
            p->sweep_graph_mode = 0;
            for (int a = 0; a < tp_ctx::kAux; ++a) cudaStreamSynchronize(ctx->aux[a]);
          }
        }
        if (p->sweep_graph) {
          for (int m = 0; m < p->n; ++m) p->leaf[m].fast_used = p->sweep_graph_fast[m] != 0;
          TPB_CUDA(cudaEventRecord(p->graph_begin, ctx->stream));
          TPB_CUDA(cudaGraphLaunch(p->sweep_graph, ctx->stream));
          TPB_CUDA(cudaEventRecord(p->graph_end, ctx->stream));
          ctx->own_kernels += p->sweep_graph_kernels;
          ctx->library_calls += p->sweep_graph_library_calls;
          replayed = true;
        }
      } else if (p->sweep_graph) {
        drop_sweep_graph(p);
      }
      if (!replayed) {
        const u64 own0 = ctx->own_kernels, lib0 = ctx->library_calls;
        jacobi_sequence(ctx, p, t);
        p->sweep_graph_kernels = ctx->own_kernels - own0;   // what a replay of this sequence launches
        p->sweep_graph_library_calls = ctx->library_calls - lib0;
      }
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
      // leaves solved by subspace iteration are accepted only with their certificate; a rejected leaf is redone
      // (more rounds, else the full eigen-solve on its intact Gram matrix), and the core with it
      const std::vector<int> rejected = evaluate_fast_leaves(ctx, p);
      if (p->leaf_steps_changed) {
        drop_sweep_graph(p);
        p->leaf_steps_changed = false;
      }
      for (int m = 0; m < p->n; ++m) {
        if (p->host_status[8 * m + 5] != 0) raise(TP_ERR_TOO_LARGE, "eigensolver did not converge");  // hooi.hpp:56-57
        flag |= p->host_status[8 * m + 4];
      }
      p->fast_rejected = 0;
      if (!rejected.empty()) {
        for (int m : rejected) p->fast_rejected += redo_rejected_leaf(ctx, p, m, p->fresh[m]) ? 1 : 0;
        plan_core(ctx, p, t->data, p->fresh);
        for (int m = 0; m < p->n; ++m)
          TPB_CUDA(cudaMemcpyAsync(p->cur[m], p->fresh[m], sizeof(double) * p->spec.L[m] * p->spec.K[m],
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        // degenerate flags: the accepted leaves' from the read-back, the redone leaves' from their new solves
        flag = 0;
        for (int m = 0; m < p->n; ++m)
          if (std::find(rejected.begin(), rejected.end(), m) == rejected.end()) flag |= p->host_status[8 * m + 4];
        flag |= read_and_clear_flags(ctx, p->leaf);
      }
      p->factors_from_caller = false;
      ++p->warm_sweeps;
      p->last_sweep_replayed = replayed;
      plan_mark_carried(p, t);
      if (replayed) {
        TPB_CUDA(cudaStreamSynchronize(ctx->stream));
        tp_sweep_timing tm{};
        TPB_CUDA(cudaEventElapsedTime(&tm.total_ms, p->graph_begin, p->graph_end));
        p->timing = tm;
        p->node_ms.assign(p->tree.size(), 0.f);
        p->node_evd_ms.assign(p->tree.size(), 0.f);
      } else {
        plan_collect_timing(ctx, p);
      }
    } else {
      p->frags_match_cur = false;
      {
        Span s(ctx, p, kTree);
        for (int m = 0; m < p->n; ++m) plan_refresh_fragments(ctx, p, m, p->cur[m]);
        s.close();
      }
      if (p->arrival)  // a by-value call is still uploading: the chains read the whole tensor
        for (size_t c = 0; c < p->arrival->row_end.size(); ++c) {
          p->arrival->issue(static_cast<int>(c));
          TPB_CUDA(cudaStreamWaitEvent(ctx->stream, p->arrival->ready[c], 0));
        }
      p->carry_live = p->carry_enabled && p->carry_valid && p->carry_tensor == t && p->carry_stamp == t->stamp &&
                      !p->carry_nodes.empty() && !t->pointer_escaped;
      p->carry_valid = false;
      p->fast_rejected = 0;
      for (int leaf = 0; leaf < p->n; ++leaf) {  // hooi.hpp:206-224
        const double* at = t->data;
        std::vector<size_t> d = dims;
        size_t step = 0;
        if (leaf == 0 && p->carry_live) {
          // this chain was computed by the previous sweep's core chain (same tensor, same F_1 .. F_{N-1})
          at = p->carry_buf.back();
          for (int m : p->gs_paths[leaf]) d[m] = static_cast<size_t>(p->spec.K[m]);
        } else {
          for (int m : p->gs_paths[leaf]) {
            Span s(ctx, p, kTree);
            double* out = p->depth_buf[step];
            plan_ttm(ctx, p, at, d, m, out);
            s.close();
            d[m] = static_cast<size_t>(p->spec.K[m]);
            at = out;
            ++step;
          }
        }
        plan_leaf(ctx, p, at, d, leaf, p->fresh[leaf], -1, false);
        // the next chain multiplies by this factor: a certified top-k solve is checked now, not at the end
        const std::vector<int> rejected = verify_fast_leaves(ctx, p);
        if (!rejected.empty()) p->fast_rejected += redo_rejected_leaf(ctx, p, leaf, p->fresh[leaf]) ? 1 : 0;
        std::swap(p->cur[leaf], p->fresh[leaf]);  // later chains see the fresh factor
        Span s(ctx, p, kTree);
        plan_refresh_fragments(ctx, p, leaf, p->cur[leaf]);
        s.close();
      }
      plan_core(ctx, p, t->data, p->cur);
      p->factors_from_caller = false;
      plan_mark_carried(p, t);
      flag = read_and_clear_flags(ctx, p->leaf);
      plan_collect_timing(ctx, p);
    }
    if (stats) {
      *stats = p->model;
      stats->degenerate = flag;
    }
  });
}

int tp_plan_set_option(tp_ctx* ctx, tp_plan* p, int option, int value) {
  return guarded([&] {
    (void)ctx;
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    tpb::drop_sweep_graph(p);  // every option changes the recorded launch sequence
    if (option == TP_OPT_OVERLAP_EVD)
      p->overlap_evd = value != 0;
    else if (option == TP_OPT_FAST_EVD)
      p->fast_evd = value != 0;
    else if (option == TP_OPT_CARRY_PATH) {
      p->carry_enabled = value != 0;
      p->carry_valid = false;
    } else if (option == TP_OPT_SPARE_SMS) {
      p->spare_sms = std::max(0, value);
    } else if (option == TP_OPT_SPARE_SMS_SHORT) {
      p->spare_sms_short = std::max(0, value);
    } else if (option == TP_OPT_SWEEP_GRAPH) {
      if (value < 0 || value > 2) raise(TP_ERR_BAD_ARGUMENT, "sweep graph mode is 0 (off), 1 (on) or 2 (auto)");
      p->sweep_graph_mode = value;
    } else if (option == TP_OPT_FORK_SUBTREES) {
      if (value < 0 || value > 2) raise(TP_ERR_BAD_ARGUMENT, "fork mode is 0 (off), 1 (on) or 2 (auto)");
      if (p->fork_mode != value) drop_sweep_graph(p);
      p->fork_mode = value;
    } else if (option == TP_OPT_LEAF_GRAPH) {
      for (LeafScratch& slot : p->leaf) {
        slot.use_graph = value != 0;
        forget_recorded_solve(slot);
      }
    } else if (option == TP_OPT_FUSED_LEAF_SOLVE) {
      for (LeafScratch& slot : p->leaf) {
        slot.use_fused = value != 0;
        forget_recorded_solve(slot);
      }
    } else {
      raise(TP_ERR_BAD_ARGUMENT, "unknown plan option");
    }
  });
}

int tp_plan_last_evd_info(tp_ctx* ctx, tp_plan* p, int* fast_eligible, int* rejected) {
  return guarded([&] {
    (void)ctx;
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    int eligible = 0;
    for (int m = 0; m < p->n; ++m)
      if (p->fast_evd && p->leaf[m].failures < 2 &&
          subspace_eligible(static_cast<long long>(p->spec.L[m]), static_cast<int>(p->spec.K[m]),
                            plan_leaf_columns(p, m)))
        ++eligible;
    if (fast_eligible) *fast_eligible = eligible;
    if (rejected) *rejected = p->fast_rejected;
  });
}

int tp_plan_last_sweep_info(tp_ctx* ctx, tp_plan* p, int* replayed_graph, int* one_launch_leaves) {
  return guarded([&] {
    (void)ctx;
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    if (replayed_graph) *replayed_graph = p->last_sweep_replayed ? 1 : 0;
    int fused = 0;
    for (int m = 0; m < p->n; ++m) {
      const LeafScratch& s = p->leaf[m];
      const long long rows = static_cast<long long>(p->spec.L[m]);
      const int k = static_cast<int>(p->spec.K[m]);
      if (p->fast_evd && s.use_fused && s.failures < 2 && subspace_eligible(rows, k, plan_leaf_columns(p, m)) &&
          leaf_solve_fused_eligible(rows, k, k + kSubspaceOversample))
        ++fused;
    }
    if (one_launch_leaves) *one_launch_leaves = fused;
  });
}

int tp_plan_node_timing(tp_ctx* ctx, tp_plan* p, int n_nodes, float* node_ms, float* evd_ms) {
  return guarded([&] {
    (void)ctx;
    if (!p) raise(TP_ERR_BAD_ARGUMENT, "null plan");
    if (n_nodes != p->tree.size()) raise(TP_ERR_SHAPE_MISMATCH, "node count differs from the plan's tree");
    for (int i = 0; i < n_nodes; ++i) {
      if (node_ms) node_ms[i] = i < static_cast<int>(p->node_ms.size()) ? p->node_ms[i] : 0.f;
      if (evd_ms) evd_ms[i] = i < static_cast<int>(p->node_evd_ms.size()) ? p->node_evd_ms[i] : 0.f;
    }
  });
}

int tp_tensor_axpby(tp_ctx* ctx, tp_tensor* y, double beta, double alpha, const tp_tensor* x) {
  return guarded([&] {
    bind(ctx);
    if (!y || !x) raise(TP_ERR_BAD_ARGUMENT, "null tensor");
    if (y->dims != x->dims) raise(TP_ERR_SHAPE_MISMATCH, "tensor shapes differ");
    TPB_CUDA(launch_axpby(ctx->stream, y->data, beta, alpha, x->data, y->size));
    y->stamp = next_tensor_stamp();
    ctx->own_kernels += 1;
  });
}

int tp_plan_last_timing(tp_ctx* ctx, tp_plan* p, tp_sweep_timing* out) {
  return guarded([&] {
    (void)ctx;
    if (!p || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    *out = p->timing;
  });
}

// core x_0 F_0 ... x_{N-1} F_{N-1} on the device, then ||t - z|| / ||t||  (hooi.hpp:232-245)
static double expansion_error(tp_ctx* ctx, const tp_tensor* t, const std::vector<size_t>& core_dims,
                              const double* core_dev, const std::vector<const double*>& factors_dev) {
  const double norm = std::sqrt(sum_squares(ctx, t->data, t->size));
  if (norm == 0.0) raise(TP_ERR_ZERO_TENSOR, "relative error undefined at zero");
  const int n = static_cast<int>(core_dims.size());
  std::vector<size_t> dims = core_dims;
  const double* src = core_dev;
  double* owned = nullptr;
  try {
    for (int m = 0; m < n; ++m) {
      const size_t rows = t->dims[m], cols = core_dims[m];
      std::vector<size_t> out_dims = dims;
      out_dims[m] = rows;
      size_t out_size = 1;
      for (size_t d : out_dims) out_size *= d;
      double* dst = device_alloc(out_size);
      // ttm(z, F_m, m): matrix rows x cols with F column-major -> M(r, c) = F[c * rows + r]
      try {
        run_ttm(ctx, src, dims, m, factors_dev[m], 1, static_cast<long long>(rows), static_cast<long long>(rows),
                nullptr, dst);
        TPB_CUDA(cudaStreamSynchronize(ctx->stream));
      } catch (...) {
        cudaFree(dst);
        throw;
      }
      (void)cols;
      cudaFree(owned);
      owned = dst;
      src = dst;
      dims = out_dims;
    }
    if (dims != t->dims) raise(TP_ERR_SHAPE_MISMATCH, "reconstruction shape differs");
    const double diff = diff_sum_squares(ctx, t->data, src, t->size);
    cudaFree(owned);
    return std::sqrt(diff) / norm;
  } catch (...) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(owned);
    throw;
  }
}

int tp_plan_reconstruction_error(tp_ctx* ctx, tp_plan* p, const tp_tensor* t, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!p || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    if (!t) raise(TP_ERR_BAD_ARGUMENT, "null tensor");
    check_tensor_matches(p, t);
    std::vector<size_t> core_dims(p->spec.K.begin(), p->spec.K.end());
    std::vector<const double*> factors(p->cur.begin(), p->cur.end());
    *out = expansion_error(ctx, t, core_dims, p->core, factors);
  });
}

int tp_plan_fit_from_norms(tp_ctx* ctx, tp_plan* p, const tp_tensor* t, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!p || !out || !t) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    check_tensor_matches(p, t);
    const double t2 = sum_squares(ctx, t->data, t->size);
    if (t2 == 0.0) raise(TP_ERR_ZERO_TENSOR, "relative error undefined at zero");
    const double g2 = sum_squares(ctx, p->core, p->core_size);
    *out = std::sqrt(std::max(t2 - g2, 0.0) / t2);
  });
}

int tp_reconstruction_error(tp_ctx* ctx, const tp_tensor* t, const size_t* core_dims, const double* core,
                            const double* const* factors, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!t || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    const double norm2 = sum_squares(ctx, t->data, t->size);
    if (norm2 == 0.0) raise(TP_ERR_ZERO_TENSOR, "relative error undefined at zero");  // hooi.hpp:233-234 comes first
    if (!core_dims || !core || !factors) raise(TP_ERR_SHAPE_MISMATCH, "reconstruction shape differs");
    const int n = static_cast<int>(t->dims.size());
    std::vector<size_t> cd(core_dims, core_dims + n);
    const size_t core_size = checked_size(n, core_dims);
    std::vector<double*> owned;
    auto cleanup = [&] {
      cudaStreamSynchronize(ctx->stream);
      for (double* d : owned) cudaFree(d);
    };
    try {
      double* core_dev = device_alloc(core_size);
      owned.push_back(core_dev);
      TPB_CUDA(cudaMemcpyAsync(core_dev, core, core_size * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      std::vector<const double*> f(n);
      for (int m = 0; m < n; ++m) {
        if (!factors[m]) raise(TP_ERR_SHAPE_MISMATCH, "reconstruction shape differs");
        double* d = device_alloc(t->dims[m] * cd[m]);
        owned.push_back(d);
        TPB_CUDA(cudaMemcpyAsync(d, factors[m], t->dims[m] * cd[m] * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        f[m] = d;
      }
      *out = expansion_error(ctx, t, cd, core_dev, f);
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

// ------------------------------------------------------------- device-pointer building blocks
static LeafScratch& dev_scratch(tp_ctx* ctx) {
  if (!ctx->dev_scratch) ctx->dev_scratch = new LeafScratch;
  return *static_cast<LeafScratch*>(ctx->dev_scratch);
}

// SMs a product of the tp_dev_* entry points leaves to asynchronous leaf solves in flight (as plan_ttm does).
static int dev_sm_budget(const tp_ctx* ctx, double flops) {
  bool busy = false;
  for (const tp_ctx::Lane& lane : ctx->lanes) busy = busy || lane.busy;
  if (!busy) return ctx->sm_count;
  return std::max(1, ctx->sm_count - (flops < 2e11 ? 16 : 2));
}

int tp_dev_ttm_partial(tp_ctx* ctx, const double* x, int n_modes, const size_t* dims, int mode, const double* factor,
                       size_t L_full, size_t l0, size_t K, int n_dest, const size_t* dest_cuts, double* z) {
  return guarded([&] {
    bind(ctx);
    if (!x || !factor || !z) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    checked_size(n_modes, dims);
    std::vector<size_t> d(dims, dims + n_modes);
    long long outer, inner;
    mode_extents(d, mode, outer, inner);
    const long long len = static_cast<long long>(d[mode]);
    if (l0 + d[mode] > L_full) raise(TP_ERR_SHAPE_MISMATCH, "factor rows do not cover the block's mode slice");
    if (K == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
    if (n_dest < 1 || n_dest > kMaxTtmDest) raise(TP_ERR_BAD_ARGUMENT, "between 1 and 16 destinations");
    std::vector<long long> cuts(n_dest + 1);
    for (int i = 0; i <= n_dest; ++i) cuts[i] = dest_cuts ? static_cast<long long>(dest_cuts[i]) : (i == 0 ? 0 : static_cast<long long>(K));
    if (cuts[0] != 0 || cuts[n_dest] != static_cast<long long>(K)) raise(TP_ERR_BAD_ARGUMENT, "destination cuts must span [0, K]");
    for (int i = 0; i < n_dest; ++i)
      if (cuts[i + 1] < cuts[i]) raise(TP_ERR_BAD_ARGUMENT, "destination cuts must ascend");
    const TtmFragmentLayout f = ttm_fragment_layout(static_cast<long long>(K), len);
    double* frag = ensure_frag_scratch(ctx, f.doubles);
    // M = F^T restricted to rows l0.. of F: M(k, l) = factor[k * L_full + l0 + l]
    TPB_CUDA(prep_factor_fragments(ctx->stream, factor + l0, static_cast<long long>(L_full), 1,
                                   static_cast<long long>(K), len, f, frag));
    TPB_CUDA(launch_ttm(ctx->stream, x, outer, len, inner, frag, f, static_cast<long long>(K), z,
                        dev_sm_budget(ctx, 2.0 * static_cast<double>(K) * outer * len * inner), n_dest, cuts.data()));
    ctx->own_kernels += 2;
  });
}

int tp_dev_ttm_scatter(tp_ctx* ctx, const double* x, int n_modes, const size_t* dims, int mode, const double* factor,
                       size_t L_full, size_t l0, size_t K, int n_dest, const size_t* dest_cuts,
                       double* const* dest_ptrs) {
  return guarded([&] {
    bind(ctx);
    if (!x || !factor || !dest_ptrs || !dest_cuts) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    checked_size(n_modes, dims);
    std::vector<size_t> d(dims, dims + n_modes);
    long long outer, inner;
    mode_extents(d, mode, outer, inner);
    const long long len = static_cast<long long>(d[mode]);
    if (l0 + d[mode] > L_full) raise(TP_ERR_SHAPE_MISMATCH, "factor rows do not cover the block's mode slice");
    if (K == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
    if (n_dest < 1 || n_dest > kMaxTtmDest) raise(TP_ERR_BAD_ARGUMENT, "between 1 and 16 destinations");
    std::vector<long long> cuts(n_dest + 1), offsets(n_dest, 0);
    for (int i = 0; i <= n_dest; ++i) cuts[i] = static_cast<long long>(dest_cuts[i]);
    if (cuts[0] != 0 || cuts[n_dest] != static_cast<long long>(K)) raise(TP_ERR_BAD_ARGUMENT, "destination cuts must span [0, K]");
    // the kernels address chunk d as z + dest_off[d]: anchor at the first non-empty chunk's buffer and express the
    // others (possibly peer-mapped memory) as element distances from it
    int anchor = -1;
    for (int i = 0; i < n_dest; ++i) {
      if (cuts[i + 1] < cuts[i]) raise(TP_ERR_BAD_ARGUMENT, "destination cuts must ascend");
      if (cuts[i + 1] == cuts[i]) continue;
      if (!dest_ptrs[i]) raise(TP_ERR_BAD_ARGUMENT, "null destination for a non-empty chunk");
      if (reinterpret_cast<uintptr_t>(dest_ptrs[i]) % sizeof(double)) raise(TP_ERR_BAD_ARGUMENT, "misaligned destination");
      if (anchor < 0) anchor = i;
    }
    if (anchor < 0) return;
    double* const z = dest_ptrs[anchor];
    for (int i = 0; i < n_dest; ++i)
      if (cuts[i + 1] > cuts[i])
        offsets[i] = static_cast<long long>((reinterpret_cast<intptr_t>(dest_ptrs[i]) - reinterpret_cast<intptr_t>(z)) /
                                            static_cast<intptr_t>(sizeof(double)));
    const TtmFragmentLayout f = ttm_fragment_layout(static_cast<long long>(K), len);
    double* frag = ensure_frag_scratch(ctx, f.doubles);
    TPB_CUDA(prep_factor_fragments(ctx->stream, factor + l0, static_cast<long long>(L_full), 1,
                                   static_cast<long long>(K), len, f, frag));
    TPB_CUDA(launch_ttm(ctx->stream, x, outer, len, inner, frag, f, static_cast<long long>(K), z,
                        dev_sm_budget(ctx, 2.0 * static_cast<double>(K) * outer * len * inner), n_dest, cuts.data(),
                        offsets.data()));
    ctx->own_kernels += 2;
  });
}

int tp_dev_reduce_slots(tp_ctx* ctx, double* out, const double* const* slots_host, int n_slots, size_t count) {
  return guarded([&] {
    bind(ctx);
    if (!out || !slots_host) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    if (n_slots < 1 || n_slots > kMaxReduceSlots) raise(TP_ERR_BAD_ARGUMENT, "between 1 and 16 slots");
    TPB_CUDA(launch_reduce_slots(ctx->stream, out, slots_host, n_slots, count));
    ctx->own_kernels += 1;
  });
}

int tp_dev_assemble_mode(tp_ctx* ctx, double* dst, size_t outer, size_t full_len, size_t inner, const double* src,
                         size_t l0, size_t count) {
  return guarded([&] {
    bind(ctx);
    if (!dst || !src) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    if (l0 + count > full_len) raise(TP_ERR_SHAPE_MISMATCH, "slice exceeds the mode extent");
    TPB_CUDA(launch_assemble_mode(ctx->stream, dst, static_cast<long long>(outer), static_cast<long long>(full_len),
                                  static_cast<long long>(inner), src, static_cast<long long>(l0),
                                  static_cast<long long>(count)));
    ctx->own_kernels += 1;
  });
}

int tp_dev_copy_box(tp_ctx* ctx, double* dst, const size_t* dst_dims, const size_t* dst_lo, const double* src,
                    const size_t* src_dims, const size_t* src_lo, const size_t* box, int n_modes) {
  return guarded([&] {
    bind(ctx);
    if (!dst || !src || !dst_dims || !dst_lo || !src_dims || !src_lo || !box) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    if (n_modes < 1 || n_modes > kMaxBoxModes) raise(TP_ERR_BAD_DIMS, "tensor needs 1..16 modes");
    long long dd[kMaxBoxModes], dl[kMaxBoxModes], sd[kMaxBoxModes], sl[kMaxBoxModes], bx[kMaxBoxModes];
    for (int m = 0; m < n_modes; ++m) {
      if (dst_lo[m] + box[m] > dst_dims[m] || src_lo[m] + box[m] > src_dims[m])
        raise(TP_ERR_SHAPE_MISMATCH, "box exceeds a tensor's extent", m);
      dd[m] = static_cast<long long>(dst_dims[m]);
      dl[m] = static_cast<long long>(dst_lo[m]);
      sd[m] = static_cast<long long>(src_dims[m]);
      sl[m] = static_cast<long long>(src_lo[m]);
      bx[m] = static_cast<long long>(box[m]);
    }
    TPB_CUDA(launch_copy_box(ctx->stream, dst, dd, dl, src, sd, sl, bx, n_modes));
    ctx->own_kernels += 1;
  });
}

int tp_dev_gram(tp_ctx* ctx, const double* y, size_t outer, size_t rows, size_t inner, double* gram) {
  return guarded([&] {
    bind(ctx);
    if (!y || !gram) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    if (rows == 0 || outer * inner == 0) raise(TP_ERR_SHAPE_MISMATCH, "empty matrix");
    if (rows > TP_MAX_GRAM_ROWS) raise(TP_ERR_TOO_LARGE, "unfolding has too many rows for the Gram route");
    const GramLayout g = gram_layout(static_cast<long long>(outer), static_cast<long long>(rows),
                                     static_cast<long long>(inner), ctx->sm_count);
    LeafScratch& s = dev_scratch(ctx);
    leaf_scratch_reserve(ctx, s, 1, g.workspace_doubles);
    TPB_CUDA(launch_gram(ctx->stream, y, static_cast<long long>(outer), static_cast<long long>(rows),
                         static_cast<long long>(inner), g, s.gram_ws, gram));
    ctx->own_kernels += 2;
  });
}

int tp_dev_leaf_solve(tp_ctx* ctx, double* gram, size_t rows, int k, double* factor, int* flag, int* info) {
  return guarded([&] {
    bind(ctx);
    if (!gram || !factor || !flag || !info) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_leaf_args(static_cast<long long>(rows), 1, k);
    LeafScratch& s = dev_scratch(ctx);
    leaf_scratch_reserve(ctx, s, static_cast<long long>(rows), 0);
    TPB_SOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(rows),
                                gram, static_cast<int>(rows), s.w, s.work, s.lwork, info));
    ctx->library_calls += 1;
    TPB_CUDA(launch_select_basis(ctx->stream, gram, s.w, static_cast<int>(rows), static_cast<int>(rows), k, factor,
                                 flag));
    ctx->own_kernels += 1;
  });
}

// Iteration buffers of a scratch that serves leaves of changing sizes (the tp_dev_* entry points).
static void reserve_iteration_buffers(tp_ctx* ctx, LeafScratch& s, long long rows, int k) {
  leaf_scratch_reserve(ctx, s, 1, 0);
  if (s.block != 0 && (s.block != k + kSubspaceOversample || rows > s.fast_rows)) {
    cudaFree(s.q); cudaFree(s.z); cudaFree(s.x); cudaFree(s.h); cudaFree(s.theta); cudaFree(s.small_work);
    cudaFree(s.verdict); cudaFree(s.chol); cudaFree(s.ritz);
    s.q = s.z = s.x = s.h = s.theta = s.small_work = s.chol = s.ritz = nullptr;
    s.verdict = nullptr;
    s.block = 0;
    forget_recorded_solve(s);
  }
  if (s.block == 0) {
    subspace_reserve(ctx, s, rows, k);
    s.fast_rows = rows;
  }
}

// Asynchronous pair: _begin queues the solve of `gram` on side stream `lane` (ordered after everything queued on the
// main stream so far) and returns; the main stream goes on with the tree.  _finish makes the main stream wait for
// it, reads the certificate of the top-k path and redoes the leaf with the full solve if it was missed.  Between
// the two calls gram, start, factor, flag and info must stay untouched.  One solve in flight per lane.
int tp_dev_leaf_solve_begin(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                            int* flag, int* info, int lane_index) {
  return tp_dev_leaf_solve_begin_ex(ctx, gram, rows, k, start, factor, flag, info, lane_index, 0);
}

int tp_dev_leaf_solve_begin_ex(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                               int* flag, int* info, int lane_index, unsigned flags) {
  return guarded([&] {
    bind(ctx);
    if (!gram || !factor || !flag || !info) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    if (lane_index < 0 || lane_index >= tp_ctx::kAux) raise(TP_ERR_BAD_ARGUMENT, "lane outside 0..3");
    check_leaf_args(static_cast<long long>(rows), 1, k);
    tp_ctx::Lane& lane = ctx->lanes[lane_index];
    if (lane.busy) raise(TP_ERR_BAD_ARGUMENT, "a solve is already in flight on this lane");
    if (!lane.scratch) {
      lane.scratch = new LeafScratch;
      TPB_CUDA(cudaEventCreateWithFlags(&lane.ready, cudaEventDisableTiming));
      TPB_CUDA(cudaEventCreateWithFlags(&lane.done, cudaEventDisableTiming));
    }
    LeafScratch& s = *static_cast<LeafScratch*>(lane.scratch);
    cudaStream_t side = ctx->aux[lane_index];
    lane.fast = start && subspace_eligible(static_cast<long long>(rows), k);
    if (lane.fast)
      reserve_iteration_buffers(ctx, s, static_cast<long long>(rows), k);
    else
      leaf_scratch_reserve(ctx, s, static_cast<long long>(rows), 0);
    TPB_CUDA(cudaEventRecord(lane.ready, ctx->stream));
    TPB_CUDA(cudaStreamWaitEvent(side, lane.ready, 0));
    if (lane.fast) {
      int* const saved_flag = s.flag;
      s.flag = flag;
      // by default the result is a function of the arguments only; with TP_LEAF_CONTINUE the lane's previous,
      // accepted solve of the same buffer and shape supplies the start block (its Ritz vectors), as a plan does
      lane.keep = (flags & TP_LEAF_CONTINUE) != 0;
      if (!(lane.keep && lane.accepted && lane.gram == gram && lane.rows == rows && lane.k == k)) s.last_ritz = nullptr;
      leaf_solve_subspace(ctx, s, gram, static_cast<long long>(rows), k, start, factor, lane_index);
      s.flag = saved_flag;
      s.fast_used = false;
    } else {
      TPB_SOLVER(cusolverDnDsyevd(ctx->aux_solver[lane_index], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  static_cast<int>(rows), gram, static_cast<int>(rows), s.w, s.work, s.lwork, info));
      ctx->library_calls += 1;
      TPB_CUDA(launch_select_basis(side, gram, s.w, static_cast<int>(rows), static_cast<int>(rows), k, factor, flag));
      ctx->own_kernels += 1;
    }
    TPB_CUDA(cudaEventRecord(lane.done, side));
    lane.busy = true;
    lane.gram = gram;
    lane.rows = rows;
    lane.k = k;
  });
}

int tp_dev_leaf_solve_reset(tp_ctx* ctx) {
  return guarded([&] {
    if (!ctx) raise(TP_ERR_BAD_ARGUMENT, "null context");
    for (tp_ctx::Lane& lane : ctx->lanes) {
      if (lane.busy) raise(TP_ERR_BAD_ARGUMENT, "a solve is still in flight");
      lane.accepted = false;
    }
  });
}

int tp_dev_leaf_solve_finish(tp_ctx* ctx, int lane_index, double* factor, int* flag, int* info, int* used_fast) {
  return guarded([&] {
    bind(ctx);
    if (lane_index < 0 || lane_index >= tp_ctx::kAux) raise(TP_ERR_BAD_ARGUMENT, "lane outside 0..3");
    if (!factor || !flag || !info) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    tp_ctx::Lane& lane = ctx->lanes[lane_index];
    if (!lane.busy) raise(TP_ERR_BAD_ARGUMENT, "no solve in flight on this lane");
    lane.busy = false;
    if (used_fast) *used_fast = 0;
    TPB_CUDA(cudaStreamWaitEvent(ctx->stream, lane.done, 0));
    if (!lane.fast) return;
    LeafScratch& s = *static_cast<LeafScratch*>(lane.scratch);
    int host[3] = {0, 0, 0};
    TPB_CUDA(cudaMemcpyAsync(&host[0], s.verdict, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaMemcpyAsync(&host[2], flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    // only the residual bound missed: iterate on from the Ritz vectors reached (as the plan does), main stream
    for (int round = 0; round < 3 && (host[0] & 1) != 0 && host[1] == 0 && host[2] == 0 && s.last_ritz; ++round) {
      int* const saved_flag = s.flag;
      s.flag = flag;
      leaf_solve_subspace(ctx, s, lane.gram, static_cast<long long>(lane.rows), lane.k, factor, factor, -1);
      s.flag = saved_flag;
      s.fast_used = false;
      TPB_CUDA(cudaMemcpyAsync(&host[0], s.verdict, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaMemcpyAsync(&host[2], flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    lane.accepted = host[0] == 0 && host[1] == 0 && host[2] == 0;
    if (!(lane.keep && lane.accepted)) s.last_ritz = nullptr;
    if (lane.accepted) {
      TPB_CUDA(cudaMemsetAsync(info, 0, sizeof(int), ctx->stream));
      if (used_fast) *used_fast = 1;
      return;
    }
    // certificate missed: the Gram matrix is intact, let the exact spectrum decide (main stream)
    TPB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    leaf_scratch_reserve(ctx, s, static_cast<long long>(lane.rows), 0);
    TPB_SOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                static_cast<int>(lane.rows), lane.gram, static_cast<int>(lane.rows), s.w, s.work,
                                s.lwork, info));
    ctx->library_calls += 1;
    TPB_CUDA(launch_select_basis(ctx->stream, lane.gram, s.w, static_cast<int>(lane.rows),
                                 static_cast<int>(lane.rows), lane.k, factor, flag));
    ctx->own_kernels += 1;
  });
}

int tp_dev_leaf_solve_warm(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                           int* flag, int* info, int* used_fast) {
  return guarded([&] {
    bind(ctx);
    if (!gram || !factor || !flag || !info) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_leaf_args(static_cast<long long>(rows), 1, k);
    if (used_fast) *used_fast = 0;
    LeafScratch& s = dev_scratch(ctx);
    if (start && subspace_eligible(static_cast<long long>(rows), k)) {
      reserve_iteration_buffers(ctx, s, static_cast<long long>(rows), k);
      int* const saved_flag = s.flag;
      s.flag = flag;  // the caller's degenerate flag
      s.last_ritz = nullptr;  // the result of this entry point depends on its arguments only (replicas stay identical)
      leaf_solve_subspace(ctx, s, gram, static_cast<long long>(rows), k, start, factor, -1);
      s.flag = saved_flag;
      s.fast_used = false;
      int host[3] = {0, 0, 0};
      TPB_CUDA(cudaMemcpyAsync(&host[0], s.verdict, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaMemcpyAsync(&host[2], flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TPB_CUDA(cudaStreamSynchronize(ctx->stream));
      if (host[0] == 0 && host[1] == 0 && host[2] == 0) {
        TPB_CUDA(cudaMemsetAsync(info, 0, sizeof(int), ctx->stream));
        if (used_fast) *used_fast = 1;
        return;
      }
      s.last_ritz = nullptr;
      TPB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));  // let the exact spectrum decide
    }
    leaf_scratch_reserve(ctx, s, static_cast<long long>(rows), 0);
    TPB_SOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(rows),
                                gram, static_cast<int>(rows), s.w, s.work, s.lwork, info));
    ctx->library_calls += 1;
    TPB_CUDA(launch_select_basis(ctx->stream, gram, s.w, static_cast<int>(rows), static_cast<int>(rows), k, factor,
                                 flag));
    ctx->own_kernels += 1;
  });
}

static void check_block(int block) {
  if (block < 1 || static_cast<size_t>(block) > small_evd_max_block())
    raise(TP_ERR_BAD_ARGUMENT, "block size outside 1.." + std::to_string(small_evd_max_block()));
}

int tp_dev_cholesky(tp_ctx* ctx, const double* s, int block, double* l, int* fail) {
  return guarded([&] {
    bind(ctx);
    if (!s || !l || !fail) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_block(block);
    TPB_CUDA(launch_cholesky(ctx->stream, s, block, l, fail));
    ctx->own_kernels += 1;
  });
}

int tp_dev_trsm_right_lt(tp_ctx* ctx, double* z, size_t rows, int block, const double* l) {
  return guarded([&] {
    bind(ctx);
    if (!z || !l) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_block(block);
    if (rows == 0) return;
    if (rows > static_cast<size_t>(TP_MAX_GRAM_ROWS)) raise(TP_ERR_TOO_LARGE, "too many rows");
    TPB_CUDA(launch_trsm_right_lt(ctx->stream, z, static_cast<int>(rows), block, l));
    ctx->own_kernels += 1;
  });
}

int tp_dev_jacobi_eig(tp_ctx* ctx, const double* h, int block, double* w, double* v, int* fail) {
  return guarded([&] {
    bind(ctx);
    if (!h || !w || !v || !fail) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_block(block);
    TPB_CUDA(launch_jacobi_eig(ctx->stream, h, block, w, v, fail));
    ctx->own_kernels += 1;
  });
}

int tp_dev_leaf_solve_fused(tp_ctx* ctx, const double* gram, size_t rows, int k, const double* start,
                            int start_is_ritz, double* ritz, double* theta, double* factor, int* flag, int* verdict,
                            double* diag) {
  return guarded([&] {
    bind(ctx);
    if (!gram || !start || !ritz || !theta || !factor || !flag || !verdict || !diag)
      raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    check_leaf_args(static_cast<long long>(rows), 1, k);
    const int b = k + kSubspaceOversample;
    if (!leaf_solve_fused_eligible(static_cast<long long>(rows), k, b))
      raise(TP_ERR_BAD_ARGUMENT, "leaf too large for the one-launch solve (rows <= 512, k + 8 <= 64, see the header)");
    TPB_CUDA(launch_leaf_solve_fused(ctx->stream, gram, static_cast<int>(rows), k, b, start, start_is_ritz ? 0 : 1,
                                     start_is_ritz ? 1 : 3, 4, kSubspaceTol, kSubspaceAngleTol, ritz, theta, factor,
                                     flag, verdict, diag));
    ctx->own_kernels += 1;
  });
}

int tp_dev_sum_squares(tp_ctx* ctx, const double* x, size_t count, double* out) {
  return guarded([&] {
    bind(ctx);
    if (!x || !out) raise(TP_ERR_BAD_ARGUMENT, "null pointer");
    TPB_CUDA(launch_sum_squares(ctx->stream, x, count, ctx->reduce_scratch, out));
    ctx->own_kernels += 2;
  });
}

int tp_ctx_release_cache(tp_ctx* ctx) {
  return guarded([&] {
    bind(ctx);
    release_host_call_cache(ctx);
  });
}

int tp_hooi_sweep_host(tp_ctx* ctx, int n_modes, const size_t* dims, const double* tensor, const tp_u64* K,
                       const double* const* factors_in, int n_nodes, const int* kind, const int* mode,
                       const int* parent, int sweep_kind, double* const* factors_out, double* core_out,
                       tp_sweep_stats* stats) {
  return tp_hooi_sweep_host_ex(ctx, n_modes, dims, tensor, K, factors_in, n_nodes, kind, mode, parent, sweep_kind, 0,
                               factors_out, core_out, stats);
}

int tp_hooi_sweep_host_ex(tp_ctx* ctx, int n_modes, const size_t* dims, const double* tensor, const tp_u64* K,
                          const double* const* factors_in, int n_nodes, const int* kind, const int* mode,
                          const int* parent, int sweep_kind, unsigned flags, double* const* factors_out,
                          double* core_out, tp_sweep_stats* stats) {
  return guarded([&] {
    bind(ctx);
    struct Busy {  // the allocator must not give up the cache this call is working with
      tp_ctx* c;
      explicit Busy(tp_ctx* ctx_) : c(ctx_) { c->host_call_busy = true; }
      ~Busy() { c->host_call_busy = false; }
    } busy(ctx);
    if (!dims || !tensor || !K || !factors_in) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    std::vector<u64> L(dims, dims + std::max(n_modes, 0));
    std::vector<long long> key{n_modes, n_nodes, sweep_kind};
    for (int m = 0; m < n_modes; ++m) {
      key.push_back(static_cast<long long>(dims[m]));
      key.push_back(static_cast<long long>(K[m]));
    }
    for (int i = 0; i < n_nodes && kind && mode && parent; ++i) {
      key.push_back(kind[i]);
      key.push_back(mode[i]);
      key.push_back(parent[i]);
    }
    auto forward = [&](int status) {
      if (status == TP_OK) return;
      const std::string msg = tp_last_error();
      const int bad = tp_last_error_mode();
      release_host_call_cache(ctx);
      raise(status, msg, bad);
    };
    bool fresh_cache = false;
    if (key != ctx->host_call_key || !ctx->host_call_plan || !ctx->host_call_tensor) {
      release_host_call_cache(ctx);
      forward(tp_plan_create(ctx, n_modes, L.data(), K, n_nodes, kind, mode, parent, sweep_kind, &ctx->host_call_plan));
      forward(tp_tensor_alloc(ctx, n_modes, dims, &ctx->host_call_tensor));
      ctx->host_call_key = key;
      fresh_cache = true;
    }
    tp_tensor* t = ctx->host_call_tensor;
    tp_plan* plan = ctx->host_call_plan;
    // TP_HOST_TENSOR_UNCHANGED: the caller promises that `tensor` still holds what the previous call uploaded from the
    // same address, so the device copy is reused and only the factors travel.
    const bool reuse_tensor = (flags & TP_HOST_TENSOR_UNCHANGED) && !fresh_cache && ctx->host_call_source == tensor;
    // factors that are bit for bit the ones the previous call returned continue that run on the device: the warm
    // eigen-solve state and the carried products stay valid, exactly as in a resident tp_plan_sweep loop
    bool same_factors = reuse_tensor && static_cast<int>(ctx->host_call_last_factors.size()) == n_modes;
    for (int m = 0; same_factors && m < n_modes; ++m) {
      const std::vector<double>& last = ctx->host_call_last_factors[m];
      same_factors = factors_in[m] && last.size() == static_cast<size_t>(dims[m] * K[m]) &&
                     std::memcmp(last.data(), factors_in[m], last.size() * sizeof(double)) == 0;
    }
    if (!reuse_tensor) t->stamp = next_tensor_stamp();
    if (!same_factors) forward(tp_plan_set_factors(ctx, plan, factors_in));
    auto remember = [&] {
      ctx->host_call_source = tensor;
      ctx->host_call_last_factors.assign(n_modes, {});
      if (!factors_out) return;
      for (int m = 0; m < n_modes; ++m)
        ctx->host_call_last_factors[m].assign(factors_out[m], factors_out[m] + dims[m] * K[m]);
    };
    if (reuse_tensor) {
      forward(tp_plan_sweep(ctx, plan, t, stats));
      if (factors_out) forward(tp_plan_get_factors(ctx, plan, factors_out));
      if (core_out) forward(tp_plan_get_core(ctx, plan, core_out));
      remember();
      return;
    }
    ctx->host_call_source = nullptr;
    // Large tensors go up in slabs of the first mode on a copy stream; the sweep starts on the slabs that have
    // arrived (jacobi_walk_streamed_root) instead of idling through the whole PCIe transfer.
    const size_t rows = dims[0];
    const size_t per_row = t->size / rows;
    int chunks = 1;
    const size_t min_bytes = ctx->streamed_upload_min_bytes;  // below this the transfer is too short to split
    if (n_modes > 1 && t->size * sizeof(double) >= min_bytes && rows >= 32)
      chunks = static_cast<int>(std::min<size_t>(8, rows / 16));
    if (chunks == 1) {
      TPB_CUDA(cudaMemcpyAsync(t->data, tensor, t->size * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      forward(tp_plan_sweep(ctx, plan, t, stats));
    } else {
      if (!ctx->copy_stream) TPB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      while (static_cast<int>(ctx->arrival_events.size()) < chunks) {
        cudaEvent_t e;
        TPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->arrival_events.push_back(e);
      }
      tp_plan::Arrival arrival;
      const size_t step = ((rows + chunks - 1) / chunks + 15) / 16 * 16;  // whole contraction chunks per slab
      for (size_t r = step; r < rows; r += step) arrival.row_end.push_back(r);
      arrival.row_end.push_back(rows);
      arrival.ready.assign(ctx->arrival_events.begin(), ctx->arrival_events.begin() + arrival.row_end.size());
      int issued = 0;
      arrival.issue = [&](int c) {
        for (; issued <= c; ++issued) {
          const size_t r0 = issued ? arrival.row_end[issued - 1] : 0, r1 = arrival.row_end[issued];
          TPB_CUDA(cudaMemcpyAsync(t->data + r0 * per_row, tensor + r0 * per_row, (r1 - r0) * per_row * sizeof(double),
                                   cudaMemcpyHostToDevice, ctx->copy_stream));
          TPB_CUDA(cudaEventRecord(arrival.ready[issued], ctx->copy_stream));
        }
      };
      plan->arrival = &arrival;
      const int status = tp_plan_sweep(ctx, plan, t, stats);
      plan->arrival = nullptr;
      if (status != TP_OK) {
        cudaStreamSynchronize(ctx->copy_stream);  // `tensor` must not be read after this call returns
        forward(status);
      }
      arrival.issue(static_cast<int>(arrival.row_end.size()) - 1);
      TPB_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    }
    if (factors_out) forward(tp_plan_get_factors(ctx, ctx->host_call_plan, factors_out));
    if (core_out) forward(tp_plan_get_core(ctx, ctx->host_call_plan, core_out));
    remember();
  });
}

}  // extern "C"
