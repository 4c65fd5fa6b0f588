/*
 * tuckerplan_b200 — C ABI of the B200-native HOOI engine.
 *
 * This is the drop-in boundary for the reference's header-only C++ API
 * (`#include "tuckerplan/tuckerplan.hpp"`, reference proj/include/tuckerplan/).
 * The reference has no FFI of its own; every entry point below names the
 * reference function it replaces (file:line relative to
 * /root/reference/proj/include/tuckerplan/).  The C++ wrappers in
 * include/tuckerplan/ (this repo) re-create the reference signatures on top of
 * these calls; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - plain pointers and sizes only; the caller owns every host buffer, the
 *     library owns device memory behind opaque handles;
 *   - every function returns TP_OK (0) or an error code; codes 1..13 are the
 *     reference's `Errc` ordinals + 1 (errors.hpp:16-30); the offending mode
 *     and message are read with tp_last_error_mode() / tp_last_error();
 *   - matrices are COLUMN-MAJOR (rows x cols, leading dimension = rows), the
 *     layout of Eigen::MatrixXd in the reference signatures; tensors are
 *     row-major, last index fastest (dense_tensor.hpp:19-30);
 *   - trees are flat arrays kind/mode/parent in the reference's stored order
 *     (parent first, node 0 = root, children in insertion order,
 *     ttm_tree.hpp:36-57); kinds are 0 root, 1 mode, 2 leaf (ttm_tree.hpp:27);
 *   - a context is bound to one CUDA device and is not thread-safe;
 *   - there is NO CPU fallback: device entry points fail with TP_ERR_CUDA when
 *     no sm_100 device / driver is present.
 */
#ifndef TUCKERPLAN_B200_H
#define TUCKERPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef uint64_t tp_u64;

/* errors.hpp:16-30 (ordinal + 1) */
enum {
  TP_OK = 0,
  TP_ERR_BAD_DIMS = 1,
  TP_ERR_K_TOO_LARGE = 2,
  TP_ERR_OVERFLOW = 3,
  TP_ERR_BAD_TREE = 4,
  TP_ERR_BAD_MODE = 5,
  TP_ERR_SHAPE_MISMATCH = 6,
  TP_ERR_INVALID_GRID = 7,
  TP_ERR_NO_VALID_GRID = 8,
  TP_ERR_MISSING_ASSIGNMENT = 9,
  TP_ERR_TOO_LARGE = 10,
  TP_ERR_ZERO_TENSOR = 11,
  TP_ERR_NEEDS_CHAIN_TREE = 12,
  TP_ERR_BAD_ARGUMENT = 13,
  /* outside the reference enum */
  TP_ERR_CUDA = 100,      /* CUDA / cuSOLVER runtime failure, or no device */
  TP_ERR_NCCL = 101,      /* NCCL failure */
  TP_ERR_CAPACITY = 102,  /* caller-provided output array too small */
  TP_ERR_INTERNAL = 103
};

enum { TP_NODE_ROOT = 0, TP_NODE_MODE = 1, TP_NODE_LEAF = 2 };      /* ttm_tree.hpp:27 */
enum { TP_CHAIN_INPUT = 0, TP_CHAIN_BY_COST = 1, TP_CHAIN_BY_RATIO = 2 }; /* tree_builders.hpp:25 */
enum { TP_SWEEP_JACOBI = 0, TP_SWEEP_GAUSS_SEIDEL = 1 };            /* hooi.hpp:132 */
/* bench.hpp:115 TreeStrategy */
enum { TP_TREE_CHAIN_INPUT = 0, TP_TREE_CHAIN_BY_COST = 1, TP_TREE_CHAIN_BY_RATIO = 2,
       TP_TREE_BALANCED = 3, TP_TREE_OPTIMAL = 4 };

#define TP_MAX_MODES 16        /* mode_set.hpp:15 */
#define TP_MAX_GRAM_ROWS 2048  /* hooi.hpp:32 */

const char* tp_last_error(void);   /* message of the last failure on this thread */
int tp_last_error_mode(void);      /* Error::mode() of that failure, -1 if none */
const char* tp_version(void);

/* ------------------------------------------------------------------ planner
 * Pure host code, exact u64 arithmetic, selections bit-identical to the
 * reference. */

/* validate_spec — problem.hpp:37-53 */
int tp_validate_spec(int n_modes, const tp_u64* L, const tp_u64* K);
/* input/core/partial_cardinality — problem.hpp:67-86 (done_mask bit m = mode m multiplied) */
int tp_partial_cardinality(int n_modes, const tp_u64* L, const tp_u64* K, uint32_t done_mask, tp_u64* out);

/* optimal_tree — tree_opt.hpp:126-138.  Writes up to `cap` nodes. */
int tp_optimal_tree(int n_modes, const tp_u64* L, const tp_u64* K, int cap, int* kind, int* mode, int* parent,
                    int* n_nodes, tp_u64* total_macs, tp_u64* dp_states);
/* optimal_cost_reuse_greedy — tree_opt.hpp:143-150 */
int tp_reuse_greedy_cost(int n_modes, const tp_u64* L, const tp_u64* K, tp_u64* cost);
/* chain_tree — tree_builders.hpp:49-60 */
int tp_chain_tree(int n_modes, const tp_u64* L, const tp_u64* K, int order, int cap, int* kind, int* mode,
                  int* parent, int* n_nodes);
/* balanced_tree — tree_builders.hpp:85-91 */
int tp_balanced_tree(int n_modes, const tp_u64* L, const tp_u64* K, int cap, int* kind, int* mode, int* parent,
                     int* n_nodes);
/* build_tree — bench.hpp:128-137 */
int tp_build_tree(int n_modes, const tp_u64* L, const tp_u64* K, int strategy, int cap, int* kind, int* mode,
                  int* parent, int* n_nodes);
/* validate_tree — ttm_tree.hpp:103-119 */
int tp_validate_tree(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind,
                     const int* mode, const int* parent);
/* is_canonical / canonicalize / tree_depth — ttm_tree.hpp:123-187 */
int tp_tree_is_canonical(int n_nodes, const int* kind, const int* mode, const int* parent, int* out);
int tp_canonicalize(int n_modes, int n_nodes, const int* kind, const int* mode, const int* parent, int cap,
                    int* out_kind, int* out_mode, int* out_parent, int* out_n_nodes);
int tp_tree_depth(int n_nodes, const int* kind, const int* mode, const int* parent, int* depth);
/* node_cardinalities + tree_cost — tree_cost.hpp:25-63.  card_in/card_out/per_node_macs have n_nodes entries
 * (any may be NULL). */
int tp_tree_cost(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                 const int* parent, tp_u64* total_macs, tp_u64* per_node_macs, tp_u64* card_in, tp_u64* card_out,
                 int* n_internal, int* depth);

/* grid_count psi(P,N) — grid.hpp:49-70 */
int tp_grid_count(tp_u64 procs, int n_modes, tp_u64* out);
/* validate_grid — grid.hpp:36-45 */
int tp_validate_grid(int n_modes, const tp_u64* L, const tp_u64* K, const tp_u64* q, tp_u64 procs);
/* enumerate_grids — grid.hpp:96-111.  grids_out is cap_grids x n_modes, lexicographic order. */
int tp_enumerate_grids(int n_modes, const tp_u64* L, const tp_u64* K, tp_u64 procs, size_t cap_grids,
                       tp_u64* grids_out, size_t* n_grids);
/* block_bounds / block_of — grid.hpp:114-125.  cuts has parts+1 entries. */
int tp_block_bounds(tp_u64 len, tp_u64 parts, tp_u64* cuts);
int tp_block_of(tp_u64 c, tp_u64 len, tp_u64 parts, tp_u64* out);
/* static_volume — grid_volume.hpp:32-46.  per_node_ttm has n_nodes entries (0 for root/leaves), may be NULL. */
int tp_static_volume(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                     const int* parent, const tp_u64* q, tp_u64 procs, tp_u64* total, tp_u64* per_node_ttm);
/* optimal_static_grid — grid_volume.hpp:56-110 (first minimum in lexicographic order). */
int tp_optimal_static_grid(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind,
                           const int* mode, const int* parent, tp_u64 procs, int threads, tp_u64* q_out,
                           tp_u64* total, tp_u64* per_node_ttm);

/* Per-node grids — grid_dynamic.hpp.  A scheme = the root's anchor grid + one grid per TTM node; node_grids is
 * n_nodes x n_modes row-major, rows of the root and of leaves are ignored on input and zero on output.
 * scheme_volume — grid_dynamic.hpp:37-62: per node (q_n - 1)|Out_u| plus |In_u| where the grid differs from the
 * parent's; per_node_ttm / per_node_regrid have n_nodes entries and may be NULL. */
int tp_scheme_volume(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                     const int* parent, const tp_u64* root_grid, const tp_u64* node_grids, tp_u64 procs,
                     tp_u64* total, tp_u64* per_node_ttm, tp_u64* per_node_regrid);
/* optimal_dynamic_scheme — grid_dynamic.hpp:141-167 (ties: keep the parent's grid; first regrid target in
 * enumeration order); legacy_target != 0 = DynamicOptions::legacy_regrid_target (grid_dynamic.hpp:64-66). */
int tp_optimal_dynamic_scheme(int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind,
                              const int* mode, const int* parent, tp_u64 procs, int legacy_target,
                              tp_u64* root_grid_out, tp_u64* node_grids_out, tp_u64* total, tp_u64* per_node_ttm,
                              tp_u64* per_node_regrid);
/* count_moved — simulate.hpp:104-121: elements of a tensor with extents ext whose owner rank differs between the
 * two grids (what a regrid ships, summed over ranks). */
int tp_count_moved(int n_modes, const tp_u64* ext, const tp_u64* from_grid, const tp_u64* to_grid, tp_u64* out);

/* --------------------------------------------------------- seeded host data
 * libstdc++ mt19937_64 + ONE normal_distribution<double>(0,1) object. */

/* random_tensor — dense_tensor.hpp:43-49.  out has prod(dims) entries. */
int tp_random_tensor(int n_modes, const size_t* dims, tp_u64 seed, double* out);
/* the factor part of random_decomposition — hooi.hpp:109-120: per mode an L_n x K_n gaussian matrix filled column
 * by column from one shared stream, thin Q of its Householder QR.  factors_out[n] is L_n x K_n column-major. */
int tp_random_orthonormal_factors(int n_modes, const tp_u64* L, const tp_u64* K, tp_u64 seed,
                                  double* const* factors_out);
/* frobenius_norm — dense_tensor.hpp:51-55 (host data; same left-to-right sum) */
int tp_frobenius_norm_host(size_t n, const double* data, double* out);

/* ------------------------------------------------------------ device engine */
typedef struct tp_ctx tp_ctx;
typedef struct tp_tensor tp_tensor;   /* row-major FP64 tensor resident in HBM */
typedef struct tp_plan tp_plan;       /* spec + tree + arena + launch schedule for repeated sweeps */

/* number of CUDA devices visible to this process (0 and TP_OK when there is no driver) */
int tp_device_count(int* out);
int tp_ctx_create(int device, tp_ctx** out);
/* Same with creation flags.  The eigen-solve side streams normally outrank the stream the tree runs on (their kernels
 * are short and latency-bound); the flags put them on the same priority or below it (A/B measurements). */
enum { TP_CTX_SIDE_STREAMS_SAME_PRIORITY = 1, TP_CTX_SIDE_STREAMS_LOW_PRIORITY = 2 };
int tp_ctx_create_ex(int device, unsigned flags, tp_ctx** out);
int tp_ctx_destroy(tp_ctx* ctx);
/* Context options (plain values through the ABI; the library reads no environment variables).
 *   TP_CTX_OPT_STREAMED_UPLOAD_MIN_BYTES  by-value hooi_sweep calls upload tensors of at least this many bytes in
 *                                         slabs and start multiplying the slabs that have arrived (default 256 MiB)
 *   TP_CTX_OPT_TRACE_EVD                  != 0: one line per leaf and sweep on stderr with the certificate margins
 *   TP_CTX_OPT_DUMP_SWEEP_GRAPH           != 0: a recorded sweep's CUDA graph goes to /tmp/tpb_sweep_graph.dot (debugging) */
enum { TP_CTX_OPT_STREAMED_UPLOAD_MIN_BYTES = 1, TP_CTX_OPT_TRACE_EVD = 2, TP_CTX_OPT_DUMP_SWEEP_GRAPH = 3 };
int tp_ctx_set_option(tp_ctx* ctx, int option, long long value);
/* Process-wide switches.  TP_GLOBAL_OPT_TTM_TMA (default 1): 0 forces the cp.async TTM kernel where the TMA pipeline
 * would be chosen (both compute the same sums in the same order).  TP_GLOBAL_OPT_TTM_PACKED (default 1): 0 sends
 * products with a short trailing extent (1 < inner < 8) to the general kernels instead of the packed-column one
 * (same sums, same order).  TP_GLOBAL_OPT_TTM_SPLITK (default 1): 0 sends the small nodes (at most 640 column tiles,
 * contraction 32..512) to the streaming kernels instead of the kernel that splits the contraction over a CTA's warps
 * (same sums to rounding: the eight partial sums are added in warp order, so the last bits differ).
 * TP_GLOBAL_OPT_GRAM_WIDE (default 1): 0 keeps the Gram matrices of large leaves (>= 448 rows) on the 64 x 64
 * cp.async kernel instead of the 128 x 128 TMA pipeline (same sums to rounding: the contraction range is split
 * differently).  TP_GLOBAL_OPT_GRAM_WIDE_SPARE_SMS (default 0, 0..64): SMs that kernel's persistent grid leaves to
 * eigen-solves running beside it during a sweep.  TP_GLOBAL_OPT_CARRY_FIRST (0 never, 1 always, 2 = default: in
 * short sweeps): plans created afterwards walk the subtree whose products were carried over from the previous sweep
 * first instead of last (a Jacobi sweep gives the same factors in any visiting order). */
enum {
  TP_GLOBAL_OPT_TTM_TMA = 1,
  TP_GLOBAL_OPT_TTM_PACKED = 2,
  TP_GLOBAL_OPT_TTM_SPLITK = 3,
  TP_GLOBAL_OPT_GRAM_WIDE = 4,
  TP_GLOBAL_OPT_GRAM_WIDE_SPARE_SMS = 5,
  TP_GLOBAL_OPT_CARRY_FIRST = 6
};
int tp_set_global_option(int option, long long value);
int tp_ctx_synchronize(tp_ctx* ctx);
/* the CUDA stream the engine launches on (cudaStream_t as void*), for event timing by the caller */
int tp_ctx_stream(tp_ctx* ctx, void** stream_out);
/* number of kernels this context has launched so far (own kernels + cuSOLVER calls counted separately) */
int tp_ctx_launch_counts(tp_ctx* ctx, tp_u64* own_kernels, tp_u64* library_calls);

/* pinned host staging buffers for callers that want full-speed PCIe copies */
int tp_host_alloc(size_t bytes, void** out);
int tp_host_free(void* p);

/* DenseTensor upload/download (dense_tensor.hpp:19-30 value type <-> device handle) */
int tp_tensor_upload(tp_ctx* ctx, int n_modes, const size_t* dims, const double* host, tp_tensor** out);
int tp_tensor_alloc(tp_ctx* ctx, int n_modes, const size_t* dims, tp_tensor** out);   /* zeros(), :32-39 */
int tp_tensor_download(tp_ctx* ctx, const tp_tensor* t, double* host);
int tp_tensor_free(tp_ctx* ctx, tp_tensor* t);
int tp_tensor_dims(const tp_tensor* t, int* n_modes, size_t* dims /* TP_MAX_MODES entries */);
/* Raw device pointer.  The library cannot see writes through it, so from this call on no product of the tensor is
 * carried between sweeps (TP_OPT_CARRY_PATH) -- until the caller takes over the bookkeeping with
 * tp_tensor_mark_modified, to be called after every batch of writes through the pointer. */
void* tp_tensor_device_ptr(const tp_tensor* t);
int tp_tensor_mark_modified(tp_ctx* ctx, tp_tensor* t);
/* frobenius_norm — dense_tensor.hpp:51-55, on the device (deterministic pairwise reduction) */
int tp_tensor_norm(tp_ctx* ctx, const tp_tensor* t, double* out);
/* y = beta * y + alpha * x, elementwise on the device (input assembly: T = X + sigma E; no reference counterpart) */
int tp_tensor_axpby(tp_ctx* ctx, tp_tensor* y, double beta, double alpha, const tp_tensor* x);

/* ttm — ttm.hpp:73-96.  m is new_len x dims[mode], column-major host matrix.  *macs (may be NULL) is
 * ACCUMULATED with the exact new_len * size(t), overflow-checked. */
int tp_ttm(tp_ctx* ctx, const tp_tensor* t, const double* m, size_t m_rows, size_t m_cols, int mode, tp_u64* macs,
           tp_tensor** out);
/* same with the matrix already on the device as a ROW-major m_rows x m_cols array (== column-major transpose,
 * i.e. a reference factor F (L x K col-major) passed as F^T without any copy, hooi.hpp:98,153) */
int tp_ttm_device(tp_ctx* ctx, const tp_tensor* t, const double* m_dev_rowmajor, size_t m_rows, size_t m_cols,
                  int mode, tp_u64* macs, tp_tensor** out);

/* leading_left_factors — hooi.hpp:45-76.  m is rows x cols column-major on the host; vectors_out rows x k
 * column-major; *degenerate 0/1. */
int tp_leading_left_factors(tp_ctx* ctx, const double* m, size_t rows, size_t cols, int k, double* vectors_out,
                            int* degenerate);
/* Gram + truncated basis of the mode-n unfolding of a device tensor, without materialising the unfolding
 * (unfold ttm.hpp:43-53 + leading_left_factors hooi.hpp:45-76 as used at hooi.hpp:147-151) */
int tp_leaf_factor(tp_ctx* ctx, const tp_tensor* t, int mode, int k, double* vectors_out, int* degenerate);
/* Gram matrix Y_(n) Y_(n)^T only (rows x rows, symmetric, column-major, full storage) */
int tp_gram(tp_ctx* ctx, const tp_tensor* t, int mode, double* gram_out);

/* Sequentially truncated HOSVD start (no reference counterpart: SPEC.md:17 leaves initialisation beyond the random
 * start out of the reference's scope; PAPER.md:53-54 names it as what HOOI is started from).  For each mode in `order`
 * (NULL = 0 .. N-1, else a permutation): F_n = the K_n leading eigenvectors of the Gram matrix of the mode-n unfolding
 * of the current tensor, selected and signed as hooi.hpp:60-68 does, then the tensor is truncated along that mode.
 * factors_out[n]: L_n x K_n column-major (may be NULL), core_out: prod(K) doubles row-major (may be NULL),
 * *degenerate: OR of the gap flags, *macs accumulates the exact multiply-adds of the truncations. */
int tp_sthosvd(tp_ctx* ctx, const tp_tensor* t, const tp_u64* K, const int* order, double* const* factors_out,
               double* core_out, int* degenerate, tp_u64* macs);

typedef struct tp_sweep_stats {   /* SweepStats, hooi.hpp:125-130 */
  tp_u64 tree_macs;
  tp_u64 core_macs;
  int peak_live;
  int degenerate;
} tp_sweep_stats;

typedef struct tp_sweep_timing {  /* device milliseconds of the last sweep, CUDA events on the engine stream */
  float total_ms;
  float tree_ms;   /* TTM-tree phase: every tree TTM (+ the factor-fragment prep kernels) */
  float gram_ms;
  float evd_ms;    /* eigen-solve + sign/gap kernel */
  float core_ms;
} tp_sweep_timing;

/* Build the launch schedule for hooi_sweep (hooi.hpp:189-229) on a fixed spec/tree: validates, sizes the arena from
 * node_cardinalities, allocates device factors.  kind: TP_SWEEP_JACOBI or TP_SWEEP_GAUSS_SEIDEL (chain trees only,
 * TP_ERR_NEEDS_CHAIN_TREE otherwise). */
int tp_plan_create(tp_ctx* ctx, int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind,
                   const int* mode, const int* parent, int sweep_kind, tp_plan** out);
int tp_plan_destroy(tp_ctx* ctx, tp_plan* plan);
/* Execution options (results are identical either way).  TP_OPT_OVERLAP_EVD (default 1): in a Jacobi sweep run each
 * leaf's eigen-solve on a side stream beside the remaining tree TTMs; 0 serialises everything on one stream, which is
 * what per-kernel timing and profiling want. */
enum { TP_OPT_OVERLAP_EVD = 1, TP_OPT_FAST_EVD = 2, TP_OPT_CARRY_PATH = 3, TP_OPT_SPARE_SMS = 4,
       TP_OPT_SPARE_SMS_SHORT = 5, TP_OPT_SWEEP_GRAPH = 6, TP_OPT_LEAF_GRAPH = 7, TP_OPT_FUSED_LEAF_SOLVE = 8,
       TP_OPT_FORK_SUBTREES = 9 };
/* TP_OPT_SPARE_SMS / _SHORT (defaults 2 / 16): SMs a long / short tree product leaves to eigen-solves in flight.
 * TP_OPT_SWEEP_GRAPH (0 off, 1 on, 2 auto = default): replay the steady-state Jacobi sweep -- tree, Gram kernels, leaf
 *   solves, core chain, status read-back -- as ONE CUDA graph; auto does so for sweeps below ~5e10 flops, where the
 *   ~100 launches of a sweep would otherwise pace it.  Per-node timings are not available for replayed sweeps.
 * TP_OPT_LEAF_GRAPH (default 1): replay a large leaf's multi-launch top-k iteration as a CUDA graph.
 * TP_OPT_FUSED_LEAF_SOLVE (default 1): leaves with L_n <= 512 and K_n + 8 <= 64 run their whole certified top-k
 *   solve in one launch (csrc/leaf_solve_kernels.cu).
 * TP_OPT_FORK_SUBTREES (0 off, 1 on, 2 auto = default): in a Jacobi sweep the subtrees below a tree node run on
 *   streams of their own (siblings get one output buffer each instead of one per depth), so the short products and
 *   Gram kernels of small tensors overlap; auto forks the sweeps TP_OPT_SWEEP_GRAPH's auto replays. */
int tp_plan_set_option(tp_ctx* ctx, tp_plan* plan, int option, int value);
/* TP_OPT_CARRY_PATH (default 1; Gauss-Seidel plans carry the first leaf's chain): the core chain core_from_factors (hooi.hpp:93-100) contracts the modes
 * along one root-to-leaf path of the TTM tree; with the new factors its partial products are exactly the
 * intermediates the next sweep's tree needs at those nodes, so they are kept on the device and the next tp_plan_sweep
 * on the same, unchanged tensor starts from them: per sweep every tree node is computed once and the core costs one
 * small product instead of a second pass over the tensor.  The carried products are dropped by tp_plan_set_factors,
 * by a sweep on another tensor, and whenever the tensor may have changed (tp_tensor_axpby, tp_tensor_device_ptr --
 * take the pointer again after writing through it).  SweepStats stay the analytic (reference) counts.
 * TP_OPT_FAST_EVD (default 1): leaves with 2 (K_n + 8) <= L_n (and K_n + 8 <= 112 or L_n >= 704) compute only
 * the K_n leading eigenvectors by warm-started block subspace iteration + Rayleigh-Ritz, accepted only with a
 * certificate: (1) every kept Ritz pair has ||G x - theta x|| <= 1e-13 theta_max; (2) no larger eigenvalue was missed
 * -- G is positive semidefinite, so whatever the block does not account for is bounded by trace(G) - sum(theta) plus
 * the block residual, and that bound must lie below theta_K; (3) the Davis-Kahan bound ||R_kept|| / gap on the angle
 * to the true leading subspace is <= 1e-10, so small spectral gaps are never trusted to the iteration.  A leaf that
 * only misses (1) iterates on (up to three more rounds from the Ritz vectors it reached); a leaf that still misses,
 * misses (2)/(3), loses a factorisation or has a "degenerate" gap estimate is redone with the full eigen-solve, so
 * the factors are the reference's (hooi.hpp:55-69) to rounding either way.  tp_plan_last_evd_info: leaves eligible for the fast path, and how many of them the last sweep had to
 * redo with the full solve. */
int tp_plan_last_evd_info(tp_ctx* ctx, tp_plan* plan, int* fast_eligible, int* rejected);
/* whether the last tp_plan_sweep was a replay of the recorded whole-sweep graph (TP_OPT_SWEEP_GRAPH), and how many of
 * the plan's leaves take the one-launch solve (TP_OPT_FUSED_LEAF_SOLVE) */
int tp_plan_last_sweep_info(tp_ctx* ctx, tp_plan* plan, int* replayed_graph, int* one_launch_leaves);
/* Decomposition::factors (hooi.hpp:78-81) <-> device: factors[n] is L_n x K_n column-major on the host */
int tp_plan_set_factors(tp_ctx* ctx, tp_plan* plan, const double* const* factors);
int tp_plan_get_factors(tp_ctx* ctx, tp_plan* plan, double* const* factors_out);
/* the plan's factors and core <- tp_sthosvd of the device tensor, without leaving the device */
int tp_plan_init_sthosvd(tp_ctx* ctx, tp_plan* plan, const tp_tensor* t, const int* order);
/* Decomposition::core — prod(K) doubles, row-major */
int tp_plan_get_core(tp_ctx* ctx, tp_plan* plan, double* core_out);
int tp_plan_core_norm(tp_ctx* ctx, tp_plan* plan, double* out);
/* core_from_factors — hooi.hpp:93-100 with the plan's current factors (used by random_decomposition, :121) */
int tp_plan_compute_core(tp_ctx* ctx, tp_plan* plan, const tp_tensor* t);
/* One hooi_sweep on the device-resident tensor: the plan's factors are the input Decomposition and are replaced by
 * the output one; the core is recomputed (hooi.hpp:227).  stats may be NULL. */
int tp_plan_sweep(tp_ctx* ctx, tp_plan* plan, const tp_tensor* t, tp_sweep_stats* stats);
int tp_plan_last_timing(tp_ctx* ctx, tp_plan* plan, tp_sweep_timing* out);
/* per tree node of the last sweep (n_nodes entries each, either may be NULL): node_ms = device time of the node's
 * TTM launch (mode nodes) or Gram kernels (leaves); evd_ms = eigen-solve + basis selection (leaves, else 0).
 * Jacobi plans only. */
int tp_plan_node_timing(tp_ctx* ctx, tp_plan* plan, int n_nodes, float* node_ms, float* evd_ms);
/* reconstruction_error — hooi.hpp:232-245, full expansion on the device (materialises |T| elements). */
int tp_plan_reconstruction_error(tp_ctx* ctx, tp_plan* plan, const tp_tensor* t, double* out);
/* same quantity from ||T||^2 - ||G||^2 (valid for orthonormal factors and the core of those factors) */
int tp_plan_fit_from_norms(tp_ctx* ctx, tp_plan* plan, const tp_tensor* t, double* out);

/* reconstruction_error for an arbitrary host Decomposition (core row-major with dims core_dims, factors[n]
 * dims[n] x core_dims[n] column-major) */
int tp_reconstruction_error(tp_ctx* ctx, const tp_tensor* t, const size_t* core_dims, const double* core,
                            const double* const* factors, double* out);

/* ------------------------------------------------- device-pointer building blocks (multi-GPU driver)
 * The Cartesian-grid executor (paper_1707_05594_b200/distributed.py, one process per GPU) owns its device buffers
 * and the collectives; these entry points are the local kernels it launches between them, all on the context's
 * stream, all asynchronous.  Pointers are device pointers unless named *_host. */

/* Local part of a mode-`mode` TTM of the block x (row-major, extents dims) with rows [l0, l0+dims[mode]) of the
 * replicated factor (factor: L_full x K column-major):  z(a,k,b) = sum_l F(l0+l, k) x(a,l,b), all K rows.  With
 * n_dest > 1 the K rows are split at dest_cuts[0..n_dest] and written destination-major, one contiguous chunk
 * (outer, rows_d, inner) per peer of the mode-`mode` process group — the send buffer of the reduce-scatter that the
 * paper's scheme needs exactly when the grid splits the contracted mode (grid_volume.hpp:41). */
int tp_dev_ttm_partial(tp_ctx* ctx, const double* x, int n_modes, const size_t* dims, int mode, const double* factor,
                       size_t L_full, size_t l0, size_t K, int n_dest, const size_t* dest_cuts, double* z);
/* Same product, scattered: chunk d (output rows dest_cuts[d]..dest_cuts[d+1], a contiguous (outer, rows_d, inner)
 * tensor) is written to dest_ptrs[d], which may be any device-accessible address -- in particular a receive slot in a
 * peer GPU's memory mapped over NVLink, so that the kernel's epilogue is the send of the reduce-scatter and no copy or
 * collective call follows (the receivers then add their slots in rank order with tp_dev_reduce_slots).  Entries of
 * empty chunks are ignored. */
int tp_dev_ttm_scatter(tp_ctx* ctx, const double* x, int n_modes, const size_t* dims, int mode, const double* factor,
                       size_t L_full, size_t l0, size_t K, int n_dest, const size_t* dest_cuts,
                       double* const* dest_ptrs);
/* out[i] = slots[0][i] + ... + slots[n_slots-1][i], i < count, summed in slot order (deterministic). */
int tp_dev_reduce_slots(tp_ctx* ctx, double* out, const double* const* slots_host, int n_slots, size_t count);
/* dst(a, l0+l, b) = src(a, l, b): places a peer's mode slice (outer, count, inner) into (outer, full_len, inner). */
int tp_dev_assemble_mode(tp_ctx* ctx, double* dst, size_t outer, size_t full_len, size_t inner, const double* src,
                         size_t l0, size_t count);
/* dst[dst_lo + i] = src[src_lo + i] for every index i of the box (extents `box`), both tensors row-major with extents
 * dst_dims / src_dims: one piece of a redistribution between two block layouts (the paper's regrid, PAPER.md:767;
 * counted by simulate.hpp:97-113).  src may be memory of a peer device. */
int tp_dev_copy_box(tp_ctx* ctx, double* dst, const size_t* dst_dims, const size_t* dst_lo, const double* src,
                    const size_t* src_dims, const size_t* src_lo, const size_t* box, int n_modes);
/* gram (rows x rows, full symmetric) of the mode-n unfolding of the block y viewed as (outer, rows, inner). */
int tp_dev_gram(tp_ctx* ctx, const double* y, size_t outer, size_t rows, size_t inner, double* gram);
/* top-k eigenvectors of gram (destroyed) with the reference's sign rule into factor (rows x k column-major);
 * *flag (device int) is OR-ed with the degenerate-gap flag; *info (device int) receives the solver status. */
int tp_dev_leaf_solve(tp_ctx* ctx, double* gram, size_t rows, int k, double* factor, int* flag, int* info);
/* Same, warm-started: `start` (rows x k column-major, e.g. the previous factor; may be NULL) seeds the certified top-k
 * subspace iteration (see TP_OPT_FAST_EVD); the certificate is checked before returning (one stream synchronisation)
 * and the full eigen-solve takes over when it fails.  gram is left intact by the fast path, destroyed by the fallback.
 * *used_fast (host, may be NULL) reports which path produced the factor. */
int tp_dev_leaf_solve_warm(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                           int* flag, int* info, int* used_fast);
/* Asynchronous pair for executors that overlap the leaf solves with the tree (the grid executor): _begin queues the
 * solve on side stream `lane` (0..3), ordered after everything queued on the context's stream so far, and returns;
 * _finish makes the context's stream wait for it, checks the top-k certificate (one stream synchronisation) and
 * falls back to the full solve on the intact Gram matrix.  gram, start, factor, flag and info must stay untouched
 * between the two calls; one solve in flight per lane. */
int tp_dev_leaf_solve_begin(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                            int* flag, int* info, int lane);
int tp_dev_leaf_solve_finish(tp_ctx* ctx, int lane, double* factor, int* flag, int* info, int* used_fast);
/* _begin with flags.  TP_LEAF_CONTINUE: when the lane's previous solve was of the same gram buffer and shape and was
 * accepted with its certificate, its Ritz vectors (all K_n + 8 of them) are the start block instead of `start` -- the
 * warm start of consecutive sweeps, as a resident plan does it.  The result then depends on the lane's history, which
 * is fine where one rank solves a leaf and shares the factor (the grid executor), not where replicas must agree bit
 * for bit. */
/* tp_dev_leaf_solve_reset forgets every lane's history (a new run: results again depend on the arguments only). */
enum { TP_LEAF_CONTINUE = 1 };
int tp_dev_leaf_solve_reset(tp_ctx* ctx);
int tp_dev_leaf_solve_begin_ex(tp_ctx* ctx, double* gram, size_t rows, int k, const double* start, double* factor,
                               int* flag, int* info, int lane, unsigned flags);
/* The whole certified top-k solve of a small leaf in ONE launch (csrc/leaf_solve_kernels.cu; what tp_plan_sweep uses
 * for leaves with rows <= 512 and k + 8 <= 64): power steps, Rayleigh-Ritz, certificate and the reference's selection
 * rules, rounds repeated on the device until the certificate holds.  All pointers are device pointers.  `start`:
 * rows x k column-major factor (start_is_ritz = 0) or the rows x (k + 8) ascending Ritz vectors a previous call left in
 * `ritz` (start_is_ritz = 1; may alias `ritz`).  Out: ritz rows x (k + 8), theta k + 8 (ascending), factor rows x k,
 * *flag |= degenerate, verdict[4] (verdict[0] == 0 && verdict[1] == 0: certified; [2] Jacobi sweeps, [3] power steps),
 * diag[16] ([0..3] worst residual / bound, angle bound, tail bound / theta_k, rounds; [4..11] SM cycles spent in the
 * kernel's phases: start block, G Q products, small Gram products, Cholesky, triangular solves, Jacobi, Ritz vectors +
 * residuals, certificate).  TP_ERR_BAD_ARGUMENT if the leaf is too large for this path. */
int tp_dev_leaf_solve_fused(tp_ctx* ctx, const double* gram, size_t rows, int k, const double* start,
                            int start_is_ritz, double* ritz, double* theta, double* factor, int* flag, int* verdict,
                            double* diag);
/* *out (device double) = sum x[i]^2 */
int tp_dev_sum_squares(tp_ctx* ctx, const double* x, size_t count, double* out);

/* Small dense steps of the certified top-k eigen-solve (the part of hooi.hpp:55 `SelfAdjointEigenSolver` this engine
 * replaces for the leaves); all pointers are device pointers, matrices column-major, block <= 112.
 *   tp_dev_cholesky      S (block x block, SPD, full storage) -> lower factor L, upper triangle zeroed;
 *                        *fail |= 1 if a pivot is not positive
 *   tp_dev_trsm_right_lt Z (rows x block) <- Z L^{-T}, in place
 *   tp_dev_jacobi_eig    H (block x block, symmetric, full storage) -> eigenvalues ascending in w, eigenvectors as
 *                        columns of v; fail[0] |= 2 if not converged, fail[1] = max(fail[1], sweeps used) */
int tp_dev_cholesky(tp_ctx* ctx, const double* s, int block, double* l, int* fail);
int tp_dev_trsm_right_lt(tp_ctx* ctx, double* z, size_t rows, int block, const double* l);
int tp_dev_jacobi_eig(tp_ctx* ctx, const double* h, int block, double* w, double* v, int* fail);

/* ------------------------------------------------------------ grid executor: HOOI on P GPUs of one box
 * The paper's distribution scheme executed inside ONE process ("single process driving P devices"):
 * rank p of the Cartesian grid lives on CUDA device devices[p]; tensors are block-distributed by floor cuts
 * (grid.hpp:114-119) with row-major owner ranks (simulate.hpp:69-73), factors replicated.  A product along a split
 * mode is followed by the reduce-scatter of PAPER.md:582-588, done here by the TTM kernel's epilogue storing every
 * chunk straight into its owner's memory over NVLink (peer access), an event, and an ordered sum; leaves add partial
 * Gram matrices at an owner rank, which solves and copies the factor to every replica; a node whose grid differs from
 * its parent's first redistributes its input (regrid).  The same device may be named more than once
 * ("virtual ranks" on one GPU: same code, peer pointers are ordinary pointers).  Jacobi schedule only.
 *   root_grid   n_modes extents, product = n_ranks, validated like validate_grid (grid.hpp:36-45)
 *   node_grids  NULL (the root grid everywhere = a static grid, grid_volume.hpp) or n_nodes x n_modes as in
 *               tp_scheme_volume (rows of TTM nodes are read), e.g. the output of tp_optimal_dynamic_scheme
 *   flags       TP_GRID_NCCL: leaf all-reduce and factor broadcast through NCCL (ncclCommInitAll; libnccl.so.2 is
 *               loaded at run time; needs distinct devices) instead of peer-memory reads and copies */
typedef struct tp_grid tp_grid;
enum { TP_GRID_NCCL = 1 };
int tp_grid_create(int n_ranks, const int* devices, int n_modes, const tp_u64* L, const tp_u64* K, int n_nodes,
                   const int* kind, const int* mode, const int* parent, const tp_u64* root_grid,
                   const tp_u64* node_grids, unsigned flags, tp_grid** out);
int tp_grid_destroy(tp_grid* grid);
int tp_grid_ranks(const tp_grid* grid, int* n_ranks);
/* rank's block of the input tensor under the root grid: first index and extent per mode (either may be NULL) */
int tp_grid_block(const tp_grid* grid, int rank, size_t* lo, size_t* dims);
/* the whole host tensor (row-major, extents L) cut into blocks and uploaded; or one rank's block, already cut */
int tp_grid_set_tensor(tp_grid* grid, const double* host_tensor);
int tp_grid_set_block(tp_grid* grid, int rank, const double* host_block);
/* Decomposition::factors (hooi.hpp:78-81), L_n x K_n column-major each; replicated to every rank */
int tp_grid_set_factors(tp_grid* grid, const double* const* factors);
int tp_grid_get_factors(tp_grid* grid, double* const* factors_out);
/* one hooi_sweep (hooi.hpp:189-229, SweepKind::jacobi) on the grid; the factors are replaced, the core recomputed */
int tp_grid_sweep(tp_grid* grid, tp_sweep_stats* stats);
/* the core (extents K, row-major) assembled from the ranks' blocks */
int tp_grid_get_core(tp_grid* grid, double* core_out);
int tp_grid_norms(tp_grid* grid, double* tensor_norm, double* core_norm);
int tp_grid_fit_from_norms(tp_grid* grid, double* out);
/* elements the ranks shipped in the last sweep, per tree node and summed over ranks: reduce-scatter of the node's
 * product and regrid of its input -- the quantities simulate.hpp traces and grid_volume.hpp / grid_dynamic.hpp
 * model (a product carried over from the previous core chain is booked to the sweep that consumes it) */
int tp_grid_last_volumes(const tp_grid* grid, int n_nodes, tp_u64* ttm_elements, tp_u64* regrid_elements);
/* device time of the last sweep, of each node's product (max over ranks; kernel + exchange + ordered sum), and the
 * number of leaves served by the certified top-k solve so far */
int tp_grid_last_timing(const tp_grid* grid, float* total_ms, int n_nodes, float* node_ms, int* fast_solves);
int tp_grid_launch_counts(const tp_grid* grid, tp_u64* own_kernels, tp_u64* library_calls);

/* By-value hooi_sweep (hooi.hpp:189-191): host tensor + host factors in, host factors + core out; uploads, runs,
 * downloads.  This is the call the reference-facing C++ wrapper makes. */
/* Consecutive calls with the same shape, ranks, tree and schedule reuse the device tensor, plan and workspaces kept
 * in the context (tp_ctx_release_cache frees them early; tp_ctx_destroy does too). */
int tp_ctx_release_cache(tp_ctx* ctx);
/* tp_hooi_sweep_host_ex flags.  TP_HOST_TENSOR_UNCHANGED: the caller promises that `tensor` (same address) still holds
 * what the previous call on this context uploaded; the device copy is then reused and only factors and core travel.
 * If in addition factors_in are bit for bit the factors that call returned, the sweep continues the resident run
 * (warm eigen-solves, carried products) exactly like a tp_plan_sweep loop.  A loop of by-value hooi_sweep calls on one
 * tensor -- the reference CLI's pattern, tools/tuckerplan_cli.cpp:416-419 -- therefore pays the upload once. */
enum { TP_HOST_TENSOR_UNCHANGED = 1 };
int tp_hooi_sweep_host_ex(tp_ctx* ctx, int n_modes, const size_t* dims, const double* tensor, const tp_u64* K,
                          const double* const* factors_in, int n_nodes, const int* kind, const int* mode,
                          const int* parent, int sweep_kind, unsigned flags, double* const* factors_out,
                          double* core_out, tp_sweep_stats* stats);
int tp_hooi_sweep_host(tp_ctx* ctx, int n_modes, const size_t* dims, const double* tensor, const tp_u64* K,
                       const double* const* factors_in, int n_nodes, const int* kind, const int* mode,
                       const int* parent, int sweep_kind, double* const* factors_out, double* core_out,
                       tp_sweep_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* TUCKERPLAN_B200_H */
