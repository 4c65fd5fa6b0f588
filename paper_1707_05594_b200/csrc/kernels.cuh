// Launchers of the hand-written sm_100a kernels (definitions in *_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>

namespace tpb {

// Kernel attributes (the opt-in for more than 48 KB of dynamic shared memory) and occupancy figures belong to one
// device's context, and one process may drive several devices (tp_ctx_create(device) per GPU, the grid executor):
// launchers cache them per device.  The slots are atomics because contexts on different host threads may launch the
// same kernel concurrently; a lost race only repeats an idempotent query.
constexpr int kMaxDevices = 64;
struct PerDeviceInt {
  std::atomic<int> value[kMaxDevices];
  // slot of the calling thread's current device (nullptr past kMaxDevices: callers then skip the cache)
  std::atomic<int>* slot() {
    int device = 0;
    if (cudaGetDevice(&device) != cudaSuccess || device < 0 || device >= kMaxDevices) return nullptr;
    return &value[device];
  }
};

// ---- mode-n TTM (ttm_kernels.cu) -------------------------------------------
struct TtmFragmentLayout {
  int kt = 1;        // 8-row output tiles per CTA (rows of the new mode handled per K block = 8 * kt)
  int k_blocks = 1;  // ceil(new_len / (8 kt))
  int kc = 16;       // contraction steps per pipeline stage
  int n_chunks = 1;  // ceil(len / kc)
  size_t layout_doubles = 0;  // one fragment-ordered copy
  size_t doubles = 0;         // the buffer: two copies (consecutive-row and interleaved-row k order)
};

int ttm_pick_kt(long long new_len);
TtmFragmentLayout ttm_fragment_layout(long long new_len, long long len);

// M(k, l) = m[k * row_stride + l * col_stride], k < new_len, l < len  ->  fragment order, zero padded.
cudaError_t prep_factor_fragments(cudaStream_t stream, const double* m, long long row_stride, long long col_stride,
                                  long long new_len, long long len, const TtmFragmentLayout& f, double* out);

constexpr int kMaxTtmDest = 16;
// Z(a,k,b) = sum_l M(k,l) X(a,l,b); x is (outer, len, inner) row-major, z is (outer, new_len, inner).
// With n_dest > 1 the output rows are split at dest_cuts[0..n_dest] (dest_cuts[0] = 0, dest_cuts[n_dest] = new_len)
// and written destination-major: chunk d is the contiguous tensor (outer, dest_cuts[d+1]-dest_cuts[d], inner).
// dest_offsets (optional, n_dest entries, in elements relative to z): where each chunk starts instead of the packed
// destination-major layout -- e.g. the distance to a peer GPU's receive slot, so that the stores go straight there.
cudaError_t launch_ttm(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                       const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z, int sm_count,
                       int n_dest = 1, const long long* dest_cuts = nullptr, const long long* dest_offsets = nullptr);

// Process-wide A/B switch: false forces the cp.async kernel even where the TMA pipeline is eligible.
std::atomic<bool>& ttm_tma_enabled();
// Few columns, contraction up to 512: one n-tile per CTA, the contraction split over its warps (ttm_splitk_kernels.cu).
// Eligibility is a function of the shape alone.
std::atomic<bool>& ttm_splitk_enabled();
bool ttm_splitk_eligible(long long outer, long long len, long long inner, int kt, int k_blocks, int n_dest);
cudaError_t launch_ttm_splitk(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                              const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z);
// Short trailing extents (1 < inner < 8): columns packed across slabs, contiguous slab chunks (ttm_packed_kernels.cu).
std::atomic<bool>& ttm_packed_enabled();
bool ttm_packed_eligible(const double* x, long long outer, long long len, long long inner, const double* z, int kt,
                         int n_dest);
cudaError_t launch_ttm_packed(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                              const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z,
                              int sm_count);

// Warp-specialised TMA variant (ttm_tma_kernels.cu): used by launch_ttm for 16-byte-aligned, even extents with enough
// columns to fill the machine.  mfrag must be the copy matching the mode (interleaved rows when inner > 1).
// The encoded 3-D tensor map (CUtensorMap*) of x viewed as (outer, len, inner) with 16 x 16 boxes and the 128-byte
// swizzle: dims (inner, len, outer), or (len, outer, 1) when inner == 1.  Cached per host thread; nullptr on failure.
const void* ttm_tensor_map(const double* x, long long outer, long long len, long long inner);
bool ttm_tma_eligible(const double* x, long long outer, long long len, long long inner, const double* z, int kt,
                      int k_blocks, int sm_count);
cudaError_t launch_ttm_tma(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                           const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z,
                           int sm_count, int n_dest, const long long* dest_cuts, const long long* dest_offsets = nullptr);

// ---- Gram of the mode-n unfolding, read in place (gram_kernels.cu) -----------
struct GramLayout {
  int tiles = 1;     // ceil(rows / 64); wide: ceil(rows / 128)
  int splits = 1;    // deterministic split of the column (contraction) range
  long long chunks = 0;
  size_t workspace_doubles = 0;  // splits * rows * rows (wide: enough for the narrow layout too)
  bool wide = false;  // 128 x 128 tiles on the TMA pipeline (gram_tma_kernels.cu), large leaves only
  int sm_count = 0;   // the SMs the layout was made for (wide: the persistent grid)
};
GramLayout gram_layout(long long outer, long long rows, long long inner, int sm_count);
// Process-wide A/B switch: false keeps large leaves on the 64 x 64 cp.async kernel.
std::atomic<bool>& gram_wide_enabled();
// SMs the wide kernel's persistent grid leaves free while eigen-solves are in flight beside it (plan walks only).
std::atomic<int>& gram_wide_spare_sms();
bool gram_wide_shape(long long outer, long long rows, long long inner);
GramLayout gram_wide_layout(long long outer, long long rows, long long inner, int sm_count);
// partial tiles only; launch_gram adds the ordered sum
cudaError_t launch_gram_wide(cudaStream_t stream, const double* y, long long outer, long long rows, long long inner,
                             const GramLayout& g, double* workspace, int sm_count);
// gram (rows x rows, full symmetric storage) = sum_{a,b} Y(a,:,b) Y(a,:,b)^T, y viewed as (outer, rows, inner).
cudaError_t launch_gram(cudaStream_t stream, const double* y, long long outer, long long rows, long long inner,
                        const GramLayout& g, double* workspace, double* gram);

// ---- small helpers (misc_kernels.cu) ------------------------------------------
// out[0] = sum x[i]^2 (deterministic two-level reduction); scratch needs reduce_scratch_doubles() entries.
size_t reduce_scratch_doubles();
cudaError_t launch_sum_squares(cudaStream_t stream, const double* x, size_t n, double* scratch, double* out);
cudaError_t launch_diff_sum_squares(cudaStream_t stream, const double* x, const double* y, size_t n, double* scratch,
                                    double* out);
// out[i] = slots[0][i] + slots[1][i] + ... in that order (the reduction half of a reduce-scatter; fixed order)
constexpr int kMaxReduceSlots = 16;
cudaError_t launch_reduce_slots(cudaStream_t stream, double* out, const double* const* slots, int n_slots, size_t n);
// End of a sweep (engine.cu jacobi_sequence): cur[m] <- fresh[m] for every mode, and the leaves' status words gathered
// into status_ints (8 per mode: verdict[0..3] where verdict[m] != null, flag, info) / status_doubles (4 per mode: the
// certificate margins); the degenerate flags are cleared.
constexpr int kMaxFinishModes = 16;  // TP_MAX_MODES
struct FinishSweepArgs {
  int n_modes = 0;
  double* cur[kMaxFinishModes];
  const double* fresh[kMaxFinishModes];
  size_t elems[kMaxFinishModes];
  const int* verdict[kMaxFinishModes];
  const double* diag[kMaxFinishModes];
  int* flag[kMaxFinishModes];
  const int* info[kMaxFinishModes];
  int* status_ints = nullptr;
  double* status_doubles = nullptr;
};
cudaError_t launch_finish_sweep(cudaStream_t stream, const FinishSweepArgs& args);
// dst(a, l0 + l, b) = src(a, l, b): drops the piece (outer, count, inner) into the tensor (outer, full_len, inner)
cudaError_t launch_assemble_mode(cudaStream_t stream, double* dst, long long outer, long long full_len,
                                 long long inner, const double* src, long long l0, long long count);
// dst[dst_lo + i] = src[src_lo + i] over an n-mode box (row-major tensors with extents dst_dims / src_dims): one piece
// of a redistribution between block layouts; src may be memory of a peer device
constexpr int kMaxBoxModes = 16;
cudaError_t launch_copy_box(cudaStream_t stream, double* dst, const long long* dst_dims, const long long* dst_lo,
                            const double* src, const long long* src_dims, const long long* src_lo,
                            const long long* box, int n);
// y[i] = beta * y[i] + alpha * x[i]
cudaError_t launch_axpby(cudaStream_t stream, double* y, double beta, double alpha, const double* x, size_t n);
// Top-k eigenvectors from an ascending eigen-solve result (vectors column-major rows x ncols, values w[ncols]) with
// the reference's sign rule and degenerate-gap flag (hooi.hpp:60-74).  factor is rows x k column-major; *flag is OR-ed.
cudaError_t launch_select_basis(cudaStream_t stream, const double* vectors, const double* w, int rows, int ncols,
                                int k, double* factor, int* flag);
// out[i] = deterministic pseudo-random value in [-0.5, 0.5)
cudaError_t launch_fill_pseudo_random(cudaStream_t stream, double* out, size_t n, unsigned long long salt);
// evd_kernels.cu: single-launch small dense steps of the top-k eigen-solve (block size b <= small_evd_max_block()).
size_t small_evd_max_block();
cudaError_t launch_cholesky(cudaStream_t stream, const double* s, int b, double* l, int* fail);         // S = L L^T
cudaError_t launch_trsm_right_lt(cudaStream_t stream, double* z, int n, int b, const double* l);        // Z <- Z L^-T
cudaError_t launch_jacobi_eig(cudaStream_t stream, const double* h, int b, double* w, double* v, int* fail);
cudaError_t launch_reverse_columns(cudaStream_t stream, double* dst, const double* src, int rows, int ncols);
// Certificate of the k largest of ncols ascending Ritz pairs (x orthonormal, zv = G x): residual bound, nothing larger
// missed (trace bound), subspace angle bound; see misc_kernels.cu.  verdict[0] |= 1 | 4; diag receives 4 margins.
cudaError_t launch_ritz_certificate(cudaStream_t stream, const double* gram, const double* zv, const double* x,
                                    const double* theta, int rows, int ncols, int k, double tol, double angle_tol,
                                    int* verdict, double* diag);


// leaf_solve_kernels.cu: the whole certified top-k solve of a small leaf (rows <= 512, block <= 64, see the file) in
// one launch.  start_mode 0: `start` holds rows x b ascending Ritz vectors of the previous solve; 1: a rows x k factor.
// ritz (rows x b) / theta (b) receive all Ritz pairs ascending, factor (rows x k) the reference's selection;
// verdict (4 ints) / diag (4 doubles) the certificate and its margins.
bool leaf_solve_fused_eligible(long long rows, int k, int b);
cudaError_t launch_leaf_solve_fused(cudaStream_t stream, const double* gram, int rows, int k, int b,
                                    const double* start, int start_mode, int first_steps, int max_rounds, double tol,
                                    double angle_tol, double* ritz, double* theta, double* factor, int* flag,
                                    int* verdict, double* diag);

}  // namespace tpb
