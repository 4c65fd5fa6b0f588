// Launchers of the hand-written sm_100a kernels (definitions in *_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace tpb {

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

// Warp-specialised TMA variant (ttm_tma_kernels.cu): used by launch_ttm for 16-byte-aligned, even extents with enough
// columns to fill the machine.  mfrag must be the copy matching the mode (interleaved rows when inner > 1).
bool ttm_tma_eligible(const double* x, long long outer, long long len, long long inner, const double* z, int kt,
                      int k_blocks, int sm_count);
cudaError_t launch_ttm_tma(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                           const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z,
                           int sm_count, int n_dest, const long long* dest_cuts, const long long* dest_offsets = nullptr);

// ---- Gram of the mode-n unfolding, read in place (gram_kernels.cu) -----------
struct GramLayout {
  int tiles = 1;     // ceil(rows / 64)
  int splits = 1;    // deterministic split of the column (contraction) range
  long long chunks = 0;
  size_t workspace_doubles = 0;  // splits * rows * rows
};
GramLayout gram_layout(long long outer, long long rows, long long inner, int sm_count);
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
// dst(a, l0 + l, b) = src(a, l, b): drops the piece (outer, count, inner) into the tensor (outer, full_len, inner)
cudaError_t launch_assemble_mode(cudaStream_t stream, double* dst, long long outer, long long full_len,
                                 long long inner, const double* src, long long l0, long long count);
// y[i] = beta * y[i] + alpha * x[i]
cudaError_t launch_axpby(cudaStream_t stream, double* y, double beta, double alpha, const double* x, size_t n);
// Top-k eigenvectors from an ascending eigen-solve result (vectors column-major rows x ncols, values w[ncols]) with
// the reference's sign rule and degenerate-gap flag (hooi.hpp:60-74).  factor is rows x k column-major; *flag is OR-ed.
cudaError_t launch_select_basis(cudaStream_t stream, const double* vectors, const double* w, int rows, int ncols,
                                int k, double* factor, int* flag);
// out[i] = deterministic pseudo-random value in [-0.5, 0.5)
cudaError_t launch_fill_pseudo_random(cudaStream_t stream, double* out, size_t n, unsigned long long salt);
// *verdict |= 1 unless every one of the k largest Ritz pairs has ||(ZV)_j - theta_j X_j|| <= tol * theta_max
// evd_kernels.cu: single-launch small dense steps of the top-k eigen-solve (block size b <= small_evd_max_block()).
size_t small_evd_max_block();
cudaError_t launch_cholesky(cudaStream_t stream, const double* s, int b, double* l, int* fail);         // S = L L^T
cudaError_t launch_trsm_right_lt(cudaStream_t stream, double* z, int n, int b, const double* l);        // Z <- Z L^-T
cudaError_t launch_jacobi_eig(cudaStream_t stream, const double* h, int b, double* w, double* v, int* fail);
cudaError_t launch_reverse_columns(cudaStream_t stream, double* dst, const double* src, int rows, int ncols);
cudaError_t launch_ritz_residuals(cudaStream_t stream, const double* zv, const double* x, const double* theta,
                                  int rows, int ncols, int k, double tol, int* verdict);

}  // namespace tpb
