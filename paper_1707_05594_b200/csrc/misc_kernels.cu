// Small device helpers around the two hot kernels: deterministic norms and the
// eigenvector selection with the reference's sign / gap rules.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kReduceBlocks = 1184;  // 8 per SM on a 148-SM part
constexpr int kReduceThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_sums[kReduceThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
  __syncthreads();
  double total = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kReduceThreads / 32; ++w) total += warp_sums[w];
  return total;  // valid on thread 0
}

// Every block accumulates a fixed, index-determined subset, so the result does not depend on scheduling.
template <bool DIFF>
__global__ void __launch_bounds__(kReduceThreads) partial_sum_squares(const double* __restrict__ x,
                                                                       const double* __restrict__ y, size_t n,
                                                                       double* __restrict__ partial) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = DIFF ? x[i + u * stride] - y[i + u * stride] : x[i + u * stride];
      acc[u] = fma(v, v, acc[u]);
    }
  }
  for (; i < n; i += stride) {
    const double v = DIFF ? x[i] - y[i] : x[i];
    acc[0] = fma(v, v, acc[0]);
  }
  const double total = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kReduceThreads) final_sum(const double* __restrict__ partial, int n,
                                                            double* __restrict__ out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += kReduceThreads) v += partial[i];
  const double total = block_sum(v);
  if (threadIdx.x == 0) *out = total;
}

// One block per kept eigenvector j: column rows-1-j of the ascending eigenvector matrix, sign chosen so the
// largest-magnitude entry (first on ties) is positive (reference hooi.hpp:60-68).  Block 0 also evaluates the
// spectral-gap flag (hooi.hpp:70-74).
__global__ void __launch_bounds__(256) select_basis_kernel(const double* __restrict__ vectors,
                                                           const double* __restrict__ w, int rows, int ncols, int k,
                                                           double* __restrict__ factor, int* __restrict__ flag) {
  const int j = blockIdx.x;
  const double* col = vectors + static_cast<long long>(ncols - 1 - j) * rows;
  __shared__ double best_abs[256];
  __shared__ int best_idx[256];
  double ba = -1.0;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > ba) {  // strict: keeps the first index within this thread's ascending walk
      ba = a;
      bi = i;
    }
  }
  best_abs[threadIdx.x] = ba;
  best_idx[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double oa = best_abs[threadIdx.x + off];
      const int oi = best_idx[threadIdx.x + off];
      if (oa > best_abs[threadIdx.x] || (oa == best_abs[threadIdx.x] && oi < best_idx[threadIdx.x])) {
        best_abs[threadIdx.x] = oa;
        best_idx[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  // an all-NaN column (a failed iteration whose result the caller discards) leaves no index behind
  const double sign = (best_idx[0] < rows && col[best_idx[0]] < 0.0) ? -1.0 : 1.0;
  double* dst = factor + static_cast<long long>(j) * rows;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) dst[i] = sign * col[i];
  if (j == 0 && threadIdx.x == 0 && k < ncols) {
    const double top = fmax(w[ncols - 1], 0.0);
    const double gap = w[ncols - k] - w[ncols - 1 - k];
    if (gap <= 1e-10 * fmax(top, 1e-300)) atomicOr(flag, 1);
  }
}

__global__ void __launch_bounds__(256) axpby_kernel(double* __restrict__ y, double beta, double alpha,
                                                    const double* __restrict__ x, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    y[i] = fma(alpha, x[i], beta * y[i]);
}

// Deterministic filler for the oversampling columns of the subspace-iteration start block (splitmix64 hash of the
// element index; only the span matters and it is re-orthonormalised before use).
__global__ void __launch_bounds__(256) fill_pseudo_random_kernel(double* __restrict__ out, size_t n,
                                                                 unsigned long long salt) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull + salt;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

// dst[:, j] = src[:, ncols - 1 - j] (rows x ncols, column-major): ascending Ritz vectors -> dominant direction first.
__global__ void __launch_bounds__(256) reverse_columns_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                                              int rows, int ncols) {
  const size_t n = static_cast<size_t>(rows) * ncols;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const size_t col = i / rows, row = i - col * rows;
    dst[i] = src[(ncols - 1 - col) * static_cast<size_t>(rows) + row];
  }
}

// Certificate of a block of b Ritz pairs (ascending; X orthonormal, ZV = G X) for the k largest -- one CTA:
//   1. every kept pair has ||G x - theta x|| <= tol * theta_max;
//   2. nothing larger was missed: G is positive semidefinite, so an eigenvalue not matched by one of the b Ritz values
//      is at most tau = trace(G) - sum(theta) + b ||R||_F (Kahan: b eigenvalues lie within ||R||_2 of the Ritz values
//      of an orthonormal block); those matched by the oversampling pairs are at most theta_{k+1} + ||R||_F;
//      delta = theta_k - max(theta_{k+1} + ||R||_F, tau) must be positive;
//   3. the subspace angle bound ||R_kept||_F / delta (Davis-Kahan) is at most angle_tol.
// verdict[0] |= 1 (residual) | 4 (gap / angle); diag = {worst kept residual / (tol theta_max), ||R_kept||_F / delta,
// tau / theta_k, 0}.  Warps own columns, lanes stride the rows; all sums have a fixed order.
constexpr int kCertThreads = 1024;
constexpr int kCertMaxBlock = 1024;
__global__ void __launch_bounds__(kCertThreads) ritz_certificate_kernel(
    const double* __restrict__ gram, const double* __restrict__ zv, const double* __restrict__ x,
    const double* __restrict__ theta, int rows, int ncols, int k, double tol, double angle_tol,
    int* __restrict__ verdict, double* __restrict__ diag) {
  __shared__ double col_res[kCertMaxBlock];
  __shared__ double red[kCertThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = warp; c < ncols; c += kCertThreads / 32) {
    const double th = theta[c];
    const double* a = zv + static_cast<long long>(c) * rows;
    const double* b = x + static_cast<long long>(c) * rows;
    double acc = 0.0;
    for (int i = lane; i < rows; i += 32) {
      const double r = a[i] - th * b[i];
      acc = fma(r, r, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) col_res[c] = acc;
  }
  double part = 0.0;
  for (int i = tid; i < rows; i += kCertThreads) part += gram[static_cast<long long>(i) * rows + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  __syncthreads();
  if (tid != 0) return;
  double trace = 0.0;
  for (int w = 0; w < kCertThreads / 32; ++w) trace += red[w];
  const double top = fmax(fabs(theta[ncols - 1]), 1e-300);
  double sum_theta = 0.0, r_all2 = 0.0, r_kept2 = 0.0, worst = 0.0;
  for (int c = 0; c < ncols; ++c) {
    sum_theta += theta[c];
    r_all2 += col_res[c];
    if (c >= ncols - k) {
      r_kept2 += col_res[c];
      worst = fmax(worst, sqrt(col_res[c]));
    }
  }
  const double r_all = sqrt(r_all2), r_kept = sqrt(r_kept2);
  const double tau = fmax(trace - sum_theta, 0.0) + ncols * r_all;
  const double theta_k = theta[ncols - k];
  const double below = k < ncols ? fmax(theta[ncols - k - 1] + r_all, tau) : tau;
  const double delta = theta_k - below;
  int bits = 0;
  if (!(worst <= tol * top)) bits |= 1;
  if (!(delta > 0.0) || !(r_kept <= angle_tol * delta)) bits |= 4;
  if (bits) atomicOr(verdict, bits);
  diag[0] = worst / (tol * top);
  diag[1] = delta > 0.0 ? r_kept / delta : DBL_MAX;
  diag[2] = tau / fmax(theta_k, 1e-300);
  diag[3] = 0.0;
}

struct SlotList {
  const double* p[kMaxReduceSlots];
};

// End of a Jacobi sweep in one launch: every mode's new factor copied over the current one, and the leaves' status
// words gathered into one block the host reads with a single copy (8 ints per mode: verdict[0..3], degenerate flag,
// solver info; then 4 doubles per mode: the certificate margins); the degenerate flags are cleared for the next sweep.
__global__ void __launch_bounds__(256) finish_sweep_kernel(const FinishSweepArgs a) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t first = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (int m = 0; m < a.n_modes; ++m) {
    const double* __restrict__ src = a.fresh[m];
    double* __restrict__ dst = a.cur[m];
    for (size_t i = first; i < a.elems[m]; i += stride) dst[i] = src[i];
  }
  if (blockIdx.x == 0 && threadIdx.x < a.n_modes) {
    const int m = threadIdx.x;
    int* const si = a.status_ints + 8 * m;
    double* const sd = a.status_doubles + 4 * m;
    if (a.verdict[m]) {
      for (int i = 0; i < 4; ++i) si[i] = a.verdict[m][i];
      for (int i = 0; i < 4; ++i) sd[i] = a.diag[m][i];
    }
    if (a.flag[m]) {
      si[4] = *a.flag[m];
      si[5] = *a.info[m];
      *a.flag[m] = 0;
    }
  }
}

__global__ void __launch_bounds__(256) reduce_slots_kernel(double* __restrict__ out, SlotList slots, int n_slots,
                                                           size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    double sum = slots.p[0][i];
    for (int s = 1; s < n_slots; ++s) sum += slots.p[s][i];
    out[i] = sum;
  }
}

__global__ void __launch_bounds__(256) assemble_mode_kernel(double* __restrict__ dst, long long full_len,
                                                            long long inner, const double* __restrict__ src,
                                                            long long l0, long long count, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const long long piece = count * inner;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const long long a = static_cast<long long>(i) / piece;
    const long long r = static_cast<long long>(i) - a * piece;
    dst[(a * full_len + l0) * inner + r] = src[i];
  }
}

// dst[dst_lo + i] = src[src_lo + i] for every index i of an n-mode box; both tensors row-major with their own extents.
struct BoxCopy {
  int n;
  long long box[kMaxBoxModes];         // extents of the box
  long long src_stride[kMaxBoxModes];  // element strides of the source tensor
  long long dst_stride[kMaxBoxModes];
  long long src_base, dst_base;        // offsets of the box origin
};

__global__ void __launch_bounds__(256) copy_box_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                                       BoxCopy c, size_t total) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    long long rest = static_cast<long long>(i), s = c.src_base, d = c.dst_base;
    for (int m = c.n - 1; m >= 0; --m) {
      const long long at = rest % c.box[m];
      rest /= c.box[m];
      s += at * c.src_stride[m];
      d += at * c.dst_stride[m];
    }
    dst[d] = src[s];
  }
}

}  // namespace

cudaError_t launch_copy_box(cudaStream_t stream, double* dst, const long long* dst_dims, const long long* dst_lo,
                            const double* src, const long long* src_dims, const long long* src_lo,
                            const long long* box, int n) {
  if (n < 1 || n > kMaxBoxModes) return cudaErrorInvalidValue;
  BoxCopy c{};
  c.n = n;
  size_t total = 1;
  long long ss = 1, ds = 1;
  for (int m = n - 1; m >= 0; --m) {
    c.box[m] = box[m];
    c.src_stride[m] = ss;
    c.dst_stride[m] = ds;
    c.src_base += src_lo[m] * ss;
    c.dst_base += dst_lo[m] * ds;
    ss *= src_dims[m];
    ds *= dst_dims[m];
    total *= static_cast<size_t>(box[m]);
  }
  if (total == 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, kReduceBlocks));
  copy_box_kernel<<<blocks, 256, 0, stream>>>(dst, src, c, total);
  return cudaGetLastError();
}

cudaError_t launch_finish_sweep(cudaStream_t stream, const FinishSweepArgs& args) {
  if (args.n_modes < 1 || args.n_modes > kMaxFinishModes) return cudaErrorInvalidValue;
  size_t most = 0;
  for (int m = 0; m < args.n_modes; ++m) most = std::max(most, args.elems[m]);
  const unsigned blocks = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((most + 255) / 256, kReduceBlocks)));
  finish_sweep_kernel<<<blocks, 256, 0, stream>>>(args);
  return cudaGetLastError();
}

cudaError_t launch_reduce_slots(cudaStream_t stream, double* out, const double* const* slots, int n_slots, size_t n) {
  if (n_slots < 1 || n_slots > kMaxReduceSlots) return cudaErrorInvalidValue;
  SlotList list{};
  for (int s = 0; s < n_slots; ++s) list.p[s] = slots[s];
  reduce_slots_kernel<<<kReduceBlocks, 256, 0, stream>>>(out, list, n_slots, n);
  return cudaGetLastError();
}

cudaError_t launch_assemble_mode(cudaStream_t stream, double* dst, long long outer, long long full_len,
                                 long long inner, const double* src, long long l0, long long count) {
  const size_t n = static_cast<size_t>(outer) * count * inner;
  assemble_mode_kernel<<<kReduceBlocks, 256, 0, stream>>>(dst, full_len, inner, src, l0, count, n);
  return cudaGetLastError();
}

cudaError_t launch_axpby(cudaStream_t stream, double* y, double beta, double alpha, const double* x, size_t n) {
  axpby_kernel<<<kReduceBlocks, 256, 0, stream>>>(y, beta, alpha, x, n);
  return cudaGetLastError();
}

size_t reduce_scratch_doubles() { return kReduceBlocks; }

cudaError_t launch_sum_squares(cudaStream_t stream, const double* x, size_t n, double* scratch, double* out) {
  partial_sum_squares<false><<<kReduceBlocks, kReduceThreads, 0, stream>>>(x, nullptr, n, scratch);
  final_sum<<<1, kReduceThreads, 0, stream>>>(scratch, kReduceBlocks, out);
  return cudaGetLastError();
}

cudaError_t launch_diff_sum_squares(cudaStream_t stream, const double* x, const double* y, size_t n, double* scratch,
                                    double* out) {
  partial_sum_squares<true><<<kReduceBlocks, kReduceThreads, 0, stream>>>(x, y, n, scratch);
  final_sum<<<1, kReduceThreads, 0, stream>>>(scratch, kReduceBlocks, out);
  return cudaGetLastError();
}

cudaError_t launch_select_basis(cudaStream_t stream, const double* vectors, const double* w, int rows, int ncols,
                                int k, double* factor, int* flag) {
  select_basis_kernel<<<k, 256, 0, stream>>>(vectors, w, rows, ncols, k, factor, flag);
  return cudaGetLastError();
}

cudaError_t launch_reverse_columns(cudaStream_t stream, double* dst, const double* src, int rows, int ncols) {
  const size_t n = static_cast<size_t>(rows) * ncols;
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, kReduceBlocks));
  reverse_columns_kernel<<<std::max(blocks, 1), 256, 0, stream>>>(dst, src, rows, ncols);
  return cudaGetLastError();
}

cudaError_t launch_fill_pseudo_random(cudaStream_t stream, double* out, size_t n, unsigned long long salt) {
  fill_pseudo_random_kernel<<<kReduceBlocks, 256, 0, stream>>>(out, n, salt);
  return cudaGetLastError();
}

cudaError_t launch_ritz_certificate(cudaStream_t stream, const double* gram, const double* zv, const double* x,
                                    const double* theta, int rows, int ncols, int k, double tol, double angle_tol,
                                    int* verdict, double* diag) {
  if (ncols > kCertMaxBlock || k < 1 || k > ncols) return cudaErrorInvalidValue;
  ritz_certificate_kernel<<<1, kCertThreads, 0, stream>>>(gram, zv, x, theta, rows, ncols, k, tol, angle_tol, verdict,
                                                          diag);
  return cudaGetLastError();
}

}  // namespace tpb
