// Small dense building blocks of the top-k eigen-solve (engine.cu: leaf_solve_subspace).  The block subspace
// iteration needs, besides GEMM-shaped products (cuBLAS), three latency-bound operations on tiny matrices that the
// vendor libraries serve with dozens of launches each: a b x b Cholesky factorisation, the triangular solve that
// turns Z into an orthonormal basis, and the eigen-decomposition of the b x b Rayleigh-Ritz matrix (b = K_n + 8).
// Each is one launch here, so a leaf's whole iteration is a short, fixed kernel sequence that the engine replays as
// a CUDA graph.  All kernels are deterministic.
#include <cuda_runtime.h>

#include <cfloat>

#include "evd_device.cuh"
#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kMaxBlock = kEvdMaxBlock;  // largest iteration block: 2 b^2 doubles of shared memory must fit in 227 KB
constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;

// L L^T = S for the symmetric positive definite b x b matrix S (column-major, full storage).  Single CTA, S lives in
// shared memory; warps own trailing columns, lanes rows.  The trailing update works on the unscaled column,
// S(i,k) -= S(i,j) S(k,j) / d_j, so a step needs one barrier; the columns are scaled by 1/sqrt(d_j) on the way out.
// *fail |= 1 when a pivot is not positive (rank-deficient iteration block -> the caller falls back to the full
// eigen-solve).
template <int kBlockCap>
__global__ void __launch_bounds__(kSmallThreads) cholesky_kernel(const double* __restrict__ s_in, int b,
                                                                 double* __restrict__ l_out, int* __restrict__ fail) {
  extern __shared__ double sm[];  // b x b, column-major
  __shared__ double pivot[kMaxBlock];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < b * b; e += kSmallThreads) sm[e] = s_in[e];
  for (int e = tid; e < kMaxBlock; e += kSmallThreads) pivot[e] = 1.0;
  __syncthreads();
  bool bad = false;
  for (int j = 0; j < b; ++j) {
    const double d = sm[j * b + j];  // final since the previous step's barrier; nobody writes it again
    if (!(d > 0.0)) {                // uniform: every thread reads the same value
      bad = true;
      break;
    }
    if (tid == 0) pivot[j] = sqrt(d);
    const double dinv = 1.0 / d;
    // this lane's rows of column j, shared by every trailing column the warp updates (as many 32-row passes as the
    // block-size class needs)
    constexpr int kPasses = (kBlockCap + 31) / 32;
    double cj[kPasses];
#pragma unroll
    for (int r = 0; r < kPasses; ++r) {
      const int i = lane + 32 * r;
      cj[r] = (i > j && i < b) ? sm[j * b + i] : 0.0;
    }
    for (int k = j + 1 + warp; k < b; k += kSmallWarps) {
      const double skj = sm[j * b + k] * dinv;
      double v[kPasses];
#pragma unroll
      for (int r = 0; r < kPasses; ++r) {
        const int i = lane + 32 * r;
        v[r] = (i >= k && i < b) ? sm[k * b + i] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < kPasses; ++r) {
        const int i = lane + 32 * r;
        if (i >= k && i < b) sm[k * b + i] = fma(-cj[r], skj, v[r]);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(fail, 1);
  for (int col = warp; col < b; col += kSmallWarps) {
    const double piv = pivot[col];
    for (int row = lane; row < b; row += 32)
      l_out[col * b + row] = row > col ? sm[col * b + row] / piv : (row == col ? piv : 0.0);
  }
}

// The same factorisation for blocks of at most 64 by ONE warp in registers (evd_device.cuh: panels of eight columns,
// shuffles along the dependent chain, the trailing update on the FP64 tensor pipe): no CTA barrier per column.
template <int kCap>
__global__ void __launch_bounds__(kSmallThreads) cholesky_panel_kernel(const double* __restrict__ s_in, int b,
                                                                       double* __restrict__ l_out,
                                                                       int* __restrict__ fail) {
  extern __shared__ __align__(16) double sm[];  // m x m (+ a fragment's reach past the last column), then 1 / L(j, j)
  const int m = (b + 1) & ~1;
  double* const invd = sm + m * m + 8 * m;
  const int tid = threadIdx.x;
  for (int e = tid; e < m * m; e += kSmallThreads) {
    const int col = e / m, row = e - col * m;
    sm[e] = (col < b && row < b) ? s_in[col * b + row] : 0.0;
  }
  const bool ok = cholesky_warp<kCap>(sm, invd, b, m, 0.0);
  if (tid == 0 && !ok) atomicOr(fail, 1);
  for (int e = tid; e < b * b; e += kSmallThreads) {
    const int col = e / b, row = e - col * b;
    l_out[e] = row >= col ? sm[col * m + row] : 0.0;
  }
}

// Z <- Z L^{-T} for blocks of at most 64 columns: trsm_rows_blocked of evd_device.cuh, 128 rows per CTA (a warp owns 32
// rows for the whole solve; the trailing column blocks take their update on the FP64 tensor pipe).
constexpr int kTrsmBlockedThreads = 128;
__global__ void __launch_bounds__(kTrsmBlockedThreads) trsm_blocked_kernel(double* __restrict__ z, int n, int b,
                                                                           const double* __restrict__ l) {
  extern __shared__ __align__(16) double sm[];  // L: m x m (+ a fragment's reach), then 1 / L(j, j)
  const int m = (b + 1) & ~1;
  double* const invd = sm + m * m + 8 * m;
  const int tid = threadIdx.x;
  for (int e = tid; e < m * m + 8 * m; e += kTrsmBlockedThreads) {
    const int col = e / m, row = e - col * m;
    sm[e] = (col < b && row < b) ? l[col * b + row] : 0.0;
  }
  for (int j = tid; j < b; j += kTrsmBlockedThreads) invd[j] = 1.0 / l[j * b + j];
  __syncthreads();
  const int row0 = blockIdx.x * kTrsmBlockedThreads;
  trsm_rows_blocked(z + row0, sm, invd, n - row0, b, n, m);
}

// Z <- Z L^{-T} (Z: n x b column-major, in place): every row x solves x L^T = z.  A row is spread over 8 lanes, lane
// l keeping columns l, l + 8, ... in registers; column j is finished by its owner (x_j = z_j / L_jj), broadcast by
// one shuffle, and eliminated from the columns to its right by all 8 lanes at once (independent FMAs, no reduction).
// A warp serves 4 rows, a CTA 32.
constexpr int kTrsmThreads = 256;
constexpr int kTrsmRows = kTrsmThreads / 8;
// kTrsmSlots = columns a lane keeps = block-size class / 8; the loops below are fully unrolled over it, so small
// blocks get a small kernel (the 112-column instance alone is ~1600 predicated FMAs of straight-line code)
template <int kTrsmSlots>
__global__ void __launch_bounds__(kTrsmThreads) trsm_right_lt_kernel(double* __restrict__ z, int n, int b,
                                                                     const double* __restrict__ l) {
  extern __shared__ double ls[];  // b x b, column-major lower
  const int tid = threadIdx.x, lane = tid & 31;
  const int sub = lane & 7;  // which columns of the row this lane keeps
  const int row = blockIdx.x * kTrsmRows + (tid >> 5) * 4 + (lane >> 3);
  for (int e = tid; e < b * b; e += kTrsmThreads) ls[e] = l[e];
  double x[kTrsmSlots];
  const bool live = row < n;
#pragma unroll
  for (int m = 0; m < kTrsmSlots; ++m) {
    const int col = sub + 8 * m;
    x[m] = (live && col < b) ? z[static_cast<long long>(col) * n + row] : 0.0;
  }
  __syncthreads();
  const unsigned group_base = lane & ~7u;
#pragma unroll
  for (int mj = 0; mj < kTrsmSlots; ++mj) {
    if (8 * mj >= b) break;  // uniform
#pragma unroll
    for (int lj = 0; lj < 8; ++lj) {
      const int j = 8 * mj + lj;
      if (j >= b) break;  // uniform
      if (sub == lj) x[mj] /= ls[j * b + j];
      const double xj = __shfl_sync(0xffffffffu, x[mj], group_base | lj);
#pragma unroll
      for (int m = mj; m < kTrsmSlots; ++m) {
        const int i = sub + 8 * m;  // column to the right of j kept by this lane
        if (i > j && i < b) x[m] = fma(-xj, ls[j * b + i], x[m]);
      }
    }
  }
  if (live) {
#pragma unroll
    for (int m = 0; m < kTrsmSlots; ++m) {
      const int col = sub + 8 * m;
      if (col < b) z[static_cast<long long>(col) * n + row] = x[m];
    }
  }
}

// Eigen-decomposition of the symmetric b x b matrix H by the parallel cyclic Jacobi method: the sweep loop lives in
// evd_device.cuh (jacobi_sweeps_smem), shared with the single-launch leaf solve (leaf_solve_kernels.cu).  Single CTA;
// H and the accumulated rotations V live in shared memory (leading dimension m = b rounded up to even: the odd case
// plays against an all-zero dummy index that is never rotated).  Output: eigenvalues ascending in w, matching
// eigenvectors as columns of v_out (b x b column-major).
// *fail |= 2 if the off-diagonal mass has not vanished after kMaxSweeps sweeps; fail[1] = max(fail[1], sweeps used).
// Instantiated per block-size class: (512 threads, b <= 32) and (512, b <= 64) run the one-barrier iteration with
// fixed pair positions (jacobi_pingpong_smem: H and V twice in shared memory); (512, b <= 112) the two-barrier one in
// place (shared-memory-bandwidth-bound, the batched loads want the registers).
template <int kJacobiThreads, int kBlockCap>
__global__ void __launch_bounds__(kJacobiThreads) jacobi_eig_kernel(const double* __restrict__ h_in, int b,
                                                                   double* __restrict__ w, double* __restrict__ v_out,
                                                                   int* __restrict__ fail) {
  extern __shared__ __align__(16) double sm[];
  const int m = (b + 1) & ~1;
  double* const h = sm;          // m x m
  double* const v = sm + m * m;  // m x m
  constexpr int kJacobiWarps = kJacobiThreads / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double unscale = 1.0;
  int sweep;
  if constexpr (kBlockCap <= 64) {
    // the one-barrier iteration (evd_device.cuh) wants entries of order one: scale by a power of two (exact)
    __shared__ double wmax[kJacobiWarps];
    double top = 0.0;
    for (int e = tid; e < b * b; e += kJacobiThreads) top = fmax(top, fabs(h_in[e]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = fmax(top, __shfl_xor_sync(0xffffffffu, top, o));
    if (lane == 0) wmax[warp] = top;
    __syncthreads();
    for (int i = 0; i < kJacobiWarps; ++i) top = fmax(top, wmax[i]);
    double scale = 1.0;
    const int ex = (__double2hiint(top) >> 20) & 0x7ff;
    if (ex >= 64 && ex <= 1982) {
      scale = __hiloint2double((2046 - ex) << 20, 0);
      unscale = __hiloint2double(ex << 20, 0);
    }
    for (int col = warp; col < m; col += kJacobiWarps)
      for (int row = lane; row < m; row += 32) {
        h[col * m + row] = (col < b && row < b) ? h_in[col * b + row] * scale : 0.0;
        v[col * m + row] = (col == row) ? 1.0 : 0.0;
      }
    __syncthreads();
    sweep = jacobi_pingpong_smem<kJacobiThreads, kBlockCap, kJacobiWarps>(h, v + m * m, v, v + 2 * m * m, b, m);
  } else {
    for (int col = warp; col < m; col += kJacobiWarps)
      for (int row = lane; row < m; row += 32) {
        h[col * m + row] = (col < b && row < b) ? h_in[col * b + row] : 0.0;
        v[col * m + row] = (col == row) ? 1.0 : 0.0;
      }
    __syncthreads();
    sweep = jacobi_sweeps_smem<kJacobiThreads, kBlockCap>(h, v, b, m);
  }
  if (tid == 0) {
    if (sweep == kJacobiMaxSweeps) atomicOr(fail, 2);
    atomicMax(fail + 1, sweep);
  }
  // ascending order by rank (ties by index); eigenvectors follow their values
  for (int i = warp; i < b; i += kJacobiWarps) {
    const double li = h[i * m + i] * unscale;
    int rank = 0;
    for (int j = lane; j < b; j += 32) {
      const double lj = h[j * m + j] * unscale;
      rank += (lj < li) || (lj == li && j < i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) w[rank] = li;
    for (int r = lane; r < b; r += 32) v_out[rank * b + r] = v[i * m + r];
  }
}

template <typename Kernel>
cudaError_t allow_shared(Kernel kernel, size_t bytes, PerDeviceInt& configured) {
  std::atomic<int>* const slot = configured.slot();
  if (slot && slot->load(std::memory_order_relaxed)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess && slot) slot->store(1, std::memory_order_relaxed);
  return e;
}

}  // namespace

size_t small_evd_max_block() { return kMaxBlock; }

cudaError_t launch_cholesky(cudaStream_t stream, const double* s, int b, double* l, int* fail) {
  static PerDeviceInt configured[3];
  const size_t smem = sizeof(double) * b * b;
  cudaError_t e;
  const int m = (b + 1) & ~1;
  const size_t panel_smem = sizeof(double) * (static_cast<size_t>(m) * m + 9 * m);
  if (b <= 32) {
    e = allow_shared(cholesky_panel_kernel<32>, sizeof(double) * (32 * 32 + 9 * 32), configured[0]);
    if (e != cudaSuccess) return e;
    cholesky_panel_kernel<32><<<1, kSmallThreads, panel_smem, stream>>>(s, b, l, fail);
  } else if (b <= 64) {
    e = allow_shared(cholesky_panel_kernel<64>, sizeof(double) * (64 * 64 + 9 * 64), configured[1]);
    if (e != cudaSuccess) return e;
    cholesky_panel_kernel<64><<<1, kSmallThreads, panel_smem, stream>>>(s, b, l, fail);
  } else {
    e = allow_shared(cholesky_kernel<kMaxBlock>, sizeof(double) * kMaxBlock * kMaxBlock, configured[2]);
    if (e != cudaSuccess) return e;
    cholesky_kernel<kMaxBlock><<<1, kSmallThreads, smem, stream>>>(s, b, l, fail);
  }
  return cudaGetLastError();
}

cudaError_t launch_trsm_right_lt(cudaStream_t stream, double* z, int n, int b, const double* l) {
  static PerDeviceInt configured[2];
  cudaError_t e;
  if (b <= 64) {
    const int m = (b + 1) & ~1;
    const size_t smem = sizeof(double) * (static_cast<size_t>(m) * m + 9 * m);
    e = allow_shared(trsm_blocked_kernel, sizeof(double) * (64 * 64 + 9 * 64), configured[0]);
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>((n + kTrsmBlockedThreads - 1) / kTrsmBlockedThreads);
    trsm_blocked_kernel<<<grid, kTrsmBlockedThreads, smem, stream>>>(z, n, b, l);
  } else {
    const size_t smem = sizeof(double) * b * b;
    const unsigned grid = static_cast<unsigned>((n + kTrsmRows - 1) / kTrsmRows);
    e = allow_shared(trsm_right_lt_kernel<kMaxBlock / 8>, sizeof(double) * kMaxBlock * kMaxBlock, configured[1]);
    if (e != cudaSuccess) return e;
    trsm_right_lt_kernel<kMaxBlock / 8><<<grid, kTrsmThreads, smem, stream>>>(z, n, b, l);
  }
  return cudaGetLastError();
}

cudaError_t launch_jacobi_eig(cudaStream_t stream, const double* h, int b, double* w, double* v, int* fail) {
  static PerDeviceInt configured[3];
  const int m = (b + 1) & ~1;
  // blocks of at most 64: H and V twice (the one-barrier iteration writes each step into a second buffer)
  const size_t smem = sizeof(double) * (b <= 64 ? 4 : 2) * m * m;
  cudaError_t e;
  if (b <= 32) {
    e = allow_shared(jacobi_eig_kernel<512, 32>, sizeof(double) * 4 * 32 * 32, configured[0]);
    if (e != cudaSuccess) return e;
    jacobi_eig_kernel<512, 32><<<1, 512, smem, stream>>>(h, b, w, v, fail);
  } else if (b <= 64) {
    e = allow_shared(jacobi_eig_kernel<512, 64>, sizeof(double) * 4 * 64 * 64, configured[1]);
    if (e != cudaSuccess) return e;
    jacobi_eig_kernel<512, 64><<<1, 512, smem, stream>>>(h, b, w, v, fail);
  } else {
    e = allow_shared(jacobi_eig_kernel<512, kMaxBlock>, sizeof(double) * 2 * kMaxBlock * kMaxBlock, configured[2]);
    if (e != cudaSuccess) return e;
    jacobi_eig_kernel<512, kMaxBlock><<<1, 512, smem, stream>>>(h, b, w, v, fail);
  }
  return cudaGetLastError();
}

}  // namespace tpb
