// Mode-n tensor-times-matrix on the strided unfolding, FP64 tensor cores.
//
//   Z(a, k, b) = sum_l M(k, l) * X(a, l, b)        X viewed as (outer, L, inner), row-major
//
// replaces the reference's slab-wise Eigen GEMM loop (reference ttm.hpp:73-96)
// with one launch that never materialises an unfolding:
//
//   * the contraction runs on DMMA.8x8x4 (mma.sync m8n8k4 f64 — the only FP64
//     tensor-core shape sm_100a executes natively; tcgen05 has no f64 kind).
//     M is the MMA A operand (rows k), an 8-column strip of X the B operand.
//   * columns are grouped into "n-tiles" of 8: for inner > 1 eight consecutive
//     b of one slab a (contiguous in memory), for inner == 1 eight consecutive
//     slabs a (the contraction index is then the contiguous one).
//   * a CTA owns WARPS*NT consecutive n-tiles and all 8*KT rows of one K block;
//     X chunks of KC contraction steps stream through a STAGES-deep cp.async
//     ring in shared memory, XOR-swizzled so that the 64-bit fragment loads of a
//     half-warp hit 16 distinct bank pairs; the factor streams beside it in
//     "fragment order" (prepared once per factor by prep_factor_fragments), so
//     an A fragment is one conflict-free LDS.64 per lane and needs no bounds
//     checks (padding rows/columns are stored as zeros).
//   * every element of X is read from HBM exactly once per K block and every
//     element of Z written once; accumulation order is fixed (deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace tpb {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct TtmParams {
  const double* __restrict__ x;
  double* __restrict__ z;
  const double* __restrict__ mfrag;  // [k blocks][chunks][KC/4][KT][32]
  long long outer, len, inner, new_len;
  long long n_tiles;  // total 8-column tiles
  int tiles_per_slab; // ceil(inner / 8), inner > 1 only
  int n_chunks;       // ceil(len / KC)
  int vec;            // 16-byte global accesses are aligned and never straddle an extent
};

// One CTA: rows [kb*8*KT, +8*KT) of the output mode, n-tiles [blockIdx.x*TILE_N, +TILE_N).
template <int KT, int NT, int KC, int STAGES, bool LAST>
__global__ void __launch_bounds__(kThreads, (KT * NT <= 20) ? 2 : 1) ttm_dmma_kernel(const TtmParams p) {
  constexpr int TILE_N = kWarps * NT;
  constexpr int XS = TILE_N * KC * 8;     // doubles per stage of X
  constexpr int MS = (KC / 4) * KT * 32;  // doubles per stage of factor fragments
  static_assert((TILE_N & (TILE_N - 1)) == 0, "TILE_N must be a power of two");
  static_assert(KC % 16 == 0, "swizzle assumes 16-double rows");

  extern __shared__ __align__(16) double smem[];
  double* const xs = smem;
  double* const ms = smem + STAGES * XS;
  __shared__ long long tile_base[TILE_N];
  __shared__ int tile_lim[TILE_N];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = blockIdx.y;
  const long long tile0 = static_cast<long long>(blockIdx.x) * TILE_N;

  if (tid < TILE_N) {
    const long long g = tile0 + tid;
    long long base = 0;
    int lim = 0;
    if (g < p.n_tiles) {
      if (LAST) {
        base = g * 8 * p.len;
        lim = static_cast<int>(min(8LL, p.outer - g * 8));
      } else {
        const long long a = g / p.tiles_per_slab;
        const long long b0 = (g - a * p.tiles_per_slab) * 8;
        base = a * p.len * p.inner + b0;
        lim = static_cast<int>(min(8LL, p.inner - b0));
      }
    }
    tile_base[tid] = base;
    tile_lim[tid] = lim;
  }
  __syncthreads();

  const double* const mfrag_kb = p.mfrag + static_cast<long long>(kb) * p.n_chunks * MS;

  auto issue_chunk = [&](int chunk, int stage) {
    double* const xd = xs + stage * XS;
    const long long l0 = static_cast<long long>(chunk) * KC;
    if (!LAST) {
      if (p.vec) {
#pragma unroll 2
        for (int idx = tid; idx < TILE_N * KC * 4; idx += kThreads) {
          const int c = idx & 3, t = (idx >> 2) & (TILE_N - 1), l = idx / (4 * TILE_N);
          const bool ok = (l0 + l < p.len) && (2 * c < tile_lim[t]);
          const double* src = ok ? p.x + tile_base[t] + (l0 + l) * p.inner + 2 * c : p.x;
          cp_async16(xd + t * (KC * 8) + l * 8 + ((2 * c) ^ (((l >> 1) & 1) << 2)), src, ok);
        }
      } else {
        for (int idx = tid; idx < TILE_N * KC * 8; idx += kThreads) {
          const int b = idx & 7, t = (idx >> 3) & (TILE_N - 1), l = idx / (8 * TILE_N);
          const bool ok = (l0 + l < p.len) && (b < tile_lim[t]);
          const double* src = ok ? p.x + tile_base[t] + (l0 + l) * p.inner + b : p.x;
          cp_async8(xd + t * (KC * 8) + l * 8 + (b ^ (((l >> 1) & 1) << 2)), src, ok);
        }
      }
    } else {
      if (p.vec) {
#pragma unroll 2
        for (int idx = tid; idx < TILE_N * 8 * (KC / 2); idx += kThreads) {
          const int c = idx % (KC / 2), r = (idx / (KC / 2)) & 7, t = idx / (4 * KC);
          const bool ok = (r < tile_lim[t]) && (l0 + 2 * c < p.len);
          const double* src = ok ? p.x + tile_base[t] + r * p.len + l0 + 2 * c : p.x;
          cp_async16(xd + t * (8 * KC) + r * KC + ((2 * c) ^ ((r & 3) << 2)), src, ok);
        }
      } else {
        for (int idx = tid; idx < TILE_N * 8 * KC; idx += kThreads) {
          const int l = idx % KC, r = (idx / KC) & 7, t = idx / (8 * KC);
          const bool ok = (r < tile_lim[t]) && (l0 + l < p.len);
          const double* src = ok ? p.x + tile_base[t] + r * p.len + l0 + l : p.x;
          cp_async8(xd + t * (8 * KC) + r * KC + (l ^ ((r & 3) << 2)), src, ok);
        }
      }
    }
    const double* msrc = mfrag_kb + static_cast<long long>(chunk) * MS;
    double* const md = ms + stage * MS;
    for (int idx = tid; idx < MS / 2; idx += kThreads) cp_async16(md + 2 * idx, msrc + 2 * idx, true);
  };

  double acc[KT][NT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < p.n_chunks) issue_chunk(s, s);
    cp_async_commit();
  }

  const int frag_k = lane & 3, frag_n = lane >> 2;
  for (int chunk = 0; chunk < p.n_chunks; ++chunk) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int next = chunk + STAGES - 1;
      if (next < p.n_chunks) issue_chunk(next, next % STAGES);
      cp_async_commit();
    }
    const double* const xd = xs + (chunk % STAGES) * XS + (warp * NT) * (KC * 8);
    const double* const md = ms + (chunk % STAGES) * MS + lane;
#pragma unroll
    for (int s = 0; s < KC / 4; ++s) {
      double a[KT];
#pragma unroll
      for (int i = 0; i < KT; ++i) a[i] = md[(s * KT + i) * 32];
      const int l = 4 * s + frag_k;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        double b;
        if (LAST)
          b = xd[j * (KC * 8) + frag_n * KC + (l ^ ((frag_n & 3) << 2))];
        else
          b = xd[j * (KC * 8) + l * 8 + (frag_n ^ (((l >> 1) & 1) << 2))];
#pragma unroll
        for (int i = 0; i < KT; ++i) dmma884(acc[i][j][0], acc[i][j][1], a[i], b);
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue: lane holds rows k = 8 i + lane/4 and columns 2 (lane%4), 2 (lane%4) + 1 of each of its n-tiles.
  const int col = 2 * (lane & 3);
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = warp * NT + j;
    const int lim = tile_lim[t];
    if (lim == 0) continue;
    const long long g = tile0 + t;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      const long long k = static_cast<long long>(kb) * (8 * KT) + 8 * i + (lane >> 2);
      if (k >= p.new_len) continue;
      if (LAST) {
        const long long a = g * 8 + col;
        if (col < lim) p.z[a * p.new_len + k] = acc[i][j][0];
        if (col + 1 < lim) p.z[(a + 1) * p.new_len + k] = acc[i][j][1];
      } else {
        const long long a = g / p.tiles_per_slab;
        const long long b = (g - a * p.tiles_per_slab) * 8 + col;
        double* dst = p.z + (a * p.new_len + k) * p.inner + b;
        if (p.vec) {
          if (col < lim) *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (col < lim) dst[0] = acc[i][j][0];
          if (col + 1 < lim) dst[1] = acc[i][j][1];
        }
      }
    }
  }
}

// factor (rows new_len x cols len, element (k,l) at m[k*row_stride + l*col_stride]) -> fragment order:
// [k block][chunk][step][m-tile i][lane]  holding  M(kb*8KT + 8i + lane/4, chunk*KC + 4 step + lane%4), zero padded.
__global__ void prep_fragments_kernel(const double* __restrict__ m, long long row_stride, long long col_stride,
                                      long long new_len, long long len, int kt, long long steps_padded,
                                      long long total, double* __restrict__ out) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= total) return;
  const int lane = static_cast<int>(e & 31);
  const long long q = e >> 5;
  const int i = static_cast<int>(q % kt);
  const long long r = q / kt;
  const long long step = r % steps_padded, kb = r / steps_padded;
  const long long k = kb * (8LL * kt) + 8 * i + (lane >> 2);
  const long long l = 4 * step + (lane & 3);
  out[e] = (k < new_len && l < len) ? m[k * row_stride + l * col_stride] : 0.0;
}

template <int KT, int NT, int KC, int STAGES, bool LAST>
cudaError_t launch_one(cudaStream_t stream, const TtmParams& p, int k_blocks) {
  constexpr int TILE_N = kWarps * NT;
  constexpr size_t smem = sizeof(double) * STAGES * (TILE_N * KC * 8 + (KC / 4) * KT * 32);
  auto kernel = ttm_dmma_kernel<KT, NT, KC, STAGES, LAST>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long long ctas = (p.n_tiles + TILE_N - 1) / TILE_N;
  dim3 grid(static_cast<unsigned>(ctas), static_cast<unsigned>(k_blocks));
  kernel<<<grid, kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

template <int KT, int NT>
cudaError_t launch_kt(cudaStream_t stream, const TtmParams& p, int k_blocks, bool last) {
  constexpr int KC = 16;
  constexpr int STAGES = (KT * NT <= 20) ? 3 : 4;
  return last ? launch_one<KT, NT, KC, STAGES, true>(stream, p, k_blocks)
              : launch_one<KT, NT, KC, STAGES, false>(stream, p, k_blocks);
}

}  // namespace

int ttm_pick_kt(long long new_len) {
  static const int options[] = {1, 2, 3, 4, 5, 6, 8, 10, 13};
  const long long need = (new_len + 7) / 8;
  for (int kt : options)
    if (kt >= need) return kt;
  return 13;
}

TtmFragmentLayout ttm_fragment_layout(long long new_len, long long len) {
  TtmFragmentLayout f;
  f.kt = ttm_pick_kt(new_len);
  f.k_blocks = static_cast<int>((new_len + 8LL * f.kt - 1) / (8LL * f.kt));
  f.kc = 16;
  f.n_chunks = static_cast<int>((len + f.kc - 1) / f.kc);
  f.doubles = static_cast<size_t>(f.k_blocks) * f.n_chunks * (f.kc / 4) * f.kt * 32;
  return f;
}

cudaError_t prep_factor_fragments(cudaStream_t stream, const double* m, long long row_stride, long long col_stride,
                                  long long new_len, long long len, const TtmFragmentLayout& f, double* out) {
  const long long total = static_cast<long long>(f.doubles);
  const long long steps_padded = static_cast<long long>(f.n_chunks) * (f.kc / 4);
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  prep_fragments_kernel<<<blocks, threads, 0, stream>>>(m, row_stride, col_stride, new_len, len, f.kt, steps_padded,
                                                        total, out);
  return cudaGetLastError();
}

cudaError_t launch_ttm(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                       const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z) {
  TtmParams p;
  p.x = x;
  p.z = z;
  p.mfrag = mfrag;
  p.outer = outer;
  p.len = len;
  p.inner = inner;
  p.new_len = new_len;
  p.n_chunks = f.n_chunks;
  const bool last = inner == 1;
  const bool base_aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(z) % 16 == 0);
  if (last) {
    p.tiles_per_slab = 1;
    p.n_tiles = (outer + 7) / 8;
    p.vec = base_aligned && (len % 2 == 0);
  } else {
    p.tiles_per_slab = static_cast<int>((inner + 7) / 8);
    p.n_tiles = outer * p.tiles_per_slab;
    p.vec = base_aligned && (inner % 2 == 0);
  }
  switch (f.kt) {
    case 1: return launch_kt<1, 4>(stream, p, f.k_blocks, last);
    case 2: return launch_kt<2, 4>(stream, p, f.k_blocks, last);
    case 3: return launch_kt<3, 4>(stream, p, f.k_blocks, last);
    case 4: return launch_kt<4, 4>(stream, p, f.k_blocks, last);
    case 5: return launch_kt<5, 4>(stream, p, f.k_blocks, last);
    case 6: return launch_kt<6, 2>(stream, p, f.k_blocks, last);
    case 8: return launch_kt<8, 2>(stream, p, f.k_blocks, last);
    case 10: return launch_kt<10, 2>(stream, p, f.k_blocks, last);
    case 13: return launch_kt<13, 2>(stream, p, f.k_blocks, last);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpb
