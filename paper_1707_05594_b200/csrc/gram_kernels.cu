// Gram matrix of a mode-n unfolding, computed straight from the tensor.
//
//   G(i, j) = sum_{a, b} Y(a, i, b) * Y(a, j, b)        Y viewed as (outer, rows, inner)
//
// replaces reference unfold() + selfadjointView<Lower>().rankUpdate()
// (ttm.hpp:43-53, hooi.hpp:53-54): no matricisation copy — the sum over
// unfolding columns is order-invariant, so each CTA walks contiguous pieces of
// Y directly.  SYRK-style: only 64x64 tiles with tile_i >= tile_j are
// computed, on DMMA.8x8x4; the contraction range is split across CTAs and the
// partial tiles are summed in a fixed order (deterministic) by a second tiny
// kernel that also mirrors the result into full symmetric storage.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kThreads = 128;  // 4 warps x (32 x 32) warp tiles: 8 fragment loads per 16 DMMAs
constexpr int kTile = 64;
constexpr int kKC = 16;
constexpr int kStages = 3;

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

struct GramParams {
  const double* __restrict__ y;
  double* __restrict__ partial;  // [splits][rows][rows], entry (i, j) of a computed tile at i * rows + j
  long long outer, rows, inner;
  long long chunks;            // contraction chunks of kKC
  long long chunks_per_split;
  int chunks_per_slab;         // inner > 1: ceil(inner / kKC)
  int vec;
};

// INNER1: the contraction index (slab a) is the strided one and rows are contiguous -> stage as [kKC][64].
// otherwise the contraction index b is contiguous -> stage as [64][kKC].
template <bool INNER1>
__global__ void __launch_bounds__(kThreads, 4) gram_dmma_kernel(const GramParams p) {
  __shared__ __align__(16) double sa[kStages][kTile * kKC];
  __shared__ __align__(16) double sb[kStages][kTile * kKC];

  // lower-triangular tile index -> (ti, tj), ti >= tj
  int ti = 0, tj = static_cast<int>(blockIdx.x);
  while (tj > ti) {
    tj -= ti + 1;
    ++ti;
  }
  const bool diag = ti == tj;
  const long long i0 = static_cast<long long>(ti) * kTile, j0 = static_cast<long long>(tj) * kTile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // warp tile: rows wm*32..+32, cols wn*32..+32

  const long long c_begin = static_cast<long long>(blockIdx.y) * p.chunks_per_split;
  const long long c_end = min(p.chunks, c_begin + p.chunks_per_split);
  const int n_chunks = static_cast<int>(max(0LL, c_end - c_begin));

  auto load_tile = [&](double* dst, long long r0, long long chunk) {
    if (INNER1) {
      const long long a0 = chunk * kKC;
      if (p.vec) {
        for (int idx = tid; idx < kKC * (kTile / 2); idx += kThreads) {
          const int c = idx % (kTile / 2), l = idx / (kTile / 2);
          const bool ok = (a0 + l < p.outer) && (r0 + 2 * c < p.rows);
          const double* src = ok ? p.y + (a0 + l) * p.rows + r0 + 2 * c : p.y;
          cp_async16(dst + l * kTile + ((2 * c) ^ ((l & 3) << 2)), src, ok);
        }
      } else {
        for (int idx = tid; idx < kKC * kTile; idx += kThreads) {
          const int r = idx % kTile, l = idx / kTile;
          const bool ok = (a0 + l < p.outer) && (r0 + r < p.rows);
          const double* src = ok ? p.y + (a0 + l) * p.rows + r0 + r : p.y;
          cp_async8(dst + l * kTile + (r ^ ((l & 3) << 2)), src, ok);
        }
      }
    } else {
      const long long a = chunk / p.chunks_per_slab;
      const long long b0 = (chunk - a * p.chunks_per_slab) * kKC;
      const double* slab = p.y + a * p.rows * p.inner;
      if (p.vec) {
        for (int idx = tid; idx < kTile * (kKC / 2); idx += kThreads) {
          const int c = idx % (kKC / 2), r = idx / (kKC / 2);
          const bool ok = (r0 + r < p.rows) && (b0 + 2 * c < p.inner);
          const double* src = ok ? slab + (r0 + r) * p.inner + b0 + 2 * c : p.y;
          cp_async16(dst + r * kKC + ((2 * c) ^ ((r & 3) << 2)), src, ok);
        }
      } else {
        for (int idx = tid; idx < kTile * kKC; idx += kThreads) {
          const int l = idx % kKC, r = idx / kKC;
          const bool ok = (r0 + r < p.rows) && (b0 + l < p.inner);
          const double* src = ok ? slab + (r0 + r) * p.inner + b0 + l : p.y;
          cp_async8(dst + r * kKC + (l ^ ((r & 3) << 2)), src, ok);
        }
      }
    }
  };
  auto issue = [&](int n, int stage) {
    load_tile(sa[stage], i0, c_begin + n);
    if (!diag) load_tile(sb[stage], j0, c_begin + n);
  };
  auto frag = [&](const double* tile, int row, int l) -> double {
    return INNER1 ? tile[l * kTile + (row ^ ((l & 3) << 2))] : tile[row * kKC + (l ^ ((row & 3) << 2))];
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < n_chunks) issue(s, s);
    cp_async_commit();
  }
  for (int n = 0; n < n_chunks; ++n) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int next = n + kStages - 1;
      if (next < n_chunks) issue(next, next % kStages);
      cp_async_commit();
    }
    const double* ta = sa[n % kStages];
    const double* tb = diag ? ta : sb[n % kStages];
#pragma unroll
    for (int s = 0; s < kKC / 4; ++s) {
      const int l = 4 * s + (lane & 3);
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = frag(ta, wm * 32 + a * 8 + (lane >> 2), l);
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = frag(tb, wn * 32 + b * 8 + (lane >> 2), l);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
  }
  cp_async_wait<0>();

  double* out = p.partial + static_cast<long long>(blockIdx.y) * p.rows * p.rows;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const long long i = i0 + wm * 32 + a * 8 + (lane >> 2);
      const long long j = j0 + wn * 32 + b * 8 + 2 * (lane & 3);
      if (i < p.rows) {
        if (j < p.rows) out[i * p.rows + j] = acc[a][b][0];
        if (j + 1 < p.rows) out[i * p.rows + j + 1] = acc[a][b][1];
      }
    }
}

// gram(i, j) = gram(j, i) = sum_s partial[s](i, j), i >= j, splits summed in index order.
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int splits, long long rows,
                                   double* __restrict__ gram) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= rows * rows) return;
  const long long i = e / rows, j = e % rows;
  if (j > i) return;
  // splits summed in index order; the loads of a batch are independent and issued together (one exposed L2 latency
  // per 16 splits instead of one per split)
  const long long plane = rows * rows;
  const double* src = partial + e;
  double sum = 0.0;
  int s = 0;
  for (; s + 16 <= splits; s += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(src + static_cast<long long>(s + u) * plane);
#pragma unroll
    for (int u = 0; u < 16; ++u) sum += v[u];
  }
  {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = (s + u < splits) ? __ldcg(src + static_cast<long long>(s + u) * plane) : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (s + u < splits) sum += v[u];
  }
  gram[i * rows + j] = sum;
  gram[j * rows + i] = sum;
}

}  // namespace

std::atomic<bool>& gram_wide_enabled() {
  static std::atomic<bool> on{true};
  return on;
}

std::atomic<int>& gram_wide_spare_sms() {
  static std::atomic<int> sms{0};  // measured on C5: 0 -> 57.07 ms/iter, 4 -> 57.15, 16 -> 57.22
  return sms;
}

namespace {
GramLayout gram_narrow_layout(long long outer, long long rows, long long inner, int sm_count);
}

GramLayout gram_layout(long long outer, long long rows, long long inner, int sm_count) {
  if (gram_wide_enabled().load(std::memory_order_relaxed) && gram_wide_shape(outer, rows, inner)) {
    GramLayout g = gram_wide_layout(outer, rows, inner, sm_count);
    // a base address that is not 16-byte aligned sends the launch back to the narrow kernel: room for its partials too
    g.workspace_doubles = std::max(g.workspace_doubles, gram_narrow_layout(outer, rows, inner, sm_count).workspace_doubles);
    g.sm_count = sm_count;
    return g;
  }
  return gram_narrow_layout(outer, rows, inner, sm_count);
}

namespace {
GramLayout gram_narrow_layout(long long outer, long long rows, long long inner, int sm_count) {
  GramLayout g;
  g.sm_count = sm_count;
  g.tiles = static_cast<int>((rows + kTile - 1) / kTile);
  g.chunks = inner == 1 ? (outer + kKC - 1) / kKC : outer * ((inner + kKC - 1) / kKC);
  const long long lower_tiles = static_cast<long long>(g.tiles) * (g.tiles + 1) / 2;
  // Four CTAs fit per SM.  The split count s is the one that minimises waves(s) x chunks per CTA: a grid that ends
  // just past a wave boundary wastes most of its last wave (C5 leaf: 325 tiles x 8 splits = 4.4 waves cost 5; 9 splits
  // fill 4.94).  A CTA walks at least 8 chunks, except when the whole problem is a few waves of single chunks (the
  // leaves of small tensors): there the serial chunk loop of a CTA is the whole kernel time, so it is cut down to what
  // the cp.async ring holds in flight at once.
  const long long per_wave = 4LL * sm_count;
  const long long min_chunks = (g.chunks * lower_tiles <= 4 * per_wave * kStages) ? kStages : 8;
  // ... and at most 1 GiB of partial planes
  const long long plane_cap = std::max(1LL, (1LL << 27) / std::max(1LL, rows * rows));
  const long long max_splits = std::max(1LL, std::min({512LL, g.chunks / min_chunks, plane_cap}));
  long long best = 1, best_cost = -1;
  for (long long s = 1; s <= max_splits; ++s) {
    const long long per = (g.chunks + s - 1) / s;
    const long long used = (g.chunks + per - 1) / per;  // splits that actually get chunks
    const long long waves = (lower_tiles * used + per_wave - 1) / per_wave;
    const long long cost = waves * (per + 2) * 64 + used * 8;  // + 2: pipeline fill per CTA; used: the ordered sum
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = used;
    }
  }
  g.splits = static_cast<int>(best);
  g.workspace_doubles = static_cast<size_t>(g.splits) * rows * rows;
  return g;
}
}  // namespace

cudaError_t launch_gram(cudaStream_t stream, const double* y, long long outer, long long rows, long long inner,
                        const GramLayout& layout, double* workspace, double* gram) {
  GramLayout g = layout;
  if (g.wide) {
    if (reinterpret_cast<uintptr_t>(y) % 16 == 0 && ttm_tensor_map(y, outer, rows, inner)) {
      cudaError_t e = launch_gram_wide(stream, y, outer, rows, inner, g, workspace, g.sm_count);
      if (e != cudaSuccess) return e;
      const long long total = rows * rows;
      gram_reduce_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(workspace, g.splits, rows, gram);
      return cudaGetLastError();
    }
    g = gram_narrow_layout(outer, rows, inner, g.sm_count);
  }
  GramParams p;
  p.y = y;
  p.partial = workspace;
  p.outer = outer;
  p.rows = rows;
  p.inner = inner;
  p.chunks = g.chunks;
  p.chunks_per_split = (g.chunks + g.splits - 1) / g.splits;
  p.chunks_per_slab = static_cast<int>(inner == 1 ? 1 : (inner + kKC - 1) / kKC);
  const bool aligned = reinterpret_cast<uintptr_t>(y) % 16 == 0;
  p.vec = aligned && ((inner == 1 ? rows : inner) % 2 == 0);
  const unsigned lower_tiles = static_cast<unsigned>(g.tiles) * (g.tiles + 1) / 2;
  dim3 grid(lower_tiles, static_cast<unsigned>(g.splits));
  if (inner == 1)
    gram_dmma_kernel<true><<<grid, kThreads, 0, stream>>>(p);
  else
    gram_dmma_kernel<false><<<grid, kThreads, 0, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long long total = rows * rows;
  gram_reduce_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(workspace, g.splits, rows, gram);
  return cudaGetLastError();
}

}  // namespace tpb
