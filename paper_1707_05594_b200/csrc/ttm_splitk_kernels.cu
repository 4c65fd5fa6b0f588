// Mode-n TTM for nodes with FEW columns and a contraction of up to 512: the contraction is split over the warps.
//
//   Z(a, k, b) = sum_l M(k, l) * X(a, l, b)        X viewed as (outer, L, inner), row-major
//
// The streaming kernels (ttm_kernels.cu, ttm_tma_kernels.cu) give a CTA 64+ columns and walk the contraction chunk by
// chunk through a shared-memory ring.  On the small nodes deep in a TTM tree (a few thousand columns, L = 50..400)
// that is a handful of CTAs each paying L / 16 dependent pipeline steps: 6-29 us for work whose roofline is ~1 us.
// Here
//
//   * a CTA owns 8 / S n-tiles (8 columns each) of one K block; S = 1, 2, 4 or 8 warps share an n-tile and split its
//     contraction range between them (S is the largest split that still gives at most one wave of CTAs: splitting
//     shortens the dependent chain of a warp, more CTAs than the machine holds at once lengthen the launch);
//   * there is no shared-memory staging: a DMMA B fragment (4 contraction steps x 8 columns) is 4 runs of 64
//     contiguous bytes (inner > 1) or 8 runs of 32 bytes (inner == 1), i.e. whole sectors, so every lane loads its
//     elements straight from global memory, 16 / 8 / 6 contraction steps at a time (by the number of m-tiles, so
//     that a round's operands fit the registers of two resident CTAs), all issued -- together with the round's
//     factor fragments -- before the first DMMA of the round;
//   * the factor arrives in the same fragment order as for the other kernels (one coalesced 256-byte load per
//     fragment, L2 resident);
//   * the S partial tiles of an n-tile are added in warp order through shared memory (deterministic) and stored.
//
// Eligibility depends on the shape only (never on the SM budget of the call), so a given node is always computed by
// the same kernel in the same summation order -- the engine's bit-identity guarantees (carried path, recorded sweeps,
// forked walks) rest on that.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kRound = 16;            // contraction steps of 4 a warp loads before it multiplies
constexpr long long kMaxTiles = 640;  // n-tiles x K blocks of a launch: beyond, the unsplit streaming kernels are as fast
constexpr long long kMaxLen = 512;
constexpr long long kOneWave = 296;   // CTAs of this kernel a B200 holds at once (148 SMs x 2); a constant, not the
                                      // call's SM budget: the split, hence the summation order, depends on the shape only

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Predicated VOLATILE load: written as plain (or ld.global.nc) loads, the loads of a round are sunk to their uses --
// by the compiler into the DMMA branches, and by ptxas even across a warp barrier -- to save registers, which turns
// one exposed memory latency per round into one per contraction step.  Volatile accesses stay where they are.
__device__ __forceinline__ double load_if(const double* ptr, bool ok) {
  double v;
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.ne.b32 q, %2, 0;\n"
      "mov.f64 %0, 0d0000000000000000;\n"
      "@q ld.volatile.global.f64 %0, [%1];\n"
      "}\n"
      : "=d"(v)
      : "l"(ptr), "r"(static_cast<int>(ok)));
  return v;
}

struct SplitKParams {
  const double* __restrict__ x;
  double* __restrict__ z;
  const double* __restrict__ mfrag;  // [k blocks][steps_padded][KT][32], consecutive-row copy
  long long outer, len, inner, new_len;
  int tiles_per_slab;                // ceil(inner / 8), inner > 1 only
  int steps_padded;                  // 4 * n_chunks
  int steps;                         // ceil(len / 4)
  int steps_per_warp;
  int split;                         // S: warps per n-tile
  long long n_tiles;
};

template <int KT, bool LAST>
__global__ void __launch_bounds__(kThreads, 2) ttm_splitk_kernel(const SplitKParams p) {
  __shared__ double red[kWarps][KT * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = p.split, per_cta = kWarps / S;
  const long long tile = static_cast<long long>(blockIdx.x) * per_cta + warp / S;
  const int part = warp % S;
  const int kb = blockIdx.y;
  const int n = lane >> 2, kk = lane & 3;

  // column of this lane and its stride along the contraction
  const double* base = p.x;
  long long stride = 1;
  bool valid = tile < p.n_tiles;
  if (LAST) {
    const long long a = tile * 8 + n;
    valid = valid && a < p.outer;
    base = p.x + (valid ? a : 0) * p.len;
  } else {
    const long long slab = valid ? tile / p.tiles_per_slab : 0;
    const long long b0 = valid ? (tile - slab * p.tiles_per_slab) * 8 : 0;
    valid = valid && b0 + n < p.inner;
    base = p.x + slab * p.len * p.inner + (valid ? b0 + n : 0);
    stride = p.inner;
  }
  const int s0 = part * p.steps_per_warp;
  const int s1 = (tile < p.n_tiles) ? min(p.steps, s0 + p.steps_per_warp) : s0;

  double acc[KT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double* const mf = p.mfrag + static_cast<long long>(kb) * p.steps_padded * (KT * 32) + lane;
  // a round = RND contraction steps: every load of the round (B from the tensor, A from the factor fragments) is issued
  // before its first DMMA, so a round costs one memory latency, not one per step
  constexpr int RND = KT <= 2 ? kRound : (KT <= 4 ? kRound / 2 : 6);  // the round's operands fit 128 registers
  for (int r0 = s0; r0 < s1; r0 += RND) {
    double b[RND], a[RND][KT];
#pragma unroll
    for (int j = 0; j < RND; ++j) {
      const long long l = 4LL * (r0 + j) + kk;
      const bool ok = r0 + j < s1 && l < p.len && valid;
      b[j] = load_if(base + (ok ? l : 0) * stride, ok);
    }
#pragma unroll
    for (int j = 0; j < RND; ++j)
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const bool ok = r0 + j < s1;
        a[j][i] = load_if(mf + (static_cast<long long>(ok ? r0 + j : 0) * KT + i) * 32, ok);
      }
    // no branch around the DMMAs of a ragged last round (their operands are zeros): with one, the loads above are
    // scheduled into the branches, next to their uses; the warp barrier keeps ptxas from sinking them as well
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RND; ++j)
#pragma unroll
      for (int i = 0; i < KT; ++i) dmma884(acc[i][0], acc[i][1], a[j][i], b[j]);
  }

  // partial tiles -> shared memory: value (i, row r, column c) of a warp's tile at i * 64 + r * 8 + c
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    red[warp][i * 64 + n * 8 + 2 * kk] = acc[i][0];
    red[warp][i * 64 + n * 8 + 2 * kk + 1] = acc[i][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < per_cta * KT * 64; e += kThreads) {
    const int q = e / (KT * 64), v = e - q * (KT * 64);
    const long long t = static_cast<long long>(blockIdx.x) * per_cta + q;
    if (t >= p.n_tiles) break;
    double sum = red[q * S][v];
    for (int w = 1; w < S; ++w) sum += red[q * S + w][v];
    const int col = v & 7, r = (v >> 3) & 7, i = v >> 6;
    const long long k = static_cast<long long>(kb) * (8 * KT) + 8 * i + r;
    if (k >= p.new_len) continue;
    if (LAST) {
      const long long a = t * 8 + col;
      if (a < p.outer) p.z[a * p.new_len + k] = sum;
    } else {
      const long long slab = t / p.tiles_per_slab;
      const long long b0 = (t - slab * p.tiles_per_slab) * 8;
      if (b0 + col < p.inner) p.z[(slab * p.new_len + k) * p.inner + b0 + col] = sum;
    }
  }
}

template <int KT>
cudaError_t launch_splitk(cudaStream_t stream, const SplitKParams& p, long long n_tiles, int k_blocks, bool last) {
  const long long per_cta = kWarps / p.split;
  dim3 grid(static_cast<unsigned>((n_tiles + per_cta - 1) / per_cta), static_cast<unsigned>(k_blocks));
  if (last)
    ttm_splitk_kernel<KT, true><<<grid, kThreads, 0, stream>>>(p);
  else
    ttm_splitk_kernel<KT, false><<<grid, kThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

long long splitk_tiles(long long outer, long long inner) {
  return inner == 1 ? (outer + 7) / 8 : outer * ((inner + 7) / 8);
}

}  // namespace

std::atomic<bool>& ttm_splitk_enabled() {
  static std::atomic<bool> on{true};
  return on;
}

bool ttm_splitk_eligible(long long outer, long long len, long long inner, int kt, int k_blocks, int n_dest) {
  if (!ttm_splitk_enabled().load(std::memory_order_relaxed)) return false;
  if (n_dest != 1 || kt > 6 || len < 32 || len > kMaxLen || outer < 1 || inner < 1) return false;
  if (inner > 1 && inner < 8) return false;  // short trailing extents: the packed kernel's n-tiles have no padding
  return splitk_tiles(outer, inner) * k_blocks <= kMaxTiles;
}

cudaError_t launch_ttm_splitk(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                              const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z) {
  SplitKParams p;
  p.x = x;
  p.z = z;
  p.mfrag = mfrag;
  p.outer = outer;
  p.len = len;
  p.inner = inner;
  p.new_len = new_len;
  p.tiles_per_slab = static_cast<int>(inner == 1 ? 1 : (inner + 7) / 8);
  p.steps_padded = f.n_chunks * (f.kc / 4);
  p.steps = static_cast<int>((len + 3) / 4);
  const long long n_tiles = splitk_tiles(outer, inner);
  p.n_tiles = n_tiles;
  p.split = 1;
  while (p.split < kWarps && n_tiles * f.k_blocks * (2 * p.split) <= kOneWave * kWarps && 4 * (2 * p.split) <= p.steps)
    p.split *= 2;
  p.steps_per_warp = (p.steps + p.split - 1) / p.split;
  const bool last = inner == 1;
  switch (f.kt) {
    case 1: return launch_splitk<1>(stream, p, n_tiles, f.k_blocks, last);
    case 2: return launch_splitk<2>(stream, p, n_tiles, f.k_blocks, last);
    case 3: return launch_splitk<3>(stream, p, n_tiles, f.k_blocks, last);
    case 4: return launch_splitk<4>(stream, p, n_tiles, f.k_blocks, last);
    case 5: return launch_splitk<5>(stream, p, n_tiles, f.k_blocks, last);
    case 6: return launch_splitk<6>(stream, p, n_tiles, f.k_blocks, last);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpb
