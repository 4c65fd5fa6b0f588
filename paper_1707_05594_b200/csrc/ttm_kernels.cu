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
//   * a CTA tile is WARPS*NT consecutive n-tiles times all 8*KT rows of one K
//     block; CTAs are persistent (grid = SMs x occupancy) and walk their tiles
//     round-robin, and the cp.async ring never drains between tiles: while the
//     last chunks of tile j are multiplied and its outputs stored, the first
//     chunks of tile j+1 are already in flight.  X chunks of KC contraction
//     steps stream through the STAGES-deep ring in shared memory, XOR-swizzled
//     so that the 64-bit fragment loads of a half-warp hit 16 distinct bank
//     pairs; the factor streams beside it in "fragment order" (prepared once
//     per factor by prep_factor_fragments), so an A fragment is one
//     conflict-free LDS.64 per lane and needs no bounds checks (padding rows
//     and columns are stored as zeros).
//   * every element of X is read from HBM exactly once per K block and every
//     element of Z written once; accumulation order is fixed (deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

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
  // Output row blocks ("destinations"): rows [dest_k0[d], dest_k0[d+1]) form their own contiguous tensor
  // (outer, rows_d, inner) starting at z + dest_off[d].  One destination = the plain layout; several = the
  // destination-major partial product a reduce-scatter over a split mode sends out (one chunk per peer).
  int n_dest;
  int dest_k0[kMaxTtmDest + 1];
  long long dest_off[kMaxTtmDest];
};

// One stage (KC contraction steps) for the first NL n-tiles of a warp.  NL is a compile-time count on purpose: a
// run-time guard around a DMMA is compiled into a predicate, and a predicated-off DMMA still takes its turn on the
// tensor pipe -- skipping dead tiles has to be a branch to another instantiation.
template <int KT, int NT, int NL, int KC, bool LAST>
__device__ __forceinline__ void consume_stage(double (&acc)[KT][NT][2], const double* __restrict__ xd,
                                              const double* __restrict__ md, int frag_k, int frag_n) {
#pragma unroll
  for (int s = 0; s < KC / 4; ++s) {
    double a[KT], b[NL];
#pragma unroll
    for (int i = 0; i < KT; ++i) a[i] = md[(s * KT + i) * 32];
    const int l = 4 * s + frag_k;
#pragma unroll
    for (int j = 0; j < NL; ++j)
      b[j] = LAST ? xd[j * (KC * 8) + frag_n * KC + (l ^ ((frag_n & 3) << 2))]
                  : xd[j * (KC * 8) + l * 8 + (frag_n ^ (((l >> 1) & 1) << 2))];
#pragma unroll
    for (int j = 0; j < NL; ++j)
#pragma unroll
      for (int i = 0; i < KT; ++i) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

// Persistent CTA: K block blockIdx.y; tile groups blockIdx.x, blockIdx.x + gridDim.x, ... of TILE_N n-tiles each.
template <int KT, int NT, int KC, int STAGES, bool LAST>
__global__ void __launch_bounds__(kThreads, (KT * NT <= 20) ? 2 : 1) ttm_dmma_kernel(const TtmParams p) {
  constexpr int TILE_N = kWarps * NT;
  constexpr int XS = TILE_N * KC * 8;     // doubles per stage of X
  constexpr int MS = (KC / 4) * KT * 32;  // doubles per stage of factor fragments
  constexpr int RING = 8;                 // tile tables alive at once (the loader runs < STAGES tiles ahead)
  static_assert((TILE_N & (TILE_N - 1)) == 0, "TILE_N must be a power of two");
  static_assert(KC % 16 == 0, "swizzle assumes 16-double rows");
  static_assert(STAGES + 1 <= RING, "tile-table ring too small");

  extern __shared__ __align__(16) double smem[];
  double* const xs = smem;
  double* const ms = smem + STAGES * XS;
  __shared__ long long tile_base[RING][TILE_N];  // element offset of the n-tile's first column at l = 0
  __shared__ long long tile_slab[RING][TILE_N];  // !LAST: slab index a of the n-tile
  __shared__ int tile_b0[RING][TILE_N];          // !LAST: first column b of the n-tile
  __shared__ int tile_lim[RING][TILE_N];         // valid columns (rows of X for LAST) in the n-tile, 0..8

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = blockIdx.y;
  const long long n_groups = (p.n_tiles + TILE_N - 1) / TILE_N;
  const long long my_tiles = blockIdx.x < n_groups ? (n_groups - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const long long total_items = my_tiles * p.n_chunks;

  // first n-tile of this CTA's j-th tile
  auto tile_first = [&](long long j) { return (static_cast<long long>(blockIdx.x) + j * gridDim.x) * TILE_N; };

  auto prep_table = [&](long long j) {
    if (tid < TILE_N) {
      const long long g = tile_first(j) + tid;
      long long base = 0, slab = 0;
      int lim = 0, b0 = 0;
      if (g < p.n_tiles) {
        if (LAST) {
          base = g * 8 * p.len;
          lim = static_cast<int>(min(8LL, p.outer - g * 8));
        } else {
          // n_tiles < 2^31 (checked by the launcher): 32-bit division
          const unsigned a = static_cast<unsigned>(g) / static_cast<unsigned>(p.tiles_per_slab);
          b0 = static_cast<int>(static_cast<unsigned>(g) - a * static_cast<unsigned>(p.tiles_per_slab)) * 8;
          slab = a;
          base = slab * p.len * p.inner + b0;
          lim = static_cast<int>(min(8LL, p.inner - b0));
        }
      }
      tile_base[j % RING][tid] = base;
      tile_slab[j % RING][tid] = slab;
      tile_b0[j % RING][tid] = b0;
      tile_lim[j % RING][tid] = lim;
    }
  };

  const double* const mfrag_kb = p.mfrag + static_cast<long long>(kb) * p.n_chunks * MS;

  // ---- loader.  With 256 threads and 16-byte copies every thread owns a fixed (n-tile, 16-byte column) pair and
  // walks the contraction rows, so its global address is a running pointer and its shared address a constant.
  constexpr int R = TILE_N / 4;       // 16-byte copies per thread per chunk (TILE_N * KC * 8 doubles / 2 / 256)
  constexpr int LSTEP = 64 / TILE_N;  // !LAST: rows between a thread's consecutive copies
  // !LAST: column pair ld_c of n-tile ld_t, rows ld_l + r * LSTEP
  const int ld_c = tid & 3, ld_t = (tid >> 2) & (TILE_N - 1), ld_l = (tid >> 2) / TILE_N;
  // LAST: 16-byte piece ld_c8 of row ld_row of n-tiles ld_t0 + 4 r
  const int ld_c8 = tid & 7, ld_row = (tid >> 3) & 7, ld_t0 = tid >> 6;
  const int dst_first = LAST ? ld_t0 * (8 * KC) + ld_row * KC + ((2 * ld_c8) ^ ((ld_row & 3) << 2))
                             : ld_t * (KC * 8) + ld_l * 8;
  const int swz0 = (ld_l >> 1) & 1;
  const double* ld_src = p.x;  // row 0 of the current load tile for this thread
  bool ld_ok = false;          // !LAST: the thread's column pair exists in its n-tile
  long long ld_a = 0;          // LAST: X row of the thread's first copy

  auto begin_load_tile = [&](long long j) {
    if (LAST) {
      ld_a = tile_first(j) * 8 + ld_t0 * 8 + ld_row;
      ld_src = p.x + ld_a * p.len + 2 * ld_c8;
    } else {
      ld_ok = 2 * ld_c < tile_lim[j % RING][ld_t];
      ld_src = p.x + tile_base[j % RING][ld_t] + 2 * ld_c + ld_l * p.inner;
    }
  };

  auto issue_chunk = [&](long long j, int chunk, int stage) {
    double* const xd = xs + stage * XS;
    const long long l0 = static_cast<long long>(chunk) * KC;
    if (p.vec) {
      if (chunk == 0) begin_load_tile(j);
      if (!LAST) {
        const double* src = ld_src + l0 * p.inner;
        const long long rows_left = p.len - l0 - ld_l;  // copy r is inside the extent iff r * LSTEP < rows_left
        const long long step = static_cast<long long>(LSTEP) * p.inner;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool ok = ld_ok && (r * LSTEP < rows_left);
          const int swz = (swz0 ^ ((r * LSTEP / 2) & 1)) << 2;
          cp_async16(xd + dst_first + r * (LSTEP * 8) + ((2 * ld_c) ^ swz), ok ? src : p.x, ok);
          src += step;
        }
      } else {
        const double* src = ld_src + l0;
        const bool col_ok = l0 + 2 * ld_c8 < p.len;
        const long long step = 32 * p.len;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool ok = col_ok && (ld_a + 32 * r < p.outer);
          cp_async16(xd + dst_first + r * (4 * 8 * KC), ok ? src : p.x, ok);
          src += step;
        }
      }
    } else {
      // unaligned / odd extents: element-wise 8-byte copies (rare shapes; correctness path)
      const long long* const base = tile_base[j % RING];
      const int* const lim = tile_lim[j % RING];
      if (!LAST) {
        for (int idx = tid; idx < TILE_N * KC * 8; idx += kThreads) {
          const int b = idx & 7, t = (idx >> 3) & (TILE_N - 1), l = idx / (8 * TILE_N);
          const bool ok = (l0 + l < p.len) && (b < lim[t]);
          const double* src = ok ? p.x + base[t] + (l0 + l) * p.inner + b : p.x;
          cp_async8(xd + t * (KC * 8) + l * 8 + (b ^ (((l >> 1) & 1) << 2)), src, ok);
        }
      } else {
        for (int idx = tid; idx < TILE_N * 8 * KC; idx += kThreads) {
          const int l = idx % KC, r = (idx / KC) & 7, t = idx / (8 * KC);
          const bool ok = (r < lim[t]) && (l0 + l < p.len);
          const double* src = ok ? p.x + base[t] + r * p.len + l0 + l : p.x;
          cp_async8(xd + t * (8 * KC) + r * KC + (l ^ ((r & 3) << 2)), src, ok);
        }
      }
    }
    const double* msrc = mfrag_kb + static_cast<long long>(chunk) * MS;
    double* const md = ms + stage * MS;
#pragma unroll
    for (int idx = tid; idx < MS / 2; idx += kThreads) cp_async16(md + 2 * idx, msrc + 2 * idx, true);
  };

  double acc[KT][NT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Epilogue of one tile: a lane holds rows k = 8 i + lane/4 and columns 2 (lane%4), +1 of each of its n-tiles.
  auto store_tile = [&](long long j) {
    const int col = 2 * (lane & 3);
    const long long first = tile_first(j);
#pragma unroll
    for (int jj = 0; jj < NT; ++jj) {
      const int t = warp * NT + jj;
      const int lim = tile_lim[j % RING][t];
      if (lim == 0) continue;
      const long long g = first + t;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const long long k_abs = static_cast<long long>(kb) * (8 * KT) + 8 * i + (lane >> 2);
        if (k_abs >= p.new_len) continue;
        int d = 0;
        while (d + 1 < p.n_dest && k_abs >= p.dest_k0[d + 1]) ++d;
        const long long k = k_abs - p.dest_k0[d];
        const long long rows_d = p.dest_k0[d + 1] - p.dest_k0[d];
        double* const zd = p.z + p.dest_off[d];
        if (LAST) {
          const long long a = g * 8 + col;
          if (col < lim) zd[a * rows_d + k] = acc[i][jj][0];
          if (col + 1 < lim) zd[(a + 1) * rows_d + k] = acc[i][jj][1];
        } else {
          const long long a = tile_slab[j % RING][t];
          const long long b = tile_b0[j % RING][t] + col;
          double* dst = zd + (a * rows_d + k) * p.inner + b;
          if (p.vec) {
            if (col < lim) *reinterpret_cast<double2*>(dst) = make_double2(acc[i][jj][0], acc[i][jj][1]);
          } else {
            if (col < lim) dst[0] = acc[i][jj][0];
            if (col + 1 < lim) dst[1] = acc[i][jj][1];
          }
        }
      }
    }
  };

  // ---- prologue: tables for the first STAGES tiles, then STAGES-1 chunks in flight
  long long prepped = min(my_tiles, static_cast<long long>(STAGES));
  for (long long j = 0; j < prepped; ++j) prep_table(j);
  __syncthreads();
  long long load_j = 0, cons_j = 0;
  int load_c = 0, cons_c = 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (load_j < my_tiles) {
      issue_chunk(load_j, load_c, s);
      if (++load_c == p.n_chunks) {
        load_c = 0;
        ++load_j;
      }
    }
    cp_async_commit();
  }
  int load_stage = STAGES - 1, cons_stage = 0;

  const int frag_k = lane & 3, frag_n = lane >> 2;
  for (long long it = 0; it < total_items; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (load_j < my_tiles) {
      issue_chunk(load_j, load_c, load_stage);
      if (++load_c == p.n_chunks) {
        load_c = 0;
        ++load_j;
      }
    }
    cp_async_commit();
    load_stage = (load_stage + 1 == STAGES) ? 0 : load_stage + 1;

    const double* const xd = xs + cons_stage * XS + (warp * NT) * (KC * 8);
    const double* const md = ms + cons_stage * MS + lane;
    cons_stage = (cons_stage + 1 == STAGES) ? 0 : cons_stage + 1;
    // n-tiles past the end of the tensor hold nothing but zeros; they are the last ones of the warp's NT
    int n_live = 0;
#pragma unroll
    for (int j = 0; j < NT; ++j) n_live += tile_lim[cons_j % RING][warp * NT + j] != 0 ? 1 : 0;
    if (n_live == NT) {
      consume_stage<KT, NT, NT, KC, LAST>(acc, xd, md, frag_k, frag_n);
    } else if (NT >= 4 && n_live == 3) {
      consume_stage<KT, NT, (NT >= 4 ? 3 : 1), KC, LAST>(acc, xd, md, frag_k, frag_n);
    } else if (NT >= 2 && n_live == 2) {
      consume_stage<KT, NT, (NT >= 2 ? 2 : 1), KC, LAST>(acc, xd, md, frag_k, frag_n);
    } else if (n_live == 1) {
      consume_stage<KT, NT, 1, KC, LAST>(acc, xd, md, frag_k, frag_n);
    }
    if (++cons_c == p.n_chunks) {
      store_tile(cons_j);
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      cons_c = 0;
      ++cons_j;
    }
    // table of the tile the loader enters next; visible after the barrier at the top of the next iteration
    if (prepped <= load_j && load_j < my_tiles) {
      prep_table(prepped);
      ++prepped;
    }
  }
  cp_async_wait<0>();
}

// factor (rows new_len x cols len, element (k,l) at m[k*row_stride + l*col_stride]) -> fragment order:
// [k block][chunk][step][m-tile i][lane]  holding  M(kb*8KT + 8i + lane/4, chunk*KC + 4 step + lane%4), zero padded.
// Two copies are written: out[0 .. total) with the k-indices of a step on consecutive rows (l = 4 step + lane%4; the
// cp.async kernel and the inner == 1 TMA kernel), and out[total .. 2 total) with them interleaved inside 8-row groups
// (steps 2g / 2g+1 take rows 8g + {0,2,4,6} / {1,3,5,7}; the inner > 1 TMA kernel, see ttm_tma_kernels.cu).
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
  const long long li = 8 * (step >> 1) + 2 * (lane & 3) + (step & 1);
  out[total + e] = (k < new_len && li < len) ? m[k * row_stride + li * col_stride] : 0.0;
}

template <int KT, int NT, int KC, int STAGES, bool LAST>
cudaError_t launch_one(cudaStream_t stream, const TtmParams& p, int k_blocks, int sm_count) {
  constexpr int TILE_N = kWarps * NT;
  constexpr size_t smem = sizeof(double) * STAGES * (TILE_N * KC * 8 + (KC / 4) * KT * 32);
  auto kernel = ttm_dmma_kernel<KT, NT, KC, STAGES, LAST>;
  static PerDeviceInt cache;  // per instantiation and device: resident CTAs per SM, 0 = not configured yet
  std::atomic<int>* const slot = cache.slot();
  int ctas_per_sm = slot ? slot->load(std::memory_order_relaxed) : 0;
  if (ctas_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
    if (e != cudaSuccess) return e;
    ctas_per_sm = occ < 1 ? 1 : occ;
    if (slot) slot->store(ctas_per_sm, std::memory_order_relaxed);
  }
  const long long groups = (p.n_tiles + TILE_N - 1) / TILE_N;
  const long long resident = std::max(1LL, static_cast<long long>(sm_count) * ctas_per_sm / k_blocks);
  dim3 grid(static_cast<unsigned>(std::min(groups, resident)), static_cast<unsigned>(k_blocks));
  kernel<<<grid, kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

// NT (n-tiles per warp) trades register reuse of the factor fragments against the number of CTA tiles: wide
// tiles when the problem has plenty of columns, narrow ones when it would not otherwise cover the SMs.
template <int KT>
cudaError_t launch_kt(cudaStream_t stream, const TtmParams& p, int k_blocks, bool last, int sm_count) {
  constexpr int KC = 16;
  constexpr int WIDE = (KT <= 5) ? 4 : 2;
  constexpr int STAGES_WIDE = (KT * WIDE <= 20) ? 3 : 4;
  const long long wide_groups = (p.n_tiles + kWarps * WIDE - 1) / (kWarps * WIDE);
  if (wide_groups * k_blocks >= sm_count) {
    return last ? launch_one<KT, WIDE, KC, STAGES_WIDE, true>(stream, p, k_blocks, sm_count)
                : launch_one<KT, WIDE, KC, STAGES_WIDE, false>(stream, p, k_blocks, sm_count);
  }
  return last ? launch_one<KT, 1, KC, 4, true>(stream, p, k_blocks, sm_count)
              : launch_one<KT, 1, KC, 4, false>(stream, p, k_blocks, sm_count);
}

}  // namespace

// Process-wide switch between the TMA pipeline and the cp.async kernel (A/B tests through tp_set_global_option;
// both kernels compute the same sums in the same order).
std::atomic<bool>& ttm_tma_enabled() {
  static std::atomic<bool> on{true};
  return on;
}

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
  f.layout_doubles = static_cast<size_t>(f.k_blocks) * f.n_chunks * (f.kc / 4) * f.kt * 32;
  f.doubles = 2 * f.layout_doubles;  // consecutive-row copy + interleaved-row copy
  return f;
}

cudaError_t prep_factor_fragments(cudaStream_t stream, const double* m, long long row_stride, long long col_stride,
                                  long long new_len, long long len, const TtmFragmentLayout& f, double* out) {
  const long long total = static_cast<long long>(f.layout_doubles);
  const long long steps_padded = static_cast<long long>(f.n_chunks) * (f.kc / 4);
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  prep_fragments_kernel<<<blocks, threads, 0, stream>>>(m, row_stride, col_stride, new_len, len, f.kt, steps_padded,
                                                        total, out);
  return cudaGetLastError();
}

cudaError_t launch_ttm(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                       const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z, int sm_count,
                       int n_dest, const long long* dest_cuts, const long long* dest_offsets) {
  const bool plain_dest = (!dest_cuts || (dest_cuts[0] == 0 && dest_cuts[1] == new_len)) && (!dest_offsets || dest_offsets[0] == 0);
  if (plain_dest && ttm_splitk_eligible(outer, len, inner, f.kt, f.k_blocks, n_dest))
    return launch_ttm_splitk(stream, x, outer, len, inner, mfrag, f, new_len, z);
  if (ttm_packed_eligible(x, outer, len, inner, z, f.kt, n_dest) && (!dest_cuts || (dest_cuts[0] == 0 && dest_cuts[1] == new_len)) &&
      (!dest_offsets || dest_offsets[0] == 0))
    return launch_ttm_packed(stream, x, outer, len, inner, mfrag, f, new_len, z, sm_count);
  if (ttm_tma_enabled().load(std::memory_order_relaxed) &&
      ttm_tma_eligible(x, outer, len, inner, z, f.kt, f.k_blocks, sm_count)) {
    bool chunks_aligned = true;
    for (int d = 0; dest_cuts && d < n_dest; ++d)
      chunks_aligned = chunks_aligned && ((dest_offsets ? dest_offsets[d] : outer * dest_cuts[d] * inner) % 2 == 0);
    if (chunks_aligned)
      return launch_ttm_tma(stream, x, outer, len, inner, inner == 1 ? mfrag : mfrag + f.layout_doubles, f, new_len, z,
                            sm_count, n_dest, dest_cuts, dest_offsets);
  }
  TtmParams p;
  if (n_dest < 1 || n_dest > kMaxTtmDest) return cudaErrorInvalidValue;
  p.n_dest = n_dest;
  bool dest_aligned = true;
  {
    long long off = 0;
    for (int d = 0; d < n_dest; ++d) {
      const long long k0 = dest_cuts ? dest_cuts[d] : 0, k1 = dest_cuts ? dest_cuts[d + 1] : new_len;
      p.dest_k0[d] = static_cast<int>(k0);
      p.dest_k0[d + 1] = static_cast<int>(k1);
      p.dest_off[d] = dest_offsets ? dest_offsets[d] : off;
      dest_aligned = dest_aligned && (p.dest_off[d] % 2 == 0);
      off += outer * (k1 - k0) * inner;
    }
    for (int d = n_dest + 1; d <= kMaxTtmDest; ++d) p.dest_k0[d] = p.dest_k0[n_dest];
    for (int d = n_dest; d < kMaxTtmDest; ++d) p.dest_off[d] = 0;
  }
  p.x = x;
  p.z = z;
  p.mfrag = mfrag;
  p.outer = outer;
  p.len = len;
  p.inner = inner;
  p.new_len = new_len;
  p.n_chunks = f.n_chunks;
  const bool last = inner == 1;
  const bool base_aligned =
      (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(z) % 16 == 0) && dest_aligned;
  if (last) {
    p.tiles_per_slab = 1;
    p.n_tiles = (outer + 7) / 8;
    p.vec = base_aligned && (len % 2 == 0);
  } else {
    p.tiles_per_slab = static_cast<int>((inner + 7) / 8);
    p.n_tiles = outer * p.tiles_per_slab;
    p.vec = base_aligned && (inner % 2 == 0);
  }
  if (p.n_tiles >= (1LL << 31)) return cudaErrorInvalidValue;  // 2^34 columns: beyond any tensor that fits in HBM
  switch (f.kt) {
    case 1: return launch_kt<1>(stream, p, f.k_blocks, last, sm_count);
    case 2: return launch_kt<2>(stream, p, f.k_blocks, last, sm_count);
    case 3: return launch_kt<3>(stream, p, f.k_blocks, last, sm_count);
    case 4: return launch_kt<4>(stream, p, f.k_blocks, last, sm_count);
    case 5: return launch_kt<5>(stream, p, f.k_blocks, last, sm_count);
    case 6: return launch_kt<6>(stream, p, f.k_blocks, last, sm_count);
    case 8: return launch_kt<8>(stream, p, f.k_blocks, last, sm_count);
    case 10: return launch_kt<10>(stream, p, f.k_blocks, last, sm_count);
    case 13: return launch_kt<13>(stream, p, f.k_blocks, last, sm_count);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpb
