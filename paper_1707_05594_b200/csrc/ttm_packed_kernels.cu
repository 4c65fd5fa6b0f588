// Mode-n TTM for a SHORT trailing extent (1 < inner <= 8), columns packed across slabs.
//
//   Z(a, k, b) = sum_l M(k, l) * X(a, l, b)        X viewed as (outer, L, inner), row-major
//
// The general kernels (ttm_kernels.cu, ttm_tma_kernels.cu) cut the columns of one slab a into n-tiles of eight
// consecutive b: with inner = 5 three of the eight columns of every DMMA are padding, and an odd inner additionally
// forces their loaders onto 8-byte copies with per-element index arithmetic.  Here
//
//   * a CTA tile is 32 consecutive slabs.  Their columns (a, b), flattened, are exactly 4 * inner full n-tiles of
//     eight -- no padding for any inner -- and the lane that holds column c of an n-tile simply reads slab c / inner,
//     column c % inner (offsets fixed for the whole launch);
//   * a slab is contiguous (L * inner doubles), so a chunk of 16 contraction rows of one slab is ONE contiguous run
//     of 16 * inner doubles: the loader moves it with 16-byte cp.async copies into shared memory as it lies, whatever
//     the parity of inner (needs L * inner even, which keeps every run 16-byte aligned);
//   * same factor fragments, DMMA.8x8x4 arithmetic, cp.async ring over (tile, chunk) items and fixed summation order
//     as ttm_dmma_kernel.
// Every element of X is read once per K block, every element of Z written once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kSlabs = 32;   // slabs per CTA tile
constexpr int kKC = 16;      // contraction rows per chunk
constexpr int kSlots = 4;    // n-tiles per warp: n-tile j belongs to warp j % 8, slot j / 8 (4 * inner <= 32 tiles)
constexpr int kStages = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem), "r"(bytes) : "memory");
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

struct PackedParams {
  const double* __restrict__ x;
  double* __restrict__ z;
  const double* __restrict__ mfrag;  // [k blocks][chunks][kKC / 4][KT][32], consecutive-row copy
  long long outer, len, new_len;
  int inner;
  int n_chunks;  // ceil(len / kKC)
};

// One chunk of kKC contraction rows for the first NQ slots of a warp.
template <int KT, int NQ>
__device__ __forceinline__ void multiply_chunk(double (&acc)[KT][kSlots][2], const double* __restrict__ xd,
                                               const double* __restrict__ md, const int (&b_off)[kSlots], int inner) {
#pragma unroll
  for (int s = 0; s < kKC / 4; ++s) {
    double a[KT], b[NQ];
#pragma unroll
    for (int i = 0; i < KT; ++i) a[i] = md[(s * KT + i) * 32];
#pragma unroll
    for (int q = 0; q < NQ; ++q) b[q] = xd[b_off[q] + 4 * s * inner];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < KT; ++i) dmma884(acc[i][q][0], acc[i][q][1], a[i], b[q]);
  }
}

// Persistent CTA: K block blockIdx.y; tiles blockIdx.x, blockIdx.x + gridDim.x, ... of kSlabs slabs each.
template <int KT>
__global__ void __launch_bounds__(kThreads, 2) ttm_packed_kernel(const PackedParams p) {
  constexpr int MS = (kKC / 4) * KT * 32;  // doubles per stage of factor fragments
  extern __shared__ __align__(16) double smem[];
  const int inner = p.inner;
  const int run = kKC * inner;             // doubles of one slab's chunk
  const int XS = kSlabs * run;             // doubles per stage of X
  double* const xs = smem;
  double* const ms = smem + kStages * XS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int kb = blockIdx.y;
  const long long n_tiles = (p.outer + kSlabs - 1) / kSlabs;
  const long long my_tiles = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const long long total_items = my_tiles * p.n_chunks;
  auto tile_slab0 = [&](long long j) { return (static_cast<long long>(blockIdx.x) + j * gridDim.x) * kSlabs; };
  const double* const mfrag_kb = p.mfrag + static_cast<long long>(kb) * p.n_chunks * MS;

  // B fragment: this lane's column g of its n-tiles -> offset of (slab, b) inside a stage; C fragment: its two
  // columns 2t, 2t + 1 -> (slab, b) for the stores
  const int used_tiles = 4 * inner;
  const int my_slots = used_tiles > warp ? (used_tiles - warp + kWarps - 1) / kWarps : 0;  // slots q with a tile
  int b_off[kSlots], c_slab[kSlots][2], c_b[kSlots][2];
#pragma unroll
  for (int q = 0; q < kSlots; ++q) {
    const int j = warp + kWarps * q;
    const int c = 8 * j + g;
    b_off[q] = (c / inner) * run + c % inner;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cc = 8 * j + 2 * t + e;
      c_slab[q][e] = cc / inner;
      c_b[q][e] = cc % inner;
    }
  }

  // loader: 16-byte units, unit u of a slab's run = its doubles [2u, 2u + 2).  A run has 8 * inner units and the
  // CTA 8 threads per slab: thread (slab ld_s, ld_u0) copies units ld_u0, ld_u0 + 8, ... -- `inner` copies per chunk,
  // 128 contiguous bytes per slab and step, no index arithmetic beyond two additions
  const int ld_s = tid >> 3, ld_u0 = tid & 7;
  auto issue_chunk = [&](long long j, int chunk, int stage) {
    const long long a = tile_slab0(j) + ld_s;
    const long long l0 = static_cast<long long>(chunk) * kKC;
    const int valid_units = static_cast<int>(min(static_cast<long long>(kKC), p.len - l0)) * inner / 2;
    const bool slab_ok = a < p.outer;
    const double* src = p.x + (a * p.len + l0) * inner + 2 * ld_u0;
    double* dst = xs + stage * XS + ld_s * run + 2 * ld_u0;
    for (int u = ld_u0; u < 8 * inner; u += 8) {
      const bool ok = slab_ok && u < valid_units;
      cp_async16(dst, ok ? src : p.x, ok);
      src += 16;
      dst += 16;
    }
    const double* msrc = mfrag_kb + static_cast<long long>(chunk) * MS;
    double* const md = ms + stage * MS;
    for (int idx = tid; idx < MS / 2; idx += kThreads) cp_async16(md + 2 * idx, msrc + 2 * idx, true);
  };

  double acc[KT][kSlots][2];
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int q = 0; q < kSlots; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;

  auto store_tile = [&](long long j) {
    const long long a0 = tile_slab0(j);
#pragma unroll
    for (int q = 0; q < kSlots; ++q) {
      if (warp + kWarps * q >= used_tiles) continue;  // uniform in the warp
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const long long k = static_cast<long long>(kb) * (8 * KT) + 8 * i + g;
        if (k >= p.new_len) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const long long a = a0 + c_slab[q][e];
          if (a < p.outer) p.z[(a * p.new_len + k) * inner + c_b[q][e]] = acc[i][q][e];
        }
      }
    }
  };

  long long load_j = 0, cons_j = 0;
  int load_c = 0, cons_c = 0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (load_j < my_tiles) {
      issue_chunk(load_j, load_c, s);
      if (++load_c == p.n_chunks) {
        load_c = 0;
        ++load_j;
      }
    }
    cp_async_commit();
  }
  int load_stage = kStages - 1, cons_stage = 0;

  for (long long it = 0; it < total_items; ++it) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (load_j < my_tiles) {
      issue_chunk(load_j, load_c, load_stage);
      if (++load_c == p.n_chunks) {
        load_c = 0;
        ++load_j;
      }
    }
    cp_async_commit();
    load_stage = (load_stage + 1 == kStages) ? 0 : load_stage + 1;

    const double* const xd = xs + cons_stage * XS + t * inner;
    const double* const md = ms + cons_stage * MS + lane;
    cons_stage = (cons_stage + 1 == kStages) ? 0 : cons_stage + 1;
    // the warp's live slots as a compile-time count: a guard around a DMMA becomes a predicate, and a predicated-off
    // DMMA still takes its turn on the tensor pipe
    switch (my_slots) {
      case 1: multiply_chunk<KT, 1>(acc, xd, md, b_off, inner); break;
      case 2: multiply_chunk<KT, 2>(acc, xd, md, b_off, inner); break;
      case 3: multiply_chunk<KT, 3>(acc, xd, md, b_off, inner); break;
      case 4: multiply_chunk<KT, 4>(acc, xd, md, b_off, inner); break;
      default: break;
    }
    if (++cons_c == p.n_chunks) {
      store_tile(cons_j);
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int q = 0; q < kSlots; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
      cons_c = 0;
      ++cons_j;
    }
  }
  cp_async_wait<0>();
}

template <int KT>
cudaError_t launch_packed(cudaStream_t stream, const PackedParams& p, int k_blocks, int sm_count) {
  const size_t smem = sizeof(double) * kStages * (static_cast<size_t>(kSlabs) * kKC * p.inner + (kKC / 4) * KT * 32);
  auto kernel = ttm_packed_kernel<KT>;
  static PerDeviceInt configured;
  std::atomic<int>* const slot = configured.slot();
  if (!slot || !slot->load(std::memory_order_relaxed)) {
    const size_t most = sizeof(double) * kStages * (static_cast<size_t>(kSlabs) * kKC * 8 + (kKC / 4) * KT * 32);
    const cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(most));
    if (e != cudaSuccess) return e;
    if (slot) slot->store(1, std::memory_order_relaxed);
  }
  static PerDeviceInt resident_ctas[9];  // per device and inner: CTAs of this shared-memory size an SM holds
  std::atomic<int>* const occ_slot = resident_ctas[p.inner].slot();
  int occ = occ_slot ? occ_slot->load(std::memory_order_relaxed) : 0;
  if (occ == 0) {
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
    if (occ_slot) occ_slot->store(occ, std::memory_order_relaxed);
  }
  const long long tiles = (p.outer + kSlabs - 1) / kSlabs;
  const long long resident = std::max(1LL, static_cast<long long>(sm_count) * occ / k_blocks);
  dim3 grid(static_cast<unsigned>(std::min(tiles, resident)), static_cast<unsigned>(k_blocks));
  kernel<<<grid, kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

std::atomic<bool>& ttm_packed_enabled() {
  static std::atomic<bool> on{true};
  return on;
}

bool ttm_packed_eligible(const double* x, long long outer, long long len, long long inner, const double* z, int kt,
                         int n_dest) {
  if (!ttm_packed_enabled().load(std::memory_order_relaxed)) return false;
  // inner == 8 is dense in the general kernels already; larger K blocks would not fit the accumulators
  if (inner < 2 || inner > 7 || kt > 4 || n_dest != 1 || outer < 1) return false;
  if ((len * inner) % 2 != 0) return false;  // every slab, hence every run of a chunk, starts 16-byte aligned
  return reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(z) % 8 == 0;
}

cudaError_t launch_ttm_packed(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                              const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z,
                              int sm_count) {
  PackedParams p;
  p.x = x;
  p.z = z;
  p.mfrag = mfrag;
  p.outer = outer;
  p.len = len;
  p.new_len = new_len;
  p.inner = static_cast<int>(inner);
  p.n_chunks = f.n_chunks;
  switch (f.kt) {
    case 1: return launch_packed<1>(stream, p, f.k_blocks, sm_count);
    case 2: return launch_packed<2>(stream, p, f.k_blocks, sm_count);
    case 3: return launch_packed<3>(stream, p, f.k_blocks, sm_count);
    case 4: return launch_packed<4>(stream, p, f.k_blocks, sm_count);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpb
