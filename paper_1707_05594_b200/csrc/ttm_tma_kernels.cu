// Mode-n TTM, warp-specialised TMA pipeline (the fast path of launch_ttm for aligned, even extents).
//
// Same arithmetic and tiling as ttm_kernels.cu (DMMA.8x8x4, M = MMA A operand in fragment order, 8-column n-tiles
// of X = B operand, persistent CTAs), but the data movement is the Blackwell way:
//
//   * warp 0 is a PRODUCER: one elected lane issues cp.async.bulk.tensor (TMA) loads of 16 x 16-double boxes of X
//     — straight from the strided unfolding through a 3-D tensor map ((inner, L, outer), or (L, outer, 1) when inner == 1), rows and
//     columns beyond the extents zero-filled by the hardware — plus one cp.async.bulk of the factor-fragment chunk,
//     all completing on the stage's `full` mbarrier (expect_tx);
//   * warps 1..8 are CONSUMERS: they wait on `full`, run their KT x NT DMMA tiles, and arrive on the stage's `empty`
//     mbarrier.  There is no CTA-wide barrier in the main loop, so loads run up to STAGES chunks ahead regardless of
//     where the consumers are, and the consumer warps drift apart instead of bursting on the DMMA pipe together.
//   * boxes land in shared memory with the hardware 128-byte swizzle (16-byte chunk index XOR row & 7).  The MMA
//     fragment mapping is chosen so that the 64-bit loads of a half-warp stay conflict-free under that swizzle:
//     for inner > 1 the four k-indices of a DMMA map to rows {0,2,4,6} (then {1,3,5,7}) of an 8-row group — the
//     factor fragments are prepared with the same interleave; for inner == 1 the eight n-indices map to rows
//     {0,2,4,6,1,3,5,7} of their half box.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kKC = 16;  // contraction steps per stage = rows (or l-values) of one TMA box
constexpr bool kSkewConsumers = true;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct TmaParams {
  double* __restrict__ z;
  const double* __restrict__ mfrag;  // [k blocks][chunks][4 steps][KT][32], rows interleaved for !LAST
  long long outer, len, inner, new_len;
  long long n_boxes;      // 16-column boxes (inner > 1) or 16-row boxes (inner == 1)
  int boxes_per_slab;     // inner > 1: ceil(inner / 16)
  int n_chunks;           // ceil(len / 16)
  int n_dest;
  int dest_k0[kMaxTtmDest + 1];
  long long dest_off[kMaxTtmDest];
};

// One stage (kKC contraction steps) for the first NL n-tiles of a consumer warp.  NL is a compile-time count on
// purpose: a run-time guard around a DMMA is compiled into a predicate, and a predicated-off DMMA still takes its
// turn on the tensor pipe -- skipping dead tiles has to be a branch to another instantiation.
template <int KT, int NT, int NL, bool LAST>
__device__ __forceinline__ void consume_stage(double (&acc)[KT][NT][2], const double* __restrict__ xd,
                                              const double* __restrict__ md, const int (&frag_off)[4], int cw) {
#pragma unroll
  for (int s = 0; s < kKC / 4; ++s) {
    double a[KT], b[NL];
#pragma unroll
    for (int i = 0; i < KT; ++i) a[i] = md[(s * KT + i) * 32];
#pragma unroll
    for (int jj = 0; jj < NL; ++jj) {
      const int t = cw * NT + jj;
      const double* const box = xd + (t >> 1) * (kKC * 16);
      // the half-box term: LAST -> rows 8..15 (offset 8 * 16, same swizzle since 8 & 7 == 0);
      //                    !LAST -> columns 8..15 = chunks 4..7 -> XOR with 4 on the chunk index = +/- 8 doubles
      b[jj] = LAST ? box[frag_off[s] + (t & 1) * (8 * 16)] : box[frag_off[s] ^ ((t & 1) << 3)];
    }
#pragma unroll
    for (int jj = 0; jj < NL; ++jj)
#pragma unroll
      for (int i = 0; i < KT; ++i) dmma884(acc[i][jj][0], acc[i][jj][1], a[i], b[jj]);
  }
}

template <int KT, int NT, int STAGES, bool LAST>
__global__ void __launch_bounds__(kThreads, (KT * NT <= 12) ? 2 : 1)
    ttm_tma_kernel(const __grid_constant__ CUtensorMap xmap, const TmaParams p) {
  constexpr int TILE_N = kConsumerWarps * NT;   // n-tiles per CTA tile
  constexpr int BOXES = TILE_N / 2;             // TMA boxes per stage (two n-tiles each)
  constexpr int XS = BOXES * kKC * 16;          // doubles per stage of X
  constexpr int MS = (kKC / 4) * KT * 32;       // doubles per stage of factor fragments
  constexpr unsigned STAGE_BYTES = (XS + MS) * sizeof(double);
  static_assert(TILE_N % 2 == 0, "a box holds two n-tiles");

  extern __shared__ unsigned char smem_raw[];
  // [STAGES][XS] boxes (each 2 KB; the base is rounded up to 1 KB so that the hardware swizzle, which works on
  // shared-memory address bits, lines up with the box rows), then [STAGES][MS], then the barriers
  unsigned char* const smem_aligned = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* const xs = reinterpret_cast<double*>(smem_aligned);
  double* const ms = xs + STAGES * XS;
  uint64_t* const full = reinterpret_cast<uint64_t*>(ms + STAGES * MS);
  uint64_t* const empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = blockIdx.y;
  // Balanced partition: CTA b owns the contiguous box range [b n / G, (b+1) n / G) and walks it in tiles of BOXES
  // boxes; boxes of the last tile beyond the range are neither loaded (their TMA coordinates are out of bounds ->
  // zero fill, no memory traffic) nor stored.
  const long long cta_begin = static_cast<long long>(blockIdx.x) * p.n_boxes / gridDim.x;
  const long long cta_end = static_cast<long long>(blockIdx.x + 1) * p.n_boxes / gridDim.x;
  const long long my_tiles = (cta_end - cta_begin + BOXES - 1) / BOXES;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    // the barriers are signalled by the TMA unit (async proxy): make their initialisation visible to it, and to
    // the other threads, before anyone arms or polls them
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  auto first_box = [&](long long j) { return cta_begin + j * BOXES; };

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const double* const mfrag_kb = p.mfrag + static_cast<long long>(kb) * p.n_chunks * MS;
      int stage = 0;
      unsigned parity = 0;
      for (long long j = 0; j < my_tiles; ++j) {
        // box coordinates of this tile: (slab, first column) for inner > 1, first row for inner == 1
        int box_c0[BOXES], box_c2[BOXES];
        const long long g0 = first_box(j);
#pragma unroll
        for (int q = 0; q < BOXES; ++q) {
          const long long g = g0 + q < cta_end ? g0 + q : p.n_boxes;  // past the range -> out of bounds
          if (LAST) {
            box_c0[q] = static_cast<int>(g * 16);  // first row; n_boxes * 16 >= outer -> all zero fill
            box_c2[q] = 0;
          } else {
            const unsigned a = static_cast<unsigned>(g) / static_cast<unsigned>(p.boxes_per_slab);
            box_c0[q] = static_cast<int>(static_cast<unsigned>(g) - a * p.boxes_per_slab) * 16;
            box_c2[q] = static_cast<int>(a);  // a == outer for boxes past the end -> zero fill
          }
        }
        for (int chunk = 0; chunk < p.n_chunks; ++chunk) {
          mbar_wait(&empty[stage], parity ^ 1u);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          double* const xd = xs + stage * XS;
#pragma unroll
          for (int q = 0; q < BOXES; ++q) {
            if (LAST)
              tma_load_3d(xd + q * (kKC * 16), &xmap, &full[stage], chunk * kKC, box_c0[q], 0);
            else
              tma_load_3d(xd + q * (kKC * 16), &xmap, &full[stage], box_c0[q], chunk * kKC, box_c2[q]);
          }
          bulk_load(ms + stage * MS, mfrag_kb + static_cast<long long>(chunk) * MS, MS * sizeof(double), &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            parity ^= 1u;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int cw = warp - 1;
  double acc[KT][NT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // per-lane fragment offsets inside a box (doubles), one per k-step; see the header comment for the mappings
  const int fk = lane & 3, fn = lane >> 2;
  int frag_off[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (LAST) {
      const int row = ((fn & 3) << 1) | (fn >> 2);            // n index -> row {0,2,4,6,1,3,5,7} of the half box
      const int l = 4 * s + fk;                               // consecutive l
      frag_off[s] = row * 16 + ((((l >> 1) ^ (row & 7)) << 1) | (l & 1));
    } else {
      const int l = 8 * (s >> 1) + 2 * fk + (s & 1);          // k index -> rows {0,2,4,6} / {1,3,5,7}
      const int col = fn;                                     // + 8 * half added below
      frag_off[s] = l * 16 + ((((col >> 1) ^ (l & 7)) << 1) | (col & 1));
    }
  }

  // The two consumer warps of an SM sub-partition (cw and cw + 4) run the same code on the same stages at the same
  // rate, so left alone they reach every stage boundary -- barrier wait, fence, arrive, no DMMA in flight --
  // together and the FP64 pipe of their sub-partition idles for the length of it.  Half a stage of head start for
  // one of them lasts for the whole kernel (both advance at the pipe's pace) and puts each warp's boundary under the
  // other's DMMAs.
  if (kSkewConsumers && cw >= kConsumerWarps / 2) {
    const long long t0 = clock64();
    while (clock64() - t0 < static_cast<long long>(KT) * NT * 64) {
    }
  }
  int stage = 0;
  unsigned parity = 0;
  for (long long j = 0; j < my_tiles; ++j) {
    // n-tiles of this warp whose box lies inside the CTA's range: the balanced partition hands small problems less
    // than a full tile per CTA, and multiplying the zero-filled rest would cost as many DMMAs as the real part
    // (the live n-tiles of a warp are a prefix of its NT: the boxes past the range are the last ones of the tile)
    int n_live = 0;
#pragma unroll
    for (int jj = 0; jj < NT; ++jj) n_live += first_box(j) + ((cw * NT + jj) >> 1) < cta_end ? 1 : 0;
    for (int chunk = 0; chunk < p.n_chunks; ++chunk) {
      mbar_wait(&full[stage], parity);
      const double* const xd = xs + stage * XS;
      const double* const md = ms + stage * MS + lane;
      if (n_live == NT) {
        consume_stage<KT, NT, NT, LAST>(acc, xd, md, frag_off, cw);
      } else if (NT >= 4 && n_live == 3) {
        consume_stage<KT, NT, (NT >= 4 ? 3 : 1), LAST>(acc, xd, md, frag_off, cw);
      } else if (NT >= 2 && n_live == 2) {
        consume_stage<KT, NT, (NT >= 2 ? 2 : 1), LAST>(acc, xd, md, frag_off, cw);
      } else if (n_live == 1) {
        consume_stage<KT, NT, 1, LAST>(acc, xd, md, frag_off, cw);
      }
      // The stage was read with ordinary (generic-proxy) shared loads; the producer will refill it through the TMA
      // unit (async proxy).  Ordering across the two proxies needs this fence before the stage is handed back —
      // without it a refill can overtake the reads (seen as stale 128-byte box rows when other kernels share the SMs).
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        parity ^= 1u;
      }
    }
    // ---- epilogue of tile j: rows k = 8 i + lane/4, n indices 2 (lane%4), +1 of each n-tile
    const long long g0 = first_box(j);
#pragma unroll
    for (int jj = 0; jj < NT; ++jj) {
      const int t = cw * NT + jj;
      const long long g = g0 + (t >> 1);
      const int half = t & 1;
      if (g < cta_end) {
        long long slab = 0;
        int c0 = 0;
        if (!LAST) {
          const unsigned a = static_cast<unsigned>(g) / static_cast<unsigned>(p.boxes_per_slab);
          slab = a;
          c0 = static_cast<int>(static_cast<unsigned>(g) - a * p.boxes_per_slab) * 16 + 8 * half;
        }
#pragma unroll
        for (int i = 0; i < KT; ++i) {
          const long long k_abs = static_cast<long long>(kb) * (8 * KT) + 8 * i + (lane >> 2);
          if (k_abs < p.new_len) {
            int d = 0;
            while (d + 1 < p.n_dest && k_abs >= p.dest_k0[d + 1]) ++d;
            const long long k = k_abs - p.dest_k0[d];
            const long long rows_d = p.dest_k0[d + 1] - p.dest_k0[d];
            double* const zd = p.z + p.dest_off[d];
            if (LAST) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int n = 2 * (lane & 3) + e;
                const long long row = g * 16 + 8 * half + (((n & 3) << 1) | (n >> 2));
                if (row < p.outer) zd[row * rows_d + k] = acc[i][jj][e];
              }
            } else {
              const long long b = c0 + 2 * (lane & 3);
              if (b < p.inner)  // inner is even on this path: the pair is in or out together
                *reinterpret_cast<double2*>(zd + (slab * rows_d + k) * p.inner + b) =
                    make_double2(acc[i][jj][0], acc[i][jj][1]);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < KT; ++i) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    }
  }
}

// ---- host side -------------------------------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* sym = nullptr;
    cudaDriverEntryPointQueryResult status;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &sym, cudaEnableDefault, &status) == cudaSuccess &&
        status == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(sym);
  });
  return fn;
}

// Tensor maps are functions of (base address, extents) only, and a plan launches the same few products every sweep:
// the encoded maps are kept in a small per-thread table (a context is used from one host thread) instead of being
// rebuilt by the driver on every launch.  Entries are replaced round-robin.
struct MapKey {
  const double* x = nullptr;
  long long outer = 0, len = 0, inner = 0;
  bool operator==(const MapKey& o) const { return x == o.x && outer == o.outer && len == o.len && inner == o.inner; }
};

const CUtensorMap* tensor_map_for(const double* x, long long outer, long long len, long long inner) {
  constexpr int kSlots = 64;
  struct Table {
    MapKey key[kSlots];
    alignas(64) CUtensorMap map[kSlots];
    int next = 0;
  };
  thread_local Table table;
  const MapKey want{x, outer, len, inner};
  for (int i = 0; i < kSlots; ++i)
    if (table.key[i] == want) return &table.map[i];
  const int at = table.next;
  table.next = (table.next + 1) % kSlots;
  CUtensorMap* const map = &table.map[at];
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const cuuint32_t box[3] = {16, 16, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r;
  if (inner == 1) {
    // (L, outer) viewed as a 3-D map with a unit slowest dimension: both modes then use the same 3-D TMA path
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(outer), 1};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(len) * 8, static_cast<cuuint64_t>(len) * outer * 8};
    r = encode_tiled()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(len),
                                static_cast<cuuint64_t>(outer)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner) * 8, static_cast<cuuint64_t>(len) * inner * 8};
    r = encode_tiled()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    table.key[at] = MapKey{};
    return nullptr;
  }
  table.key[at] = want;
  return map;
}

template <int KT, int NT, int STAGES, bool LAST>
cudaError_t launch_tma_one(cudaStream_t stream, const CUtensorMap& map, const TmaParams& p, int k_blocks,
                           int sm_count) {
  constexpr int TILE_N = kConsumerWarps * NT;
  constexpr int BOXES = TILE_N / 2;
  constexpr size_t smem = sizeof(double) * STAGES * (BOXES * kKC * 16 + (kKC / 4) * KT * 32) + 2 * STAGES * 8 + 1024;
  auto kernel = ttm_tma_kernel<KT, NT, STAGES, LAST>;
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
  const long long resident = std::max(1LL, static_cast<long long>(sm_count) * ctas_per_sm / k_blocks);
  // every resident CTA gets an equal share of the boxes (at least half a tile each, else fewer CTAs)
  const long long useful = std::max(1LL, (p.n_boxes * 2 + BOXES - 1) / BOXES);
  dim3 grid(static_cast<unsigned>(std::min(useful, resident)), static_cast<unsigned>(k_blocks));
  kernel<<<grid, kThreads, smem, stream>>>(map, p);
  return cudaGetLastError();
}

template <int KT>
cudaError_t launch_tma_kt(cudaStream_t stream, const CUtensorMap& map, const TmaParams& p, int k_blocks, bool last,
                          int sm_count) {
  constexpr int NT = (KT <= 5) ? 4 : 2;
  // stage = X boxes (NT=4: 32 KB, NT=2: 16 KB) + factor chunk (KT * 1 KB).  Up to KT*NT = 12 accumulator tiles two
  // CTAs share an SM (3 stages each); beyond that the registers allow one CTA, which then takes a deeper ring
  // (KT = 13: 7 stages = 203 KB; measured on the C5 root product: 24.18 ms with 6 stages, 24.15 with 7).
  constexpr int STAGES = (KT * NT <= 12) ? 3 : ((NT == 4) ? 5 : (KT == 13 ? 7 : 6));
  return last ? launch_tma_one<KT, NT, STAGES, true>(stream, map, p, k_blocks, sm_count)
              : launch_tma_one<KT, NT, STAGES, false>(stream, map, p, k_blocks, sm_count);
}

}  // namespace

const void* ttm_tensor_map(const double* x, long long outer, long long len, long long inner) {
  if (!encode_tiled()) return nullptr;
  return tensor_map_for(x, outer, len, inner);
}

bool ttm_tma_eligible(const double* x, long long outer, long long len, long long inner, const double* z, int kt,
                      int k_blocks, int sm_count) {
  if (!encode_tiled()) return false;
  if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(z) % 16) return false;
  const bool last = inner == 1;
  if ((last ? len : inner) % 2) return false;                              // 16-byte global strides
  if (outer >= (1LL << 31) || len >= (1LL << 31) || inner >= (1LL << 31)) return false;
  const int tile_n = kConsumerWarps * ((kt <= 5) ? 4 : 2);
  const long long boxes = last ? (outer + 15) / 16 : outer * ((inner + 15) / 16);
  if (boxes >= (1LL << 31)) return false;
  // at least one full tile per SM; smaller problems are faster on the narrow cp.async kernel (measured: the TMA
  // pipeline's start-up costs ~5 us more)
  return boxes * k_blocks >= static_cast<long long>(tile_n / 2) * sm_count;
}

cudaError_t launch_ttm_tma(cudaStream_t stream, const double* x, long long outer, long long len, long long inner,
                           const double* mfrag, const TtmFragmentLayout& f, long long new_len, double* z,
                           int sm_count, int n_dest, const long long* dest_cuts, const long long* dest_offsets) {
  const bool last = inner == 1;
  TmaParams p;
  p.z = z;
  p.mfrag = mfrag;
  p.outer = outer;
  p.len = len;
  p.inner = inner;
  p.new_len = new_len;
  p.n_chunks = f.n_chunks;
  p.boxes_per_slab = last ? 1 : static_cast<int>((inner + 15) / 16);
  p.n_boxes = last ? (outer + 15) / 16 : outer * p.boxes_per_slab;
  if (n_dest < 1 || n_dest > kMaxTtmDest) return cudaErrorInvalidValue;
  p.n_dest = n_dest;
  long long off = 0;
  for (int d = 0; d < n_dest; ++d) {
    const long long k0 = dest_cuts ? dest_cuts[d] : 0, k1 = dest_cuts ? dest_cuts[d + 1] : new_len;
    p.dest_k0[d] = static_cast<int>(k0);
    p.dest_k0[d + 1] = static_cast<int>(k1);
    p.dest_off[d] = dest_offsets ? dest_offsets[d] : off;
    if (p.dest_off[d] % 2) return cudaErrorInvalidValue;  // caller checks eligibility; chunks must stay 16-byte aligned
    off += outer * (k1 - k0) * inner;
  }
  for (int d = n_dest + 1; d <= kMaxTtmDest; ++d) p.dest_k0[d] = p.dest_k0[n_dest];
  for (int d = n_dest; d < kMaxTtmDest; ++d) p.dest_off[d] = 0;

  const CUtensorMap* cached = tensor_map_for(x, outer, len, inner);
  if (!cached) return cudaErrorInvalidValue;
  const CUtensorMap& map = *cached;

  switch (f.kt) {
    case 1: return launch_tma_kt<1>(stream, map, p, f.k_blocks, last, sm_count);
    case 2: return launch_tma_kt<2>(stream, map, p, f.k_blocks, last, sm_count);
    case 3: return launch_tma_kt<3>(stream, map, p, f.k_blocks, last, sm_count);
    case 4: return launch_tma_kt<4>(stream, map, p, f.k_blocks, last, sm_count);
    case 5: return launch_tma_kt<5>(stream, map, p, f.k_blocks, last, sm_count);
    case 6: return launch_tma_kt<6>(stream, map, p, f.k_blocks, last, sm_count);
    case 8: return launch_tma_kt<8>(stream, map, p, f.k_blocks, last, sm_count);
    case 10: return launch_tma_kt<10>(stream, map, p, f.k_blocks, last, sm_count);
    case 13: return launch_tma_kt<13>(stream, map, p, f.k_blocks, last, sm_count);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpb
