// Gram matrix of a mode-n unfolding for LARGE leaves: 128 x 128 tiles, warp-specialised TMA pipeline.
//
//   G(i, j) = sum_{a, b} Y(a, i, b) * Y(a, j, b)        Y viewed as (outer, rows, inner)
//
// Same sums as gram_kernels.cu (replaces reference unfold() + rankUpdate(), ttm.hpp:43-53, hooi.hpp:53-54), different
// data movement.  The 64 x 64 cp.async kernel moves 16 KB from L2 per 64 x 64 x 16 block of MACs -- 16 bytes per
// clock and SM at the DMMA rate, 4.6 TB/s over the chip, more than L2 delivers: it stalls at 78 % of the pipe
// (profiles/r02_v1_ncu_full_gram_summary.txt).  Here a CTA owns a 128 x 128 tile (half the operand traffic per MAC):
//
//   * warp 0 is the PRODUCER (its warpgroup gives its registers to the consumers, setmaxnreg): one lane issues cp.async.bulk.tensor loads of 16 x 16-double boxes (the tensor maps of
//     the TTM kernel: (inner, rows, outer) or (rows, outer, 1) when inner == 1), 8 boxes per operand and stage, rows
//     past the extent zero-filled by the hardware; a 4-stage ring, full / empty mbarriers, no CTA-wide barrier;
//   * warps 4..11 are CONSUMERS on DMMA.8x8x4.  The tile is cut into 4 x 4 blocks of 32 x 32; a consumer owns up to two
//     blocks.  Off the diagonal that is a 64 x 32 piece per warp.  On the diagonal only the ten blocks with
//     row block >= column block are computed, dealt out so that the two warps of every SM sub-partition hold at most
//     three between them (the FP64 pipe is per sub-partition): a diagonal tile costs 3/4 of a full one instead of all
//     of it.  Blocks whose rows lie past the extent are skipped the same way (whole blocks, by branching: a
//     predicated-off DMMA still takes its turn on the pipe);
//   * persistent CTAs walk a static list of (split, tile) items -- split by split, the tiles of a split dearest first
//     (full tiles, diagonal tiles, the ragged last tile row) -- item i to CTA i mod G; the producer runs ahead across item boundaries, so the pipeline is filled
//     once per CTA, not once per tile;
//   * the contraction range is split as before and the partial tiles are summed in split order by gram_reduce_kernel
//     (deterministic, whichever CTA computed a partial tile).
//
// Shared-memory fragment mappings (both conflict-free under the 128-byte hardware swizzle, cf. ttm_tma_kernels.cu):
// inner > 1 (contraction contiguous, box = [16 rows][16 k]): fragment row index n -> box row {0,2,4,6,1,3,5,7}[n];
// inner == 1 (rows contiguous, box = [16 k][16 rows]): the four k-indices of a DMMA -> box rows {0,2,4,6}/{1,3,5,7}.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kProducerWarps = 4;  // one warpgroup: setmaxnreg works on whole warpgroups; only warp 0 issues loads
constexpr int kThreads = 32 * (kProducerWarps + kConsumerWarps);
constexpr int kKC = 16;
constexpr int kTile = 128;
constexpr int kStages = 4;
constexpr int kBoxDoubles = 16 * 16;
constexpr int kOperandDoubles = (kTile / 16) * kBoxDoubles;  // 16 KB
constexpr size_t kSmemBytes = sizeof(double) * kStages * 2 * kOperandDoubles + 2 * kStages * 8 + 1024;

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
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct GramTmaParams {
  double* __restrict__ partial;  // [splits][rows][rows]
  long long rows;
  long long chunks, chunks_per_split;
  int chunks_per_slab;  // inner > 1: ceil(inner / 16)
  int splits;
  int tile_rows;        // T = ceil(rows / 128)
  int n_items;          // lower tiles x splits
};

// item -> (ti, tj, split).  Splits outermost: the CTAs running at any moment then share one slice of the contraction
// range (all rows x 1 / splits of the columns, ~10 MB at C5) and every operand box is read from DRAM once -- with the
// tiles outermost the walk cycles through whole row blocks of the leaf and misses L2 on most of them (measured:
// 780 MB of DRAM reads for a 128 MB leaf).  Tiles of a split in cost order: strictly-lower tiles of the full tile
// rows, their diagonal tiles, the last tile row's off-diagonal tiles, the last diagonal tile.
__device__ __forceinline__ void decode_item(const GramTmaParams& p, int item, int& ti, int& tj, int& split) {
  const int t = p.tile_rows;
  const int n_tiles = t * (t + 1) / 2;
  split = item / n_tiles;
  const int q = item - split * n_tiles;
  const int n_lower = (t - 1) * (t - 2) / 2;
  if (q < n_lower) {
    ti = 1;
    int rest = q;
    while (rest >= ti) {
      rest -= ti;
      ++ti;
    }
    tj = rest;
  } else if (q < n_lower + (t - 1)) {
    ti = tj = q - n_lower;
  } else if (q < n_lower + 2 * (t - 1)) {
    ti = t - 1;
    tj = q - n_lower - (t - 1);
  } else {
    ti = tj = t - 1;
  }
}

// The up to two 32 x 32 blocks (row block << 4 | column block, -1 = none) of consumer warp cw.  Consumers cw and
// cw + 4 share an SM sub-partition (warp w runs on sub-partition w % 4).
__device__ __forceinline__ void warp_blocks(bool diag, int cw, int& b0, int& b1) {
  if (!diag) {
    const int wm = cw >> 2, wn = cw & 3;
    b0 = ((2 * wm) << 4) | wn;
    b1 = ((2 * wm + 1) << 4) | wn;
    return;
  }
  switch (cw) {
    case 0: b0 = 0x00; b1 = 0x10; break;
    case 4: b0 = 0x11; b1 = -1; break;
    case 1: b0 = 0x20; b1 = 0x30; break;
    case 5: b0 = 0x21; b1 = -1; break;
    case 2: b0 = 0x22; b1 = 0x32; break;
    case 3: b0 = 0x31; b1 = 0x33; break;
    default: b0 = b1 = -1; break;
  }
}

// One stage of one 32 x 32 block: pa / pb = the operand tiles at the block's first row / column (32-row blocks are
// 512 doubles apart in both layouts).  8-row group a of the block: inner > 1 -> box a / 2, rows 8 (a % 2).. of it;
// inner == 1 -> box a / 2, columns 8 (a % 2).. of it = XOR 8 on the fragment offset.
// (Skipping the zero-filled k-steps of a slab's short last chunk -- inner = 100 pads to 112 -- by branching to
// instantiations with fewer steps was measured: -1 % on that shape, +8 % on the others from the larger loop body.)
template <bool INNER1>
__device__ __forceinline__ void consume_block(double (&acc)[4][4][2], const double* __restrict__ pa,
                                              const double* __restrict__ pb, const int (&frag_off)[4]) {
#pragma unroll
  for (int s = 0; s < kKC / 4; ++s) {
    double fa[4], fb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int at = (a >> 1) * kBoxDoubles + (INNER1 ? (frag_off[s] ^ ((a & 1) << 3)) : frag_off[s] + (a & 1) * (8 * 16));
      fa[a] = pa[at];
      fb[a] = pb[at];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
  }
}

template <bool INNER1>
__global__ void __launch_bounds__(kThreads, 1)
    gram_tma_kernel(const __grid_constant__ CUtensorMap ymap, const GramTmaParams p) {
  extern __shared__ unsigned char smem_raw[];
  // boxes are 2 KB with a swizzle pattern on shared-memory address bits: 1 KB alignment of the first box
  unsigned char* const smem_aligned = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* const sa = reinterpret_cast<double*>(smem_aligned);      // [kStages][kOperandDoubles]
  double* const sb = sa + kStages * kOperandDoubles;               // [kStages][kOperandDoubles]
  uint64_t* const full = reinterpret_cast<uint64_t*>(sb + kStages * kOperandDoubles);
  uint64_t* const empty = full + kStages;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  // Register split (the register file is per SM sub-partition: a ninth warp would cap every thread at 168 registers
  // and spill the consumers' 128 accumulator registers + fragments): the kernel starts with 168 per thread for its
  // three warpgroups, the producer group hands back all but 40, the two consumer groups grow to 232.
  if (warp < kProducerWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    // ------------------------------------------------------------------ producer
    if (warp == 0 && lane == 0) {
      int stage = 0;
      unsigned parity = 0;
      for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        int ti, tj, split;
        decode_item(p, item, ti, tj, split);
        const bool diag = ti == tj;
        const long long c_begin = static_cast<long long>(split) * p.chunks_per_split;
        const long long c_end = min(p.chunks, c_begin + p.chunks_per_split);
        const unsigned bytes = (diag ? 1u : 2u) * kOperandDoubles * sizeof(double);
        for (long long c = c_begin; c < c_end; ++c) {
          int k0, slab;
          if (INNER1) {
            k0 = static_cast<int>(c * kKC);
            slab = 0;
          } else {
            const long long a = c / p.chunks_per_slab;
            k0 = static_cast<int>(c - a * p.chunks_per_slab) * kKC;
            slab = static_cast<int>(a);
          }
          mbar_wait(&empty[stage], parity ^ 1u);
          mbar_expect_tx(&full[stage], bytes);
          double* const da = sa + stage * kOperandDoubles;
          double* const db = sb + stage * kOperandDoubles;
#pragma unroll
          for (int q = 0; q < kTile / 16; ++q) {
            if (INNER1)
              tma_load_3d(da + q * kBoxDoubles, &ymap, &full[stage], ti * kTile + 16 * q, k0, 0);
            else
              tma_load_3d(da + q * kBoxDoubles, &ymap, &full[stage], k0, ti * kTile + 16 * q, slab);
          }
          if (!diag) {
#pragma unroll
            for (int q = 0; q < kTile / 16; ++q) {
              if (INNER1)
                tma_load_3d(db + q * kBoxDoubles, &ymap, &full[stage], tj * kTile + 16 * q, k0, 0);
              else
                tma_load_3d(db + q * kBoxDoubles, &ymap, &full[stage], k0, tj * kTile + 16 * q, slab);
            }
          }
          if (++stage == kStages) {
            stage = 0;
            parity ^= 1u;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
  const int cw = warp - kProducerWarps;
  const int fk = lane & 3, fn = lane >> 2;
  // box row of fragment row index n when the contraction index is the contiguous one
  const int prow = ((fn & 3) << 1) | (fn >> 2);
  int frag_off[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (INNER1) {
      const int l = 8 * (s >> 1) + 2 * fk + (s & 1);
      frag_off[s] = l * 16 + ((((fn >> 1) ^ (l & 7)) << 1) | (fn & 1));
    } else {
      const int l = 4 * s + fk;
      frag_off[s] = prow * 16 + ((((l >> 1) ^ prow) << 1) | (l & 1));
    }
  }

  double acc0[4][4][2], acc1[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc0[a][b][0] = acc0[a][b][1] = acc1[a][b][0] = acc1[a][b][1] = 0.0;

  // accumulators of one block -> the split's partial plane
  auto store_block = [&](double (&acc)[4][4][2], double* out, long long i_blk, long long j_blk) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const long long i = i_blk + 8 * a + (INNER1 ? fn : prow);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 2 * fk + e;
          const long long j = j_blk + 8 * b + (INNER1 ? n : (((n & 3) << 1) | (n >> 2)));
          if (i < p.rows && j < p.rows) out[i * p.rows + j] = acc[a][b][e];
          acc[a][b][e] = 0.0;
        }
      }
    }
  };

  int stage = 0;
  unsigned parity = 0;
  for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
    int ti, tj, split;
    decode_item(p, item, ti, tj, split);
    const bool diag = ti == tj;
    const long long i0 = static_cast<long long>(ti) * kTile, j0 = static_cast<long long>(tj) * kTile;
    int blk0, blk1;
    warp_blocks(diag, cw, blk0, blk1);
    // blocks whose rows lie past the extent are dead (their columns then are too, or the tile is off the diagonal and
    // all its columns are live); a warp's second block lies below its first, so the live ones are a prefix
    if (blk1 >= 0 && i0 + 32 * (blk1 >> 4) >= p.rows) blk1 = -1;
    if (blk0 >= 0 && i0 + 32 * (blk0 >> 4) >= p.rows) blk0 = -1;
    const int n_blk = blk0 < 0 ? 0 : (blk1 < 0 ? 1 : 2);
    const int a_off0 = (blk0 >> 4) * 512, b_off0 = (blk0 & 15) * 512;
    const int a_off1 = (blk1 >> 4) * 512, b_off1 = (blk1 & 15) * 512;
    const long long c_begin = static_cast<long long>(split) * p.chunks_per_split;
    const long long c_end = min(p.chunks, c_begin + p.chunks_per_split);
    for (long long c = c_begin; c < c_end; ++c) {
      mbar_wait(&full[stage], parity);
      const double* const ta = sa + stage * kOperandDoubles;
      const double* const tb = diag ? ta : sb + stage * kOperandDoubles;
      if (n_blk >= 1) consume_block<INNER1>(acc0, ta + a_off0, tb + b_off0, frag_off);
      if (n_blk == 2) consume_block<INNER1>(acc1, ta + a_off1, tb + b_off1, frag_off);
      // generic-proxy reads of the stage before the async-proxy refill (see ttm_tma_kernels.cu)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kStages) {
        stage = 0;
        parity ^= 1u;
      }
    }
    // ---- partial tile of this split
    double* const out = p.partial + static_cast<long long>(split) * p.rows * p.rows;
    if (n_blk >= 1) store_block(acc0, out, i0 + 32 * (blk0 >> 4), j0 + 32 * (blk0 & 15));
    if (n_blk == 2) store_block(acc1, out, i0 + 32 * (blk1 >> 4), j0 + 32 * (blk1 & 15));
  }
}

// cost of a tile in quarter-tile units of DMMA time on the busiest SM sub-partition
int tile_cost(int ti, int tj, long long rows) {
  const long long live = std::min<long long>(kTile, rows - static_cast<long long>(ti) * kTile);
  const int block_rows = static_cast<int>((live + 31) / 32);
  if (ti != tj) return block_rows;  // each sub-partition: one column block x block_rows row blocks
  // diagonal: sub-partition loads of the dealing in warp_blocks, restricted to the live row blocks
  static const int deal[4][3] = {{0x00, 0x10, 0x11}, {0x20, 0x30, 0x21}, {0x22, 0x32, -1}, {0x31, 0x33, -1}};
  int worst = 0;
  for (const auto& part : deal) {
    int load = 0;
    for (int blk : part)
      if (blk >= 0 && (blk >> 4) < block_rows) ++load;
    worst = std::max(worst, load);
  }
  return worst;
}

}  // namespace

bool gram_wide_shape(long long outer, long long rows, long long inner) {
  if (rows < 4 * kTile - 64) return false;                        // at least four tile rows
  if ((inner == 1 ? rows : inner) % 2) return false;              // 16-byte global strides
  if (outer >= (1LL << 31) || rows >= (1LL << 31) || inner >= (1LL << 31)) return false;
  const long long chunks = inner == 1 ? (outer + kKC - 1) / kKC : outer * ((inner + kKC - 1) / kKC);
  return chunks >= 64;
}

GramLayout gram_wide_layout(long long outer, long long rows, long long inner, int sm_count) {
  // the split search below replays the walk for every candidate (tens of microseconds of host time): a plan asks for
  // the same few layouts every sweep, so the last ones are remembered per host thread
  struct Memo {
    long long outer = -1, rows = -1, inner = -1;
    int sm_count = -1;
    GramLayout layout;
  };
  thread_local Memo memo[8];
  thread_local int memo_next = 0;
  for (const Memo& m : memo)
    if (m.outer == outer && m.rows == rows && m.inner == inner && m.sm_count == sm_count) return m.layout;
  GramLayout g;
  g.wide = true;
  g.tiles = static_cast<int>((rows + kTile - 1) / kTile);
  g.chunks = inner == 1 ? (outer + kKC - 1) / kKC : outer * ((inner + kKC - 1) / kKC);
  const int t = g.tiles;
  // tiles in the kernel's item order (decode_item)
  std::vector<int> cost;
  for (int ti = 1; ti < t - 1; ++ti)
    for (int tj = 0; tj < ti; ++tj) cost.push_back(tile_cost(ti, tj, rows));
  for (int ti = 0; ti < t - 1; ++ti) cost.push_back(tile_cost(ti, ti, rows));
  for (int tj = 0; tj < t - 1; ++tj) cost.push_back(tile_cost(t - 1, tj, rows));
  cost.push_back(tile_cost(t - 1, t - 1, rows));
  // split count: replay the round-robin walk for every candidate and keep the one whose busiest CTA finishes first
  // (+ 3 chunks per item for the epilogue and the change of tile, + the ordered sum's cost per split)
  const int grid = std::max(1, sm_count);
  // at most 1 GiB of partial planes (tall Gram matrices have tiles enough to fill the machine without splitting)
  const long long plane_cap = std::max(1LL, (1LL << 27) / std::max(1LL, rows * rows));
  const long long max_splits = std::max(1LL, std::min({32LL, g.chunks / 8, plane_cap}));
  long long best = 1;
  double best_time = -1.0;
  std::vector<double> load(static_cast<size_t>(grid));
  for (long long s = 1; s <= max_splits; ++s) {
    const long long per = (g.chunks + s - 1) / s;
    const long long used = (g.chunks + per - 1) / per;
    if (used != s) continue;
    std::fill(load.begin(), load.end(), 0.0);
    long long item = 0;
    for (long long sp = 0; sp < s; ++sp) {
      const long long n = std::min(per, g.chunks - sp * per);
      for (int c : cost) load[static_cast<size_t>(item++ % grid)] += 0.25 * c * static_cast<double>(n) + 3.0;
    }
    double worst = 0.0;
    for (double l : load) worst = std::max(worst, l);
    worst += 2.0 * static_cast<double>(s);
    if (best_time < 0.0 || worst < best_time) {
      best_time = worst;
      best = s;
    }
  }
  g.splits = static_cast<int>(best);
  g.workspace_doubles = static_cast<size_t>(g.splits) * rows * rows;
  g.sm_count = sm_count;
  Memo& slot = memo[memo_next];
  memo_next = (memo_next + 1) % 8;
  slot.outer = outer;
  slot.rows = rows;
  slot.inner = inner;
  slot.sm_count = sm_count;
  slot.layout = g;
  return g;
}

cudaError_t launch_gram_wide(cudaStream_t stream, const double* y, long long outer, long long rows, long long inner,
                             const GramLayout& g, double* workspace, int sm_count) {
  GramTmaParams p;
  p.partial = workspace;
  p.rows = rows;
  p.chunks = g.chunks;
  p.chunks_per_split = (g.chunks + g.splits - 1) / g.splits;
  p.chunks_per_slab = static_cast<int>(inner == 1 ? 1 : (inner + kKC - 1) / kKC);
  p.splits = g.splits;
  p.tile_rows = g.tiles;
  p.n_items = g.tiles * (g.tiles + 1) / 2 * g.splits;
  // the TTM kernel's maps: (inner, rows, outer) boxes {16, 16, 1}, or (rows, outer, 1) when inner == 1
  const CUtensorMap* map = static_cast<const CUtensorMap*>(ttm_tensor_map(y, outer, rows, inner));
  if (!map) return cudaErrorInvalidValue;
  const bool inner1 = inner == 1;
  static PerDeviceInt configured[2];
  std::atomic<int>* const slot = configured[inner1 ? 1 : 0].slot();
  if (!slot || slot->load(std::memory_order_relaxed) == 0) {
    cudaError_t e = inner1 ? cudaFuncSetAttribute(gram_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(kSmemBytes))
                           : cudaFuncSetAttribute(gram_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    if (slot) slot->store(1, std::memory_order_relaxed);
  }
  const unsigned grid = static_cast<unsigned>(std::max(1, std::min(sm_count, p.n_items)));
  if (inner1)
    gram_tma_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(*map, p);
  else
    gram_tma_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(*map, p);
  return cudaGetLastError();
}

}  // namespace tpb
