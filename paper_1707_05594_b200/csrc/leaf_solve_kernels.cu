// Certified top-k eigen-solve of a SMALL leaf in ONE launch.
//
// The leaves of BASELINE configs 1-4 have Gram matrices of 48..400 rows and need 5..40 leading eigenvectors.  As a
// sequence of library GEMMs and single-step kernels (engine.cu: subspace_body) such a solve is ~40 dependent launches
// of a few microseconds each, i.e. pure launch latency, and it sits on the critical path of the sweep: the core chain
// waits for the last leaf.  Here the whole warm-started block subspace iteration runs inside one CTA:
//
//     Q (rows x b, b = k + oversampling) lives in shared memory; G (rows x rows) streams from L2 once per product
//     round:  [ Z = G Q;  Q = CholQR(Z) ] x steps   (the last step runs the Cholesky-QR pass twice: orthonormal to
//             rounding)
//             Rayleigh-Ritz: H = Q^T G Q, H = V Theta V^T (parallel cyclic Jacobi), X = Q V
//             certificate (see below); accepted -> done, else another round with more steps from the same Q
//     then the reference's selection rules (hooi.hpp:60-74): k largest, largest-|entry| sign, degenerate-gap flag.
//
// Rounds repeat on the device (no host decision): a warm start from the previous sweep's Ritz vectors passes after
// one power step, a cold start after a few rounds.  Everything is deterministic: every reduction has a fixed order.
//
// Certificate (all three must hold, else verdict[0] != 0 and the caller falls back to the full eigen-solve on the
// intact Gram matrix, so the factors are the reference's (hooi.hpp:55-69) to rounding either way):
//   1. every kept Ritz pair has ||G x - theta x|| <= tol * theta_max                         (eigenpairs to rounding)
//   2. nothing larger was missed: G is positive semidefinite, so every eigenvalue not matched by one of the b Ritz
//      values is at most  tau = trace(G) - sum(theta) + b ||R||_F  (Kahan: b eigenvalues lie within ||R||_2 of the
//      Ritz values of an orthonormal block), and the eigenvalues matched by the oversampling pairs are at most
//      theta_{k+1} + ||R||_F;  delta = theta_k - max(theta_{k+1} + ||R||_F, tau) must be positive
//   3. the subspace angle bound ||R_kept||_F / delta (Davis-Kahan) is at most 1e-10: small gaps go to the full solve.
#include <cuda_runtime.h>

#include <cfloat>

#include "evd_device.cuh"
#include "kernels.cuh"

namespace tpb {
namespace {

constexpr int kFusedThreads = 512;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kFusedMaxRows = 512;

struct FusedParams {
  const double* __restrict__ gram;   // rows x rows, symmetric, full storage
  const double* __restrict__ start;  // start_mode 0: rows x b ascending Ritz vectors of the previous solve (read
                                     // with the column order reversed: dominant direction first);
                                     // start_mode 1: rows x k factor, dominant first; the other columns are filler
  double* __restrict__ ritz;         // out: rows x b Ritz vectors, ascending (may alias `start`)
  double* __restrict__ theta;        // out: b Ritz values, ascending
  double* __restrict__ factor;       // out: rows x k, the reference's selection
  int* __restrict__ flag;            // |= 1: degenerate gap (hooi.hpp:70-74)
  int* __restrict__ verdict;         // [0] = 1 residual bound missed | 4 gap / angle criterion missed, 0 = certified
                                     // [1] != 0: a factorisation failed; [2] Jacobi sweeps of the last round;
                                     // [3] power steps used in total
  double* __restrict__ diag;         // [0] max kept residual / (tol theta_max), [1] angle bound ||R_k||_F / delta,
                                     // [2] tau / theta_k, [3] rounds used; [4..11] SM cycles per phase: start block,
                                     // G Q products, small Gram products, Cholesky, triangular solves, Jacobi,
                                     // Ritz vectors + residuals, certificate (16 doubles in all)
  int rows, k, b;
  int start_mode;
  int resident;                      // G fits in shared memory beside everything else: copy it once, stream nothing
  int slab;                          // streamed G: columns per ring buffer (16, 8 or 4: the widest that fits)
  int first_steps;                   // power steps of the first round (1 for a warm start)
  int max_rounds;
  double tol;                        // residual tolerance relative to theta_max (1e-13)
  double angle_tol;                  // bound on ||R_k||_F / delta (1e-10)
};

__device__ __forceinline__ double filler_value(unsigned long long index, unsigned long long salt) {
  unsigned long long z = (index + 1) * 0x9E3779B97F4A7C15ull + salt;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gmem) : "memory");
}
// Every product of the solve runs on the FP64 tensor pipe (DMMA.8x8x4), fragments straight from shared memory:
//   lane (g = lane / 4, t = lane % 4) holds A(row g, k t), B(k t, column g), C(row g, columns 2t and 2t + 1).
// Leading dimensions are chosen so that a fragment load is conflict free: the rows x b blocks (Q, Z) have
// ld = 4 (mod 8), ld >= rows -- eight columns a multiple of 32 bytes apart and four consecutive rows each -- and the
// columns of G sit lda = 8 (mod 16) apart -- four columns, eight consecutive rows each.  Rows [rows, ld) of Q and Z are
// kept zero, so contractions over the rows may run to the next multiple of four unguarded.
constexpr int kRing = 3;  // streamed G: slabs of columns through a ring of shared-memory buffers
constexpr int kGramSlack = 8;  // doubles behind the G buffer: the last m-tile may read up to 7 rows past a column

__host__ __device__ inline int block_ld(int rows) { return rows + ((4 - rows % 8) + 8) % 8; }
__host__ __device__ inline int gram_ld(int rows) { return rows + ((8 - rows % 16) + 16) % 16; }

// acc += A[:, 0 .. width) * B[l0 .. l0 + width, :]  for the first MTA of the m-tiles warp, warp + 16, ... and the first
// NTA n-tiles (both compile-time: the loop below is straight-line code, no guard around a DMMA).
// A: column kk at a_cols + kk * lda; B: columns ldb apart, entry (l, c) at bm[c * ldb + l].
// Rows of A beyond `rows` and columns of B beyond the block are read as whatever shared memory holds there (inside
// the allocation): a row of the product depends on its own row of A only and a column on its own column of B, and
// dmma_store drops exactly those rows and columns.  Only the ragged end of the contraction is guarded.
template <int MT, int NT, int MTA, int NTA>
__device__ __forceinline__ void dmma_accumulate_fixed(double (&acc)[MT][NT][2], const double* __restrict__ a_cols,
                                                      int lda, int width, const double* __restrict__ bm, int ldb,
                                                      int l0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const double* bp = bm + g * ldb + l0 + t;
  const double* ap = a_cols + t * lda + 8 * warp + g;
  const int tile_stride = 8 * ldb;
  const int a_step = 4 * lda;
  const int whole = width & ~3;
#pragma unroll 2
  for (int kk = 0; kk < whole; kk += 4) {
    double bf[NTA], af[MTA];
#pragma unroll
    for (int j = 0; j < NTA; ++j) bf[j] = bp[j * tile_stride];
#pragma unroll
    for (int i = 0; i < MTA; ++i) af[i] = ap[8 * kFusedWarps * i];
#pragma unroll
    for (int i = 0; i < MTA; ++i)
#pragma unroll
      for (int j = 0; j < NTA; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    bp += 4;
    ap += a_step;
  }
  if (whole < width) {  // uniform
    const bool kin = whole + t < width;
    double bf[NTA], af[MTA];
#pragma unroll
    for (int j = 0; j < NTA; ++j) bf[j] = kin ? bp[j * tile_stride] : 0.0;
#pragma unroll
    for (int i = 0; i < MTA; ++i) af[i] = kin ? ap[8 * kFusedWarps * i] : 0.0;
#pragma unroll
    for (int i = 0; i < MTA; ++i)
#pragma unroll
      for (int j = 0; j < NTA; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

template <int MT, int NT, int NTA>
__device__ __forceinline__ void dmma_accumulate_rows(double (&acc)[MT][NT][2], const double* __restrict__ a_cols,
                                                     int lda, int width, const double* __restrict__ bm, int ldb,
                                                     int l0, int mt_mine) {
  if constexpr (MT * NTA <= 16) {
    switch (mt_mine) {  // uniform in the warp
      case 1: dmma_accumulate_fixed<MT, NT, 1, NTA>(acc, a_cols, lda, width, bm, ldb, l0); break;
      case 2: if constexpr (MT >= 2) dmma_accumulate_fixed<MT, NT, 2, NTA>(acc, a_cols, lda, width, bm, ldb, l0); break;
      case 3: if constexpr (MT >= 3) dmma_accumulate_fixed<MT, NT, 3, NTA>(acc, a_cols, lda, width, bm, ldb, l0); break;
      case 4: if constexpr (MT >= 4) dmma_accumulate_fixed<MT, NT, 4, NTA>(acc, a_cols, lda, width, bm, ldb, l0); break;
      default: break;
    }
  }
}

// mt_mine: m-tiles of this warp that hold rows of the matrix; n: columns of B
template <int MT, int NT>
__device__ __forceinline__ void dmma_accumulate(double (&acc)[MT][NT][2], const double* __restrict__ a_cols, int lda,
                                                int width, const double* __restrict__ bm, int ldb, int n, int l0,
                                                int mt_mine) {
  switch ((n + 7) / 8) {  // uniform in the CTA
    case 1: dmma_accumulate_rows<MT, NT, 1>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 2: if constexpr (NT >= 2) dmma_accumulate_rows<MT, NT, 2>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 3: if constexpr (NT >= 3) dmma_accumulate_rows<MT, NT, 3>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 4: if constexpr (NT >= 4) dmma_accumulate_rows<MT, NT, 4>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 5: if constexpr (NT >= 5) dmma_accumulate_rows<MT, NT, 5>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 6: if constexpr (NT >= 6) dmma_accumulate_rows<MT, NT, 6>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 7: if constexpr (NT >= 7) dmma_accumulate_rows<MT, NT, 7>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    case 8: if constexpr (NT >= 8) dmma_accumulate_rows<MT, NT, 8>(acc, a_cols, lda, width, bm, ldb, l0, mt_mine); break;
    default: break;
  }
}

__device__ __forceinline__ int warp_m_tiles(int rows) {  // m-tiles warp, warp + 16, ... below ceil(rows / 8)
  const int warp = threadIdx.x >> 5;
  const int tiles = (rows + 7) / 8;
  return tiles > warp ? (tiles - warp + kFusedWarps - 1) / kFusedWarps : 0;
}

// out(r, c) = acc for r < rows, 0 for rows <= r < ld (the padding stays zero), c < n
template <int MT, int NT>
__device__ __forceinline__ void dmma_store(const double (&acc)[MT][NT][2], double* __restrict__ out, int rows, int ld,
                                           int n, int mt_mine) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int r = 8 * (warp + kFusedWarps * i) + g;
    if (i >= mt_mine || r >= ld) continue;
    const bool real = r < rows;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = 8 * j + 2 * t;
      if (c < n) out[c * ld + r] = real ? acc[i][j][0] : 0.0;
      if (c + 1 < n) out[(c + 1) * ld + r] = real ? acc[i][j][1] : 0.0;
    }
  }
}

// `count` whole columns of G (from global column first) into shared memory, lda apart; 16-byte copies where the
// addresses allow
__device__ __forceinline__ void copy_gram_columns(const double* __restrict__ g, double* __restrict__ dst, int rows,
                                                  int lda, int first, int count, bool wide) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int col = warp; col < count; col += kFusedWarps) {
    const double* const src = g + static_cast<size_t>(first + col) * rows;
    double* const to = dst + col * lda;
    if (wide)
      for (int ch = lane; 2 * ch < rows; ch += 32) cp_async16(to + 2 * ch, src + 2 * ch);
    else
      for (int i = lane; i < rows; i += 32) cp_async8(to + i, src + i);
  }
}

// out (rows x b, shared) = G * in (shared), G symmetric.  Two sources of G:
//   * resident: the whole matrix was copied into shared memory at kernel start (rows <= ~110: every leaf of
//     BASELINE configs 2-4) -- the product is pure arithmetic;
//   * streamed: slabs of `slab` columns through a ring of kRing shared-memory buffers filled by cp.async, kRing - 1
//     slabs in flight while one is multiplied, so every entry of G is read from L2 exactly once per product.
// The caller synchronises afterwards.
template <int MT, int NT>
__device__ __noinline__ void product_gq(const double* __restrict__ g, const double* __restrict__ in, double* __restrict__ out,
                           double* __restrict__ gbuf, bool resident, bool wide, int slab, int rows, int b, int ld,
                           int lda) {
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int mt_mine = warp_m_tiles(rows);
  if (resident) {
    dmma_accumulate<MT, NT>(acc, gbuf, lda, rows, in, ld, b, 0, mt_mine);
  } else {
    const int slab_elems = lda * slab;
    const int n_slabs = (rows + slab - 1) / slab;
    auto issue = [&](int index) {  // one commit group per slab, empty past the end so that the group count is uniform
      if (index < n_slabs)
        copy_gram_columns(g, gbuf + (index % kRing) * slab_elems, rows, lda, index * slab,
                          min(slab, rows - index * slab), wide);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    __syncthreads();  // the previous users of the ring are done
#pragma unroll
    for (int s0 = 0; s0 < kRing - 1; ++s0) issue(s0);
    for (int index = 0; index < n_slabs; ++index) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kRing - 2) : "memory");
      __syncthreads();  // slab has landed for everyone; everyone is done with the buffer the next issue refills
      issue(index + kRing - 1);
      const int l0 = index * slab;
      dmma_accumulate<MT, NT>(acc, gbuf + (index % kRing) * slab_elems, lda, min(slab, rows - l0), in, ld, b, l0,
                              mt_mine);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  dmma_store<MT, NT>(acc, out, rows, ld, b, mt_mine);
}

// x (rows x b, shared, leading dimension ld) <- x * vs (b x b, leading dimension m), in place: a warp reads only the
// rows it writes, and all of them before it writes any.
template <int MT, int NT>
__device__ __noinline__ void rotate_block(double* __restrict__ x, const double* __restrict__ vs, int rows, int b, int ld, int m) {
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int mt_mine = warp_m_tiles(rows);
  dmma_accumulate<MT, NT>(acc, x, ld, b, vs, m, b, 0, mt_mine);
  __syncwarp();
  dmma_store<MT, NT>(acc, x, rows, ld, b, mt_mine);
}

// s (b x b, leading dimension m, shared) = A^T B for A, B rows x b in shared memory (rows beyond `rows` zero); only
// the 8 x 8 tiles on and below the diagonal are computed and mirrored (both uses are symmetric: Z^T Z and Q^T (G Q)).
// A warp owns a tile; two accumulator pairs alternate along the contraction to halve the dependent chain, and the
// order of the sums is fixed.
__device__ __noinline__ void small_gram(const double* __restrict__ a, const double* __restrict__ bm, double* __restrict__ s,
                           int rows, int b, int ld, int m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int tiles = (b + 7) / 8;
  const int n_lower = tiles * (tiles + 1) / 2;
  const int rows4 = (rows + 3) & ~3;
  for (int tile = warp; tile < n_lower; tile += kFusedWarps) {
    int ti = 0, tj = tile;
    while (tj > ti) {
      tj -= ti + 1;
      ++ti;
    }
    const double* const ap = a + static_cast<size_t>(min(8 * ti + g, b - 1)) * ld + t;
    const double* const bp = bm + static_cast<size_t>(min(8 * tj + g, b - 1)) * ld + t;
    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
    int r = 0;
    for (; r + 8 <= rows4; r += 8) {
      dmma884(c0, c1, ap[r], bp[r]);
      dmma884(d0, d1, ap[r + 4], bp[r + 4]);
    }
    if (r < rows4) dmma884(c0, c1, ap[r], bp[r]);
    c0 += d0;
    c1 += d1;
    const int row = 8 * ti + g, col = 8 * tj + 2 * t;  // entry (row, col) with row's tile >= col's tile
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = col + e;
      const double val = e == 0 ? c0 : c1;
      if (row < b && c < b && (ti > tj || row >= c)) {
        s[c * m + row] = val;
        s[row * m + c] = val;
      }
    }
  }
}

// m-tiles per warp and n-tiles of the DMMA products: 32 accumulators per thread either way
template <int kCap>
struct ProductShape {
  static constexpr int kMT = kCap <= 32 ? 4 : 2;  // rows <= 128 kMT
  static constexpr int kNT = kCap / 8;
};

template <int kCap>
__global__ void __launch_bounds__(kFusedThreads, 1) leaf_solve_fused_kernel(const FusedParams p) {
  constexpr int MT = ProductShape<kCap>::kMT, NT = ProductShape<kCap>::kNT;
  extern __shared__ __align__(16) double sm[];
  const int rows = p.rows, b = p.b, k = p.k;
  const int ld = block_ld(rows);
  const int lda = gram_ld(rows);
  const int m = (b + 1) & ~1;
  double* q = sm;                     // ld x b
  double* z = q + static_cast<size_t>(ld) * b;
  double* const h = z + static_cast<size_t>(ld) * b;  // m x m
  double* const h2 = h + m * m;       // m x m: the Jacobi iteration's second buffer
  double* const v = h2 + m * m;       // m x m
  double* const v2 = v + m * m;       // m x m: the second buffer of the eigenvectors
  double* const theta = v2 + m * m;   // m (ascending)
  double* const invd = theta + m;     // m
  double* const col_res = invd + m;   // m: squared residual norm per sorted column
  // G itself (resident) or the slab ring of product_gq; every count so far is even, so this is 16-byte aligned
  double* const gbuf = col_res + m;
  const bool resident = p.resident != 0;
  const int gram_doubles = resident ? lda * rows : kRing * lda * p.slab;
  int* const order = reinterpret_cast<int*>(gbuf + gram_doubles + kGramSlack);  // m: sorted position -> Jacobi column
  int* const col_idx = order + m;     // m: first row of the largest magnitude per sorted column
  const bool wide = (rows & 1) == 0 && (reinterpret_cast<unsigned long long>(p.gram) & 15ull) == 0;
  __shared__ double scal[8];
  __shared__ double red[kFusedWarps];
  __shared__ int ctl[4];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // phase accounting (thread 0, after the barrier that ends a phase; in shared memory: the registers are the
  // products' accumulators)
  __shared__ long long phase_cycles[8], jacobi_prof[4], phase_mark;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) phase_cycles[i] = 0;
    for (int i = 0; i < 4; ++i) jacobi_prof[i] = 0;
    phase_mark = clock64();
  }
  auto end_phase = [&](int which) {
    if (tid == 0) {
      const long long now = clock64();
      phase_cycles[which] += now - phase_mark;
      phase_mark = now;
    }
  };

  if (resident) {
    copy_gram_columns(p.gram, gbuf, rows, lda, 0, rows, wide);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // ---- start block (rows [rows, ld) of both blocks zero, once: nothing below writes anything else there)
  for (int e = tid; e < ld * b; e += kFusedThreads) {
    const int c = e / ld, i = e - c * ld;
    double val = 0.0;
    if (i < rows) {
      if (p.start_mode == 0)
        val = p.start[static_cast<size_t>(b - 1 - c) * rows + i];
      else
        val = c < k ? p.start[static_cast<size_t>(c) * rows + i]
                    : filler_value(static_cast<unsigned long long>(c - k) * rows + i, 0x7461636bull);
    }
    q[e] = val;
    z[e] = 0.0;
  }
  // trace(G): fixed-order tree, once (the certificate of every round uses it)
  {
    double part = 0.0;
    for (int i = tid; i < rows; i += kFusedThreads) part += p.gram[static_cast<size_t>(i) * rows + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = part;
  }
  if (tid == 0) {
    ctl[0] = 0;  // factorisation failure
    ctl[1] = 0;  // certified
  }
  if (resident) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    double trace = 0.0;
    for (int w = 0; w < kFusedWarps; ++w) trace += red[w];
    scal[4] = trace;
  }
  __syncthreads();
  end_phase(0);

  int steps_total = 0, rounds = 0, sweeps = 0, miss = 1 | 4;
  bool failed = false;
  if (tid == 0) scal[0] = scal[1] = scal[2] = 0.0;
  for (int round = 0; round < p.max_rounds && !failed; ++round) {
    ++rounds;
    const int steps = round == 0 ? p.first_steps : round + 1;
    for (int s = 0; s < steps && !failed; ++s) {
      product_gq<MT, NT>(p.gram, q, z, gbuf, resident, wide, p.slab, rows, b, ld, lda);
      __syncthreads();
      end_phase(1);
      // Cholesky QR of Z.  Its loss of orthogonality is governed by the condition number of Z^T Z with the column
      // norms scaled out (the Gram product, the factorisation and the triangular solve are all invariant under a
      // column scaling up to rounding).  A warm start makes the columns of Z nearly orthogonal -- they are close to
      // eigenvectors times eigenvalues -- so when every scaled off-diagonal entry is below 1 / (2 (b - 1)) that
      // condition number is below 3 (Gershgorin) and ONE plain pass leaves Q orthonormal to rounding.  Otherwise:
      // a shifted pass, which keeps the span and tames the conditioning, and on the last step of a round two plain
      // passes after it (the Rayleigh-Ritz step needs an orthonormal block).
      int passes = (s + 1 == steps) ? 3 : 1;
      bool plain = false;
      for (int pass = 0; pass < passes && !failed; ++pass) {
        small_gram(z, z, h, rows, b, ld, m);
        __syncthreads();
        double shift = 0.0;
        if (pass == 0) {
          const double bound = 0.25 / (static_cast<double>(b - 1) * (b - 1));
          int fine = 1;
          for (int e = tid; e < b * b; e += kFusedThreads) {
            const int c = e / b, r = e - c * b;
            const double x = h[c * m + r], dd = h[c * m + c] * h[r * m + r];
            if (r != c && !(x * x <= bound * dd)) fine = 0;
            if (r == c && !(x > 0.0 && x <= DBL_MAX)) fine = 0;
          }
          plain = __syncthreads_and(fine) != 0;
          if (plain) {
            passes = 1;
          } else {
            double tr = 0.0;  // ||Z||_F^2, same fixed-order sum in every thread
            for (int j = 0; j < b; ++j) tr += h[j * m + j];
            shift = 1e-11 * tr;
          }
        } else if (pass == 2) {
          // Z^T Z of the block the second pass produced: if it is the identity to rounding already (the usual case:
          // the shift of the first pass was below every pivot), the third pass has nothing left to do
          double dev = 0.0;
          for (int e = tid; e < b * b; e += kFusedThreads) {
            const int c = e / b, r = e - c * b;
            dev = fmax(dev, fabs(h[c * m + r] - (r == c ? 1.0 : 0.0)));
          }
          const int settled = __syncthreads_and(dev <= 1e-14 ? 1 : 0);
          if (settled) {
            end_phase(2);
            break;
          }
        }
        end_phase(2);
        if (!cholesky_warp<kCap>(h, invd, b, m, shift)) {
          failed = true;
          break;
        }
        end_phase(3);
        trsm_rows_blocked(z, h, invd, rows, b, ld, m);
        end_phase(4);
      }
      double* const t = q;
      q = z;
      z = t;
      ++steps_total;
    }
    if (failed) break;

    // ---- Rayleigh-Ritz on span(Q)
    product_gq<MT, NT>(p.gram, q, z, gbuf, resident, wide, p.slab, rows, b, ld, lda);
    __syncthreads();
    end_phase(1);
    small_gram(q, z, h, rows, b, ld, m);
    __syncthreads();
    // scale H by a power of two so that its largest entry (on the diagonal: H is positive semidefinite) is of order
    // one -- exact, and the Jacobi rotations then need no scaling of their own
    double top_diag = 0.0;
    for (int j = 0; j < b; ++j) top_diag = fmax(top_diag, fabs(h[j * m + j]));  // same in every thread
    double scale = 1.0, unscale = 1.0;
    {
      const int e = (__double2hiint(top_diag) >> 20) & 0x7ff;
      if (e >= 64 && e <= 1982) {
        scale = __hiloint2double((2046 - e) << 20, 0);
        unscale = __hiloint2double(e << 20, 0);
      }
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += kFusedThreads) {
      const int c = e / m, r = e - c * m;
      v[e] = (r == c) ? 1.0 : 0.0;
      h[e] = (r >= b || c >= b) ? 0.0 : h[e] * scale;
    }
    __syncthreads();
    end_phase(2);
    sweeps = jacobi_pingpong_smem<kFusedThreads, kCap, 16>(h, h2, v, v2, b, m, jacobi_prof);
    end_phase(5);
    if (sweeps == kJacobiMaxSweeps) {
      failed = true;
      break;
    }
    // ascending order by rank (ties by index)
    for (int i = warp; i < b; i += kFusedWarps) {
      const double li = h[i * m + i];
      int rank = 0;
      for (int j = lane; j < b; j += 32) {
        const double lj = h[j * m + j];
        rank += (lj < li) || (lj == li && j < i);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (lane == 0) {
        theta[rank] = li * unscale;
        order[rank] = i;
      }
    }
    __syncthreads();

    // ---- X = Q V and W = (G Q) V (sorted columns), in place; then per column the Ritz vector to global memory, the
    // residual norm of R = W - X Theta and the first row of the largest magnitude
    // (columns of V gathered in DESCENDING order of the Ritz values: the dominant direction first, as the start
    // block of another round wants it)
    for (int e = tid; e < b * m; e += kFusedThreads) {
      const int c = e / m, l = e - c * m;
      h2[e] = v[order[b - 1 - c] * m + l];
    }
    __syncthreads();
    rotate_block<MT, NT>(q, h2, rows, b, ld, m);
    rotate_block<MT, NT>(z, h2, rows, b, ld, m);
    __syncthreads();
    for (int col = warp; col < b; col += kFusedWarps) {  // col: ascending position; stored at b - 1 - col
      const double th = theta[col];
      const double* const xc = q + static_cast<size_t>(b - 1 - col) * ld;
      const double* const wc = z + static_cast<size_t>(b - 1 - col) * ld;
      double r2 = 0.0, ax = -1.0;
      int ai = 0x7fffffff;
      for (int i = lane; i < rows; i += 32) {
        const double x = xc[i];
        p.ritz[static_cast<size_t>(col) * rows + i] = x;
        const double r = wc[i] - th * x;
        r2 = fma(r, r, r2);
        if (fabs(x) > ax) {
          ax = fabs(x);
          ai = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        const double oa = __shfl_xor_sync(0xffffffffu, ax, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ai, o);
        if (oa > ax || (oa == ax && oi < ai)) {
          ax = oa;
          ai = oi;
        }
      }
      if (lane == 0) {
        col_res[col] = r2;
        col_idx[col] = ai;
      }
    }
    __syncthreads();
    end_phase(6);

    // ---- certificate (one thread; tiny)
    if (tid == 0) {
      const double top = fmax(fabs(theta[b - 1]), 1e-300);
      const double trace = scal[4];
      double sum_theta = 0.0, r_all2 = 0.0, r_kept2 = 0.0, worst = 0.0;
      for (int c = 0; c < b; ++c) {
        sum_theta += theta[c];
        r_all2 += col_res[c];
        if (c >= b - k) {
          r_kept2 += col_res[c];
          worst = fmax(worst, sqrt(col_res[c]));
        }
      }
      const double r_all = sqrt(r_all2), r_kept = sqrt(r_kept2);
      const double tau = fmax(trace - sum_theta, 0.0) + b * r_all;
      const double theta_k = theta[b - k];
      const double below = fmax(theta[b - k - 1] + r_all, tau);
      const double delta = theta_k - below;
      int bits = 0;
      if (!(worst <= p.tol * top)) bits |= 1;
      if (!(delta > 0.0) || !(r_kept <= p.angle_tol * delta)) bits |= 4;
      scal[0] = worst / (p.tol * top);
      scal[1] = delta > 0.0 ? r_kept / delta : DBL_MAX;
      scal[2] = tau / fmax(theta_k, 1e-300);
      ctl[1] = bits;
    }
    __syncthreads();
    miss = ctl[1];
    __syncthreads();
    end_phase(7);
    // certified; or the pairs have converged and the gap / tail criterion still fails: more rounds cannot change that
    if (miss == 0 || (miss & 1) == 0) break;
    // another round continues from the Ritz vectors (orthonormal, dominant first; the span is Q's)
  }

  if (tid == 0) {
    p.verdict[0] = failed ? 0 : miss;
    p.verdict[1] = failed ? 1 : 0;
    p.verdict[2] = sweeps;
    p.verdict[3] = steps_total;
    p.diag[0] = scal[0];
    p.diag[1] = scal[1];
    p.diag[2] = scal[2];
    p.diag[3] = rounds;
    for (int i = 0; i < 8; ++i) p.diag[4 + i] = static_cast<double>(phase_cycles[i]);
    for (int i = 0; i < 4; ++i) p.diag[12 + i] = static_cast<double>(jacobi_prof[i]);  // checks / rotations / updates / barriers
  }
  if (failed) return;

  // ---- the reference's selection (hooi.hpp:60-74) from the sorted Ritz vectors (still in shared memory)
  for (int j = warp; j < k; j += kFusedWarps) {
    const double* const src = q + static_cast<size_t>(j) * ld;  // dominant first
    const int ai = col_idx[b - 1 - j];
    const double sign = (ai < rows && src[ai] < 0.0) ? -1.0 : 1.0;
    double* const dst = p.factor + static_cast<size_t>(j) * rows;
    for (int i = lane; i < rows; i += 32) dst[i] = sign * src[i];
  }
  if (tid == 0 && k < b) {
    const double top = fmax(theta[b - 1], 0.0);
    const double gap = theta[b - k] - theta[b - 1 - k];
    if (gap <= 1e-10 * fmax(top, 1e-300)) atomicOr(p.flag, 1);
  }
  for (int c = tid; c < b; c += kFusedThreads) p.theta[c] = theta[c];
}

constexpr size_t kFusedSmemBudget = 200 * 1024;

size_t fused_smem_bytes(int rows, int b, bool resident, int slab) {
  const size_t ld = static_cast<size_t>(block_ld(rows)), lda = static_cast<size_t>(gram_ld(rows));
  const size_t m = static_cast<size_t>((b + 1) & ~1);
  const size_t gdoubles = resident ? lda * rows : static_cast<size_t>(kRing) * lda * slab;
  const size_t doubles = 2 * ld * b + 4 * m * m + 3 * m + gdoubles + kGramSlack;
  const size_t ints = 2 * m;
  // + room for the fragment reads past the last column of a block (rotate_block: up to 7 columns of V)
  return doubles * sizeof(double) + ints * sizeof(int) + 8 * m * sizeof(double);
}

bool fused_resident(int rows, int b) { return fused_smem_bytes(rows, b, true, 0) <= kFusedSmemBudget; }

// widest slab of the streamed product that fits, 0 if none does
int fused_slab(int rows, int b) {
  for (int slab = 16; slab >= 4; slab /= 2)
    if (fused_smem_bytes(rows, b, false, slab) <= kFusedSmemBudget) return slab;
  return 0;
}

}  // namespace

bool leaf_solve_fused_eligible(long long rows, int k, int b) {
  if (rows < 2 || rows > kFusedMaxRows || b > 64 || b <= k || k < 1 || b > rows) return false;
  // the DMMA products keep 128 kMT rows in the accumulators of the CTA
  const int max_rows = 128 * (b <= 32 ? ProductShape<32>::kMT : ProductShape<64>::kMT);
  if (rows > max_rows) return false;
  return fused_resident(static_cast<int>(rows), b) || fused_slab(static_cast<int>(rows), b) > 0;
}

cudaError_t launch_leaf_solve_fused(cudaStream_t stream, const double* gram, int rows, int k, int b,
                                    const double* start, int start_mode, int first_steps, int max_rounds, double tol,
                                    double angle_tol, double* ritz, double* theta, double* factor, int* flag,
                                    int* verdict, double* diag) {
  if (!leaf_solve_fused_eligible(rows, k, b)) return cudaErrorInvalidValue;
  FusedParams p;
  p.gram = gram;
  p.start = start;
  p.ritz = ritz;
  p.theta = theta;
  p.factor = factor;
  p.flag = flag;
  p.verdict = verdict;
  p.diag = diag;
  p.rows = rows;
  p.k = k;
  p.b = b;
  p.start_mode = start_mode;
  p.resident = fused_resident(rows, b) ? 1 : 0;
  p.slab = p.resident ? 0 : fused_slab(rows, b);
  p.first_steps = first_steps < 1 ? 1 : first_steps;
  p.max_rounds = max_rounds < 1 ? 1 : max_rounds;
  p.tol = tol;
  p.angle_tol = angle_tol;
  const size_t smem = fused_smem_bytes(rows, b, p.resident != 0, p.slab);
  static PerDeviceInt configured[2];
  auto allow = [&](auto kernel, PerDeviceInt& done) -> cudaError_t {
    std::atomic<int>* const slot = done.slot();
    if (slot && slot->load(std::memory_order_relaxed)) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kFusedSmemBudget));
    if (e == cudaSuccess && slot) slot->store(1, std::memory_order_relaxed);
    return e;
  };
  cudaError_t e;
  if (b <= 32) {
    e = allow(leaf_solve_fused_kernel<32>, configured[0]);
    if (e != cudaSuccess) return e;
    leaf_solve_fused_kernel<32><<<1, kFusedThreads, smem, stream>>>(p);
  } else {
    e = allow(leaf_solve_fused_kernel<64>, configured[1]);
    if (e != cudaSuccess) return e;
    leaf_solve_fused_kernel<64><<<1, kFusedThreads, smem, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace tpb
