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
constexpr int kFusedMaxRowBlocks = kFusedMaxRows / 32;

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

// out (rows x b, leading dimension ld, shared) = G * in (shared), G symmetric (column l doubles as row l).
// A thread owns up to kItems tiles of two rows by eight columns (16 accumulators: per contraction index one 128-bit
// load of the row pair and eight broadcast loads feed 16 FMAs, which keeps the product on the FP64 pipe rather than on
// shared-memory bandwidth); a warp covers 64 consecutive rows of one column group.  Two sources of G:
//   * resident: the whole matrix was copied into shared memory at kernel start (rows <= ~110: every leaf of
//     BASELINE configs 2-4) -- the product is pure arithmetic;
//   * streamed: slabs of `slab` columns through a ring of kRing shared-memory buffers filled by cp.async, kRing - 1
//     slabs in flight while one is multiplied, so every entry of G is read from L2 exactly once per product.
// The caller synchronises afterwards.
constexpr int kRing = 3;
// Tile shapes: 2 x 8 with one tile per thread for the streamed product (large leaves: enough tiles to fill the CTA,
// FP64-pipe bound); 2 x 4 with up to three tiles per thread for the resident one (small leaves: more, shorter
// threads -- at 2 x 8 only a few warps would have work and the product becomes latency bound).
template <int TC>
struct TileShape {
  static constexpr int kItems = TC == 8 ? 1 : 3;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(gmem) : "memory");
}

template <int TC>
struct ProductTiles {
  int i0[TileShape<TC>::kItems], c0[TileShape<TC>::kItems];
  bool on[TileShape<TC>::kItems];
};

template <int TC>
__device__ __forceinline__ ProductTiles<TC> product_tiles(int rows, int b) {
  constexpr int kItems = TileShape<TC>::kItems;
  constexpr int kTileCols = TC;
  const int row_pairs = (rows + 1) / 2;
  const int pair_slots = (row_pairs + 31) & ~31;  // whole warps per column group
  const int n_items = pair_slots * ((b + kTileCols - 1) / kTileCols);
  ProductTiles<TC> t;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int item = threadIdx.x + it * kFusedThreads;
    const int cg = item / pair_slots, rp = item - cg * pair_slots;
    t.on[it] = item < n_items && rp < row_pairs;
    t.i0[it] = t.on[it] ? 2 * rp : 0;
    t.c0[it] = t.on[it] ? kTileCols * cg : 0;
  }
  return t;
}

// acc += G[:, l0 .. l0 + width) (columns held in `cols`, leading dimension rows) * in[l0 .. l0 + width, :]
template <int TC>
__device__ __forceinline__ void product_accumulate(const ProductTiles<TC>& t,
                                                   double (&acc)[TileShape<TC>::kItems][2 * TC],
                                                   const double* __restrict__ cols, const double* __restrict__ in,
                                                   int rows, int b, int ld, int l0, int width) {
  constexpr int kItems = TileShape<TC>::kItems;
  constexpr int kTileCols = TC;
  // 16-byte loads of the row pair need an even leading dimension (and the buffers are 16-byte aligned)
  const bool paired = (rows & 1) == 0;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    if (!t.on[it]) continue;
    const int r0 = t.i0[it], r1 = min(r0 + 1, rows - 1);
    const double* y[kTileCols];
#pragma unroll
    for (int c = 0; c < kTileCols; ++c) y[c] = in + static_cast<size_t>(min(t.c0[it] + c, b - 1)) * ld + l0;
#pragma unroll 2
    for (int l = 0; l < width; ++l) {
      double x0, x1;
      if (paired) {
        const double2 x = *reinterpret_cast<const double2*>(cols + l * rows + r0);
        x0 = x.x;
        x1 = x.y;
      } else {
        x0 = cols[l * rows + r0];
        x1 = cols[l * rows + r1];
      }
#pragma unroll
      for (int c = 0; c < kTileCols; ++c) {
        const double v = y[c][l];
        acc[it][c] = fma(x0, v, acc[it][c]);
        acc[it][kTileCols + c] = fma(x1, v, acc[it][kTileCols + c]);
      }
    }
  }
}

template <int TC>
__device__ void product_gq_tiles(const double* __restrict__ g, const double* __restrict__ in, double* __restrict__ out,
                                 double* __restrict__ gbuf, bool resident, int slab, int rows, int b, int ld) {
  constexpr int kItems = TileShape<TC>::kItems;
  constexpr int kTileCols = TC;
  const ProductTiles<TC> t = product_tiles<TC>(rows, b);
  double acc[kItems][2 * kTileCols];
#pragma unroll
  for (int it = 0; it < kItems; ++it)
#pragma unroll
    for (int e = 0; e < 2 * kTileCols; ++e) acc[it][e] = 0.0;
  if (resident) {
    product_accumulate<TC>(t, acc, gbuf, in, rows, b, ld, 0, rows);
  } else {
    const int slab_elems = rows * slab;
    const int n_slabs = (rows + slab - 1) / slab;
    auto issue = [&](int index) {  // one commit group per slab, empty past the end so that the group count is uniform
      if (index < n_slabs) {
        const int l0 = index * slab;
        const int count = min(slab, rows - l0) * rows;  // whole columns, contiguous in G
        const double* const src = g + static_cast<size_t>(l0) * rows;
        double* const dst = gbuf + (index % kRing) * slab_elems;
        for (int e = threadIdx.x; e < count; e += kFusedThreads) cp_async8(dst + e, src + e);
      }
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
      product_accumulate<TC>(t, acc, gbuf + (index % kRing) * slab_elems, in, rows, b, ld, l0, min(slab, rows - l0));
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    if (!t.on[it]) continue;
#pragma unroll
    for (int c = 0; c < kTileCols; ++c) {
      if (t.c0[it] + c >= b) break;
      out[static_cast<size_t>(t.c0[it] + c) * ld + t.i0[it]] = acc[it][c];
      if (t.i0[it] + 1 < rows) out[static_cast<size_t>(t.c0[it] + c) * ld + t.i0[it] + 1] = acc[it][kTileCols + c];
    }
  }
}

__device__ void product_gq(const double* __restrict__ g, const double* __restrict__ in, double* __restrict__ out,
                           double* __restrict__ gbuf, bool resident, int slab, int rows, int b, int ld) {
  if (resident)
    product_gq_tiles<4>(g, in, out, gbuf, true, slab, rows, b, ld);
  else
    product_gq_tiles<8>(g, in, out, gbuf, false, slab, rows, b, ld);
}

// s (b x b, leading dimension m, shared) = A^T B for A, B rows x b in shared memory; only the tiles on and below
// the diagonal are computed and mirrored (both uses are symmetric: Z^T Z and Q^T (G Q)).  A warp owns a 4 x 4 tile:
// lanes stride the rows, then a fixed butterfly sums the lanes (same order every run).
__device__ void small_gram(const double* __restrict__ a, const double* __restrict__ bm, double* __restrict__ s,
                           int rows, int b, int ld, int m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (b + 3) / 4;
  const int n_lower = tiles * (tiles + 1) / 2;
  for (int t = warp; t < n_lower; t += kFusedWarps) {
    int ti = 0, tj = t;
    while (tj > ti) {
      tj -= ti + 1;
      ++ti;
    }
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
    const double* ap[4];
    const double* bp[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      ap[x] = a + static_cast<size_t>(min(4 * ti + x, b - 1)) * ld;
      bp[x] = bm + static_cast<size_t>(min(4 * tj + x, b - 1)) * ld;
    }
    for (int i = lane; i < rows; i += 32) {
      double av[4], bv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        av[x] = ap[x][i];
        bv[x] = bp[x][i];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        double v = acc[x][y];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[x][y] = v;
      }
    if (lane == 0) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int r = 4 * ti + x, c = 4 * tj + y;  // entry (r, c) with r's tile >= c's tile
          if (r < b && c < b && (ti > tj || r >= c)) {
            s[c * m + r] = acc[x][y];
            s[r * m + c] = acc[x][y];
          }
        }
    }
  }
}

// In-place Cholesky factorisation of the symmetric positive definite b x b matrix s + shift I (leading dimension m,
// shared): on return the lower triangle holds L and invd[j] = 1 / L(j, j).  The trailing update works on the unscaled
// column, S(i,k) -= S(i,j) S(k,j) / d_j, so a step needs one barrier.  Returns false (uniformly) when a pivot is not
// positive.  kCap >= b.
//
// shift > 0 is the first pass of a shifted Cholesky QR: the oversampling columns of Z = G Q lie, up to the ratio
// lambda_noise / lambda_signal, inside the span of the leading ones, so Z^T Z is numerically singular whenever that
// ratio drops below ~1e-8 and an unshifted factorisation breaks down.  With the shift every pivot is positive; the
// columns it touches come out shorter than unit length, the span is unchanged, and the unshifted passes that follow
// (on a block whose condition number is now moderate) restore orthonormality.
template <int kCap>
__device__ bool cholesky_smem(double* __restrict__ s, double* __restrict__ invd, int b, int m, double shift) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double pivot[64];
  __syncthreads();
  if (shift > 0.0) {
    for (int j = threadIdx.x; j < b; j += kFusedThreads) s[j * m + j] += shift;
    __syncthreads();
  }
  for (int j = 0; j < b; ++j) {
    const double d = s[j * m + j];  // final since the previous step's barrier
    if (!(d > 0.0) || !(d <= DBL_MAX)) return false;  // uniform: every thread reads the same value
    if (threadIdx.x == 0) pivot[j] = sqrt(d);
    const double dinv = fast_rcp(d);
    constexpr int kPasses = (kCap + 31) / 32;
    double cj[kPasses];
#pragma unroll
    for (int r = 0; r < kPasses; ++r) {
      const int i = lane + 32 * r;
      cj[r] = (i > j && i < b) ? s[j * m + i] : 0.0;
    }
    for (int k = j + 1 + warp; k < b; k += kFusedWarps) {
      const double skj = s[j * m + k] * dinv;
#pragma unroll
      for (int r = 0; r < kPasses; ++r) {
        const int i = lane + 32 * r;
        if (i >= k && i < b) s[k * m + i] = fma(-cj[r], skj, s[k * m + i]);
      }
    }
    __syncthreads();
  }
  // scale the columns: L(i, j) = S(i, j) / sqrt(d_j)
  for (int col = warp; col < b; col += kFusedWarps) {
    const double piv = pivot[col];
    const double pinv = 1.0 / piv;
    for (int row = lane; row < b; row += 32)
      if (row > col) s[col * m + row] *= pinv;
      else if (row == col) s[col * m + row] = piv;
    if (lane == 0) invd[col] = pinv;
  }
  __syncthreads();
  return true;
}

// z (rows x b, shared) <- z L^{-T}, in place: row i solves x L^T = z_i.  Right-looking: once x_j = z_j / L(j,j) is
// known, the later columns of the row are updated independently (z_c -= x_j L(c,j)), so the dependent chain is one
// multiplication and one update per column instead of a length-j sum; two rows per thread where there are threads to
// spare would not help, the chain is what costs.
template <int kCap>
__device__ void trsm_rows(double* __restrict__ z, const double* __restrict__ l, const double* __restrict__ invd,
                          int rows, int b, int ld, int m) {
  for (int i = threadIdx.x; i < rows; i += kFusedThreads) {
    double* const zi = z + i;
    double next = zi[0];
    for (int j = 0; j < b; ++j) {
      const double xj = next * invd[j];
      zi[static_cast<size_t>(j) * ld] = xj;
      const double* const lj = l + j * m;
      // column j + 1 first and kept in a register: it is the next step's pivot entry
      if (j + 1 < b) next = fma(-xj, lj[j + 1], zi[static_cast<size_t>(j + 1) * ld]);
#pragma unroll 4
      for (int c = j + 2; c < b; ++c) zi[static_cast<size_t>(c) * ld] = fma(-xj, lj[c], zi[static_cast<size_t>(c) * ld]);
    }
  }
  __syncthreads();
}

template <int kCap>
__global__ void __launch_bounds__(kFusedThreads, 1) leaf_solve_fused_kernel(const FusedParams p) {
  extern __shared__ __align__(16) double sm[];
  const int rows = p.rows, b = p.b, k = p.k;
  const int ld = rows | 1;            // odd leading dimension: column-strided accesses spread over the banks
  const int m = (b + 1) & ~1;
  double* q = sm;                     // ld x b
  double* z = q + static_cast<size_t>(ld) * b;
  double* const h = z + static_cast<size_t>(ld) * b;  // m x m
  double* const v = h + m * m;        // m x m
  double* const theta = v + m * m;    // m (ascending)
  double* const invd = theta + m;     // m
  double* const col_res = invd + m;   // m: squared residual norm per sorted column
  double* const part_res = col_res + m;                   // [row blocks][m]
  double* const part_abs = part_res + kFusedMaxRowBlocks * m;  // [row blocks][m]
  int* const part_idx = reinterpret_cast<int*>(part_abs + kFusedMaxRowBlocks * m);  // [row blocks][m]
  int* const order = part_idx + kFusedMaxRowBlocks * m;   // m: sorted position -> Jacobi column
  // G itself (resident) or the slab ring of product_gq, 16-byte aligned behind the int arrays
  double* const gbuf =
      reinterpret_cast<double*>((reinterpret_cast<unsigned long long>(order + m) + 15ull) & ~15ull);
  const bool resident = p.resident != 0;
  __shared__ double scal[8];
  __shared__ double red[kFusedWarps];
  __shared__ int ctl[4];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // phase accounting (thread 0, after the barrier that ends a phase)
  long long phase_cycles[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long jacobi_prof[3] = {0, 0, 0};
  long long phase_mark = clock64();
  auto end_phase = [&](int which) {
    if (tid == 0) {
      const long long now = clock64();
      phase_cycles[which] += now - phase_mark;
      phase_mark = now;
    }
  };

  if (resident) {
    const int count = rows * rows;
    for (int e = tid; e < count; e += kFusedThreads) cp_async8(gbuf + e, p.gram + e);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // ---- start block
  for (int e = tid; e < rows * b; e += kFusedThreads) {
    const int c = e / rows, i = e - c * rows;
    double val;
    if (p.start_mode == 0)
      val = p.start[static_cast<size_t>(b - 1 - c) * rows + i];
    else
      val = c < k ? p.start[static_cast<size_t>(c) * rows + i]
                  : filler_value(static_cast<unsigned long long>(c - k) * rows + i, 0x7461636bull);
    q[static_cast<size_t>(c) * ld + i] = val;
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
  double d_res = 0.0, d_angle = 0.0, d_tau = 0.0;
  bool failed = false;
  for (int round = 0; round < p.max_rounds && !failed; ++round) {
    ++rounds;
    const int steps = round == 0 ? p.first_steps : round + 1;
    for (int s = 0; s < steps && !failed; ++s) {
      product_gq(p.gram, q, z, gbuf, resident, p.slab, rows, b, ld);
      __syncthreads();
      end_phase(1);
      // shifted Cholesky QR: one shifted pass keeps the span and tames the conditioning; the last step of a round
      // adds two plain passes, after which Q is orthonormal to rounding (the Rayleigh-Ritz step needs that)
      const int passes = (s + 1 == steps) ? 3 : 1;
      for (int pass = 0; pass < passes && !failed; ++pass) {
        small_gram(z, z, h, rows, b, ld, m);
        __syncthreads();
        double shift = 0.0;
        if (pass == 0) {
          double tr = 0.0;  // ||Z||_F^2, same fixed-order sum in every thread
          for (int j = 0; j < b; ++j) tr += h[j * m + j];
          shift = 1e-11 * tr;
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
        if (!cholesky_smem<kCap>(h, invd, b, m, shift)) {
          failed = true;
          break;
        }
        end_phase(3);
        trsm_rows<kCap>(z, h, invd, rows, b, ld, m);
        end_phase(4);
      }
      double* const t = q;
      q = z;
      z = t;
      ++steps_total;
    }
    if (failed) break;

    // ---- Rayleigh-Ritz on span(Q)
    product_gq(p.gram, q, z, gbuf, resident, p.slab, rows, b, ld);
    __syncthreads();
    end_phase(1);
    small_gram(q, z, h, rows, b, ld, m);
    for (int e = tid; e < m * m; e += kFusedThreads) {
      const int c = e / m, r = e - c * m;
      v[e] = (r == c) ? 1.0 : 0.0;
      if (r >= b || c >= b) h[e] = 0.0;
    }
    __syncthreads();
    end_phase(2);
    sweeps = jacobi_sweeps_smem<kFusedThreads, kCap>(h, v, b, m, jacobi_prof);
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
        theta[rank] = li;
        order[rank] = i;
      }
    }
    __syncthreads();

    // ---- X = Q V (sorted columns) to global; residual R = (G Q) V - X Theta and the column maxima on the way.
    // A warp owns 32 consecutive rows (one row block) and four sorted columns.
    const int row_blocks = (rows + 31) / 32;
    const int col_groups = (b + 3) / 4;
    for (int item = warp; item < row_blocks * col_groups; item += kFusedWarps) {
      const int cg = item / row_blocks, rb = item - cg * row_blocks;
      const int i = rb * 32 + lane;
      const bool live = i < rows;
      double x[4] = {0.0, 0.0, 0.0, 0.0}, w[4] = {0.0, 0.0, 0.0, 0.0};
      const double* vc[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) vc[c] = v + order[min(4 * cg + c, b - 1)] * m;
      if (live) {
        for (int l = 0; l < b; ++l) {
          const double qv = q[static_cast<size_t>(l) * ld + i], zv = z[static_cast<size_t>(l) * ld + i];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double vv = vc[c][l];
            x[c] = fma(qv, vv, x[c]);
            w[c] = fma(zv, vv, w[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = 4 * cg + c;
        if (col >= b) break;  // uniform in the warp
        if (live) p.ritz[static_cast<size_t>(col) * rows + i] = x[c];
        const double r = live ? w[c] - theta[col] * x[c] : 0.0;
        double r2 = r * r;
        double ax = live ? fabs(x[c]) : -1.0;
        int ai = live ? i : 0x7fffffff;
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
          part_res[rb * m + col] = r2;
          part_abs[rb * m + col] = ax;
          part_idx[rb * m + col] = ai;
        }
      }
    }
    __syncthreads();
    for (int col = tid; col < b; col += kFusedThreads) {
      double r2 = 0.0;
      for (int rb = 0; rb < row_blocks; ++rb) r2 += part_res[rb * m + col];
      col_res[col] = r2;
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
    d_res = scal[0];
    d_angle = scal[1];
    d_tau = scal[2];
    __syncthreads();
    end_phase(7);
    // certified; or the pairs have converged and the gap / tail criterion still fails: more rounds cannot change that
    if (miss == 0 || (miss & 1) == 0) break;
  }

  if (tid == 0) {
    p.verdict[0] = failed ? 0 : miss;
    p.verdict[1] = failed ? 1 : 0;
    p.verdict[2] = sweeps;
    p.verdict[3] = steps_total;
    p.diag[0] = d_res;
    p.diag[1] = d_angle;
    p.diag[2] = d_tau;
    p.diag[3] = rounds;
    for (int i = 0; i < 8; ++i) p.diag[4 + i] = static_cast<double>(phase_cycles[i]);
    for (int i = 0; i < 3; ++i) p.diag[12 + i] = static_cast<double>(jacobi_prof[i]);  // checks / rotations / updates
  }
  if (failed) return;

  // ---- the reference's selection (hooi.hpp:60-74) from the sorted Ritz vectors just written to global memory
  const int row_blocks = (rows + 31) / 32;
  for (int j = warp; j < k; j += kFusedWarps) {
    const int col = b - 1 - j;
    double ax = -1.0;
    int ai = 0x7fffffff;
    for (int rb = 0; rb < row_blocks; ++rb) {  // first index of the largest magnitude
      const double oa = part_abs[rb * m + col];
      const int oi = part_idx[rb * m + col];
      if (oa > ax || (oa == ax && oi < ai)) {
        ax = oa;
        ai = oi;
      }
    }
    const double* const src = p.ritz + static_cast<size_t>(col) * rows;
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
  const size_t ld = static_cast<size_t>(rows | 1), m = static_cast<size_t>((b + 1) & ~1);
  const size_t gdoubles = resident ? static_cast<size_t>(rows) * rows : static_cast<size_t>(kRing) * rows * slab;
  const size_t doubles = 2 * ld * b + 2 * m * m + 3 * m + 2 * kFusedMaxRowBlocks * m + gdoubles;
  const size_t ints = kFusedMaxRowBlocks * m + m;
  return doubles * sizeof(double) + ints * sizeof(int) + 32;  // + alignment of the G buffer
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
  // product_gq: resident G -> up to 3 tiles of 2 x 4 per thread; streamed G -> one tile of 2 x 8 per thread
  const long long pair_slots = (((rows + 1) / 2) + 31) & ~31LL;
  if (fused_resident(static_cast<int>(rows), b))
    return pair_slots * ((b + 3) / 4) <= static_cast<long long>(TileShape<4>::kItems) * kFusedThreads;
  return fused_slab(static_cast<int>(rows), b) > 0 &&
         pair_slots * ((b + 7) / 8) <= static_cast<long long>(TileShape<8>::kItems) * kFusedThreads;
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
