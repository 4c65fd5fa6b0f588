// Device-side pieces of the small dense eigen-solve shared by evd_kernels.cu (one launch per step, any leaf size) and
// leaf_solve_kernels.cu (the whole top-k solve of a small leaf in one launch).
#pragma once

#include <cuda_runtime.h>

#include <cfloat>

namespace tpb {

// 1 / d for a positive, finite d, within an ulp or two: mantissa scaled to [1, 2), single-precision seed, two
// Newton steps in double -- a third of the latency of the IEEE division on the critical path of tiny factorisations.
__device__ __forceinline__ double fast_rcp(double d) {
  const int hi = __double2hiint(d), lo = __double2loint(d);
  const int e = (hi >> 20) & 0x7ff;
  if (e < 2 || e > 2044) return 1.0 / d;  // denormal / near overflow: the slow, exact route
  const double mant = __hiloint2double((hi & 0x000fffff) | (1023 << 20), lo);
  double y = static_cast<double>(__frcp_rn(static_cast<float>(mant)));
  y = fma(y, fma(-mant, y, 1.0), y);
  y = fma(y, fma(-mant, y, 1.0), y);
  return y * __hiloint2double((2046 - e) << 20, 0);
}

// 1 / sqrt(x) for x in [1, 2] (1 + tan^2 of a Jacobi angle), within an ulp or two.
__device__ __forceinline__ double fast_rsqrt_1_2(double x) {
  double y = static_cast<double>(rsqrtf(static_cast<float>(x)));
  const double h = 0.5 * x;
  y = fma(y, fma(-h * y, y, 0.5), y);
  y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}


constexpr int kEvdMaxBlock = 112;     // largest block the single-CTA kernels take (2 b^2 doubles of shared memory)
constexpr int kJacobiMaxSweeps = 30;

// Parallel cyclic Jacobi on the symmetric matrix h (m x m in shared memory, m even, entries beyond b zero) with the
// rotations accumulated into v (m x m, identity on entry).  Round-robin pairing gives m/2 disjoint rotations per
// step; the step's update H <- J^T H J touches every 2 x 2 block (row pair, column pair) exactly once, so it needs
// no barrier between the column and the row half.  All kThreads threads of the CTA must call it together; on return
// (after a barrier) the eigenvalues sit on the diagonal of h, the eigenvectors in the columns of v, unsorted.
// Returns the number of sweeps used; kJacobiMaxSweeps means the off-diagonal mass never fell below (b eps ||H||_F)^2
// (or the input held NaN / Inf).  kBlockCap >= b sizes the per-lane register passes.
// prof (optional, thread 0 writes): SM cycles spent in [0] the convergence checks, [1] forming the rotations (up to the
// barrier that publishes them), [2] applying them (up to the barrier that ends the step).
template <int kThreads, int kBlockCap>
__device__ int jacobi_sweeps_smem(double* __restrict__ h, double* __restrict__ v, int b, int m,
                                  long long* prof = nullptr) {
  const int half = m / 2;
  __shared__ double rot_c[kEvdMaxBlock / 2], rot_s[kEvdMaxBlock / 2];
  __shared__ int rot_p[kEvdMaxBlock / 2], rot_q[kEvdMaxBlock / 2];
  constexpr int kWarps = kThreads / 32;
  __shared__ double red[2 * kWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  long long mark = prof ? clock64() : 0;
  auto lap = [&](int which) {
    if (prof && tid == 0) {
      const long long now = clock64();
      prof[which] += now - mark;
      mark = now;
    }
  };
  int sweep = 0;
  for (; sweep < kJacobiMaxSweeps; ++sweep) {
    // off-diagonal mass against the whole: the backward error of a dense symmetric solver is (b eps ||H||_F)
    double off = 0.0, all = 0.0;
    for (int col = warp; col < m; col += kWarps)
      for (int row = lane; row < m; row += 32) {
        const double x = h[col * m + row] * h[col * m + row];
        all += x;
        if (row != col) off += x;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) {
      red[warp] = off;
      red[kWarps + warp] = all;
    }
    __syncthreads();
    off = 0.0;
    all = 0.0;
    for (int i = 0; i < kWarps; ++i) {
      off += red[i];
      all += red[kWarps + i];
    }
    __syncthreads();
    lap(0);
    if (off <= (b * DBL_EPSILON) * (b * DBL_EPSILON) * all) break;  // uniform: same sums in every thread
    if (!(all <= DBL_MAX)) {  // NaN / Inf input (a failed factorisation upstream): nothing to converge to
      sweep = kJacobiMaxSweeps;
      break;
    }

    for (int step = 0; step < m - 1; ++step) {
      if (tid < half) {
        // round-robin pairing; step + tid and step + m - 1 - tid stay below 2 (m - 1): one conditional subtraction
        int p = step + tid;
        if (p >= m - 1) p -= m - 1;
        int q = step + m - 1 - tid;
        if (q >= m - 1) q -= m - 1;
        if (tid == 0) q = m - 1;
        double c = 1.0, s = 0.0;
        const double hpq = h[q * m + p];
        if (q < b && hpq != 0.0) {
          // angle |theta| <= pi/4 with tan(2 theta) = 2 h_pq / (h_qq - h_pp):
          //   t = tan(theta) = sgn(a) b2 / (|a| + sqrt(a^2 + b2^2)),  c = 1 / sqrt(1 + t^2),  s = t c.
          // The long-latency double-precision square roots and divisions sit on the critical path of every step, so
          // t is seeded in single precision from operands scaled into [-2, 2] and polished by one Newton step on
          // g(t) = b2 t^2 + 2 a t - b2 in double (g' = 2 sgn(a) r at the root, far from zero; its reciprocal only
          // scales the small correction, so single precision suffices): t is good to ~1e-14.  c and s come from t in
          // double, so c^2 + s^2 = 1 to rounding and the update is an exact similarity transform whatever t is; the
          // rotated h_pq is computed, not set to zero.
          const double a = h[q * m + q] - h[p * m + p], b2 = 2.0 * hpq;
          const double big = fmax(fabs(a), fabs(b2));
          const int e = (__double2hiint(big) >> 20) & 0x7ff;
          double t;
          if (e >= 2 && e <= 2044) {
            const double scale = __hiloint2double((2046 - e) << 20, 0);
            const double as = a * scale, bs = b2 * scale;
            const float af = static_cast<float>(as), bf = static_cast<float>(bs);
            const float rf = sqrtf(fmaf(af, af, bf * bf));
            t = static_cast<double>(__fdividef(a >= 0.0 ? bf : -bf, fabsf(af) + rf));
            const double g = fma(fma(bs, t, 2.0 * as), t, -bs);
            const double gp = 2.0 * fma(bs, t, as);
            t = fma(-g, static_cast<double>(__frcp_rn(static_cast<float>(gp))), t);
          } else {
            const double r = sqrt(a * a + b2 * b2);
            t = (a >= 0.0 ? b2 : -b2) / (fabs(a) + r);
          }
          c = fast_rsqrt_1_2(fma(t, t, 1.0));
          s = t * c;
        }
        rot_p[tid] = p;
        rot_q[tid] = q;
        rot_c[tid] = c;
        rot_s[tid] = s;
      }
      __syncthreads();
      lap(1);
      // this lane's row pairs and its rows of V (as many 32-lane passes as the block cap needs) stay the same for
      // every column pair the warp visits in this step
      constexpr int kPairPasses = (kBlockCap / 2 + 31) / 32;
      constexpr int kRowPasses = (kBlockCap + 31) / 32;
      int pi[kPairPasses], qi[kPairPasses];
      double ci[kPairPasses], si[kPairPasses];
#pragma unroll
      for (int a = 0; a < kPairPasses; ++a) {
        const int ti = lane + 32 * a;
        const bool on = ti < half;
        pi[a] = on ? rot_p[ti] : 0;
        qi[a] = on ? rot_q[ti] : 0;
        ci[a] = on ? rot_c[ti] : 1.0;
        si[a] = on ? rot_s[ti] : 0.0;
      }
      for (int tj = warp; tj < half; tj += kWarps) {
        const int pj = rot_p[tj], qj = rot_q[tj];
        const double cj = rot_c[tj], sj = rot_s[tj];
        double* const hp = h + pj * m;
        double* const hq = h + qj * m;
        double* const vp = v + pj * m;
        double* const vq = v + qj * m;
        // all loads of the column pair first, then the arithmetic, then the stores: the blocks are disjoint
        double ha[kPairPasses], hb[kPairPasses], hc[kPairPasses], hd[kPairPasses];
        double vx[kRowPasses], vy[kRowPasses];
#pragma unroll
        for (int a = 0; a < kPairPasses; ++a) {
          ha[a] = hp[pi[a]];
          hb[a] = hq[pi[a]];
          hc[a] = hp[qi[a]];
          hd[a] = hq[qi[a]];
        }
#pragma unroll
        for (int r = 0; r < kRowPasses; ++r) {
          const int row = lane + 32 * r;
          vx[r] = row < m ? vp[row] : 0.0;
          vy[r] = row < m ? vq[row] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < kPairPasses; ++a) {
          const int ti = lane + 32 * a;
          if (ti >= half) continue;
          // columns (H J_j), then rows (J_i^T ...)
          const double a1 = cj * ha[a] - sj * hb[a], b1 = sj * ha[a] + cj * hb[a];
          const double c1 = cj * hc[a] - sj * hd[a], d1 = sj * hc[a] + cj * hd[a];
          hp[pi[a]] = ci[a] * a1 - si[a] * c1;
          hp[qi[a]] = si[a] * a1 + ci[a] * c1;
          hq[pi[a]] = ci[a] * b1 - si[a] * d1;
          hq[qi[a]] = si[a] * b1 + ci[a] * d1;
        }
#pragma unroll
        for (int r = 0; r < kRowPasses; ++r) {
          const int row = lane + 32 * r;
          if (row < m) {
            vp[row] = cj * vx[r] - sj * vy[r];
            vq[row] = sj * vx[r] + cj * vy[r];
          }
        }
      }
      __syncthreads();
      lap(2);
    }
  }
  return sweep;
}

// In-place Cholesky factorisation of the symmetric positive definite b x b matrix s + shift I (leading dimension m,
// shared) by ONE warp, lane i owning rows i, i + 32, ...: no CTA barrier per column (with sixteen warps and a barrier
// per column the barrier and its stragglers were most of the time).  On return the lower triangle holds L and
// invd[j] = 1 / L(j, j); false (uniformly) when a pivot is not positive.
//
// shift > 0 is the first pass of a shifted Cholesky QR: the oversampling columns of Z = G Q lie, up to the ratio
// lambda_noise / lambda_signal, inside the span of the leading ones, so Z^T Z is numerically singular whenever that
// ratio drops below ~1e-8 and an unshifted factorisation breaks down.  With the shift every pivot is positive; the
// columns it touches come out shorter than unit length, the span is unchanged, and the unshifted passes that follow
// (on a block whose condition number is now moderate) restore orthonormality.
template <int kCap>
__device__ __noinline__ bool cholesky_warp(double* __restrict__ s, double* __restrict__ invd, int b, int m, double shift) {
  constexpr int kPasses = kCap / 32;  // rows per lane
  constexpr int kTiles = kCap / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  __shared__ int ok_flag;
  __syncthreads();
  if (warp == 0) {
    bool ok = true;
    // panels of eight columns.  The panel lives in registers, row i = lane + 32 r in x[r][.]: a column is scaled by
    // 1 / sqrt(d) and pushed into the later columns of the panel through shuffles, nothing touches shared memory on
    // the dependent chain; the columns behind the panel then take S -= L_panel L_panel^T on the FP64 tensor pipe.
    for (int j0 = 0; j0 < b && ok; j0 += 8) {
      double x[kPasses][8];
#pragma unroll
      for (int r = 0; r < kPasses; ++r)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = lane + 32 * r, c = j0 + e;
          x[r][e] = (c < b && i < b && i >= c) ? s[c * m + i] + (i == c ? shift : 0.0) : 0.0;
        }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int c = j0 + e;
        if (c >= b || !ok) break;  // uniform in the warp
        double d = __shfl_sync(0xffffffffu, x[0][e], c & 31);
        if constexpr (kPasses > 1) {
          const double upper = __shfl_sync(0xffffffffu, x[kPasses - 1][e], c & 31);
          if (c >= 32) d = upper;
        }
        if (!(d > 0.0) || !(d <= DBL_MAX)) {
          ok = false;
          break;
        }
        double rinv = rsqrt(d);
        rinv = fma(rinv, fma(-0.5 * d * rinv, rinv, 0.5), rinv);  // one Newton step: within an ulp or two
#pragma unroll
        for (int r = 0; r < kPasses; ++r) {
          const int i = lane + 32 * r;
          x[r][e] = i > c ? x[r][e] * rinv : (i == c ? d * rinv : 0.0);
          if (i == c) invd[c] = rinv;
        }
#pragma unroll
        for (int f = e + 1; f < 8; ++f) {
          const int cf = j0 + f;  // L(cf, c) sits in the lane that owns row cf
          double lf = __shfl_sync(0xffffffffu, x[0][e], cf & 31);
          if constexpr (kPasses > 1) {
            const double upper = __shfl_sync(0xffffffffu, x[kPasses - 1][e], cf & 31);
            if (cf >= 32) lf = upper;
          }
#pragma unroll
          for (int r = 0; r < kPasses; ++r) x[r][f] = fma(-x[r][e], lf, x[r][f]);
        }
      }
      if (!ok) break;
#pragma unroll
      for (int r = 0; r < kPasses; ++r)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = lane + 32 * r, c = j0 + e;
          if (c < b && i < b && i >= c) s[c * m + i] = x[r][e];
        }
      __syncwarp();
      // trailing update, tile row by tile row: every load of a tile row before its first store.  Fragments:
      // A(row, k) = -L(row, j0 + k), B(k, n) = L(column n, j0 + k); a tile may reach past row / column
      // b (reads whatever is there, stores nothing) -- only entries on and below the diagonal are kept.
      const int first = j0 / 8 + 1, tiles = (b + 7) / 8;
      for (int ti = first; ti < tiles; ++ti) {
        const int row = 8 * ti + g;
        const double a0 = -s[(j0 + t) * m + row], a1 = -s[(j0 + 4 + t) * m + row];
        double c0v[kTiles], c1v[kTiles];
#pragma unroll
        for (int tj = 1; tj < kTiles; ++tj) {
          if (tj < first || tj > ti) continue;  // uniform
          const int col = 8 * tj + 2 * t;
          c0v[tj] = s[col * m + row];
          c1v[tj] = s[(col + 1) * m + row];
          dmma884(c0v[tj], c1v[tj], a0, s[(j0 + t) * m + 8 * tj + g]);
          dmma884(c0v[tj], c1v[tj], a1, s[(j0 + 4 + t) * m + 8 * tj + g]);
        }
#pragma unroll
        for (int tj = 1; tj < kTiles; ++tj) {
          if (tj < first || tj > ti) continue;
          const int col = 8 * tj + 2 * t;
          if (row < b && col <= row) s[col * m + row] = c0v[tj];
          if (row < b && col + 1 <= row) s[(col + 1) * m + row] = c1v[tj];
        }
        __syncwarp();
      }
    }
    if (lane == 0) ok_flag = ok ? 1 : 0;
  }
  __syncthreads();
  return ok_flag != 0;
}

// z (rows x b, shared) <- z L^{-T}, in place, in blocks of eight columns; a warp owns 32 consecutive rows for the
// whole solve, so the blocks are separated by warp-level synchronisation only.  Per block:
//   * a thread solves its row against the 8 x 8 diagonal block in registers (right-looking: once x_j = z_j / L(j,j)
//     is known the later columns of the block are updated independently -- one multiplication and one update on the
//     dependent chain per column);
//   * the warp subtracts X_block L(trailing, block)^T from its rows of every later column block on the FP64 tensor
//     pipe (fragment layout as in dmma_accumulate).
// Entries of L read beyond row b only reach registers and columns that are never stored.
static __device__ __noinline__ void trsm_rows_blocked(double* __restrict__ z, const double* __restrict__ l,
                                  const double* __restrict__ invd, int rows, int b, int ld, int m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int base = 32 * warp, row = base + lane;
  const bool live = row < rows;
  const int blocks = (b + 7) / 8;
  if (base < rows) {  // uniform in the warp
    for (int blk = 0; blk < blocks; ++blk) {
      const int c0 = 8 * blk;
      double x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = (live && c0 + e < b) ? z[static_cast<size_t>(c0 + e) * ld + row] : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (c0 + e >= b) break;  // uniform
        const double xe = x[e] * invd[c0 + e];
        x[e] = xe;
        const double* const le = l + (c0 + e) * m + c0;
#pragma unroll
        for (int f = e + 1; f < 8; ++f) x[f] = fma(-xe, le[f], x[f]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (live && c0 + e < b) z[static_cast<size_t>(c0 + e) * ld + row] = x[e];
      if (blk + 1 == blocks) break;  // nothing behind the last block (all eight columns of the others exist)
      __syncwarp();
      const double* const lb0 = l + (c0 + t) * m + g;      // B(k, n) = L(n, block column k): k-step 0
      const double* const lb1 = l + (c0 + 4 + t) * m + g;  // k-step 1
      // the four m-tiles of the warp together, every load of a column block before its first store (the m-tiles
      // beyond the matrix read rows of the following columns and store nothing)
      double a0[4], a1[4];
      int rr[4];  // rows beyond the matrix read its last row instead (z may be global memory) and store nothing
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        rr[mt] = min(base + 8 * mt + g, rows - 1);
        a0[mt] = -z[static_cast<size_t>(c0 + t) * ld + rr[mt]];
        a1[mt] = -z[static_cast<size_t>(c0 + 4 + t) * ld + rr[mt]];
      }
      for (int later = blk + 1; later < blocks; ++later) {
        const int cn = 8 * later;
        const double b0 = lb0[cn], b1 = lb1[cn];
        // (columns beyond b exist only as fragment padding: read the last column instead)
        double* const out0 = z + static_cast<size_t>(min(cn + 2 * t, b - 1)) * ld;
        double* const out1 = z + static_cast<size_t>(min(cn + 2 * t + 1, b - 1)) * ld;
        double c0v[4], c1v[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          c0v[mt] = out0[rr[mt]];
          c1v[mt] = out1[rr[mt]];
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          dmma884(c0v[mt], c1v[mt], a0[mt], b0);
          dmma884(c0v[mt], c1v[mt], a1[mt], b1);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (base + 8 * mt + g < rows) {
            if (cn + 2 * t < b) out0[rr[mt]] = c0v[mt];
            if (cn + 2 * t + 1 < b) out1[rr[mt]] = c1v[mt];
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double rsqrt_seed(double x) {  // ~23 bits, straight from the special function unit
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// The same iteration with ONE barrier per step and step-independent addressing, for blocks of at most 64 (every
// rotation of a step fits one lane of a warp), run by the first kActiveWarps warps of the CTA only; the others wait at
// the closing barrier.  A step of this kernel is bound by the number of instructions its warps issue and by one chain
// of dependent operations, so both are kept short:
//   * pairs sit at fixed positions (2t, 2t + 1); instead of re-pairing indices, a step writes the rotated matrix into
//     a second buffer at positions moved by the round-robin permutation pi (position 0 stays, the other m - 1 cycle),
//     so every address is computed once, before the first step.  pi^(m - 1) = id: after a whole sweep everything is
//     back in place.  h/h2 and v/v2 are the two buffers of H (m x m) and V; every entry is written exactly once per
//     step, so nothing a slower warp still reads is overwritten: read -> rotate -> write -> barrier;
//   * every active warp forms all m/2 rotations of the step itself, in its lanes, instead of waiting for them to be
//     published.
// The caller scales h so that its largest entry is of order one (a power of two: exact); pairs whose
// (h_qq - h_pp)^2 + (2 h_pq)^2 underflows against that are left alone (the zero row and column that pad an odd block
// rotate by the identity: b2 = 0 gives s = 0, c = 1).  With cos 2t = |a| / r and sin 2t = b2 / r,
//     c = sqrt((1 + cos 2t) / 2),   s = sgn(a) sin 2t / (2 c),
// which has no cancellation and needs two reciprocal square roots (hardware seed, Newton in double); c^2 + s^2 = 1 to
// rounding whatever the seed's error, so every step is an exact similarity transform, and the rotated h_pq is
// computed, not set to zero.  h, h2, v, v2 16-byte aligned, m even.  On return (after a CTA barrier) the result is in
// h and v; same return value as above; prof: [0] convergence checks, [2] steps.  Not inlined: inside a large kernel
// the register allocator otherwise recomputes the step-independent addresses in every step.
template <int kThreads, int kBlockCap, int kActiveWarps>
__device__ __noinline__ int jacobi_pingpong_smem(double* h, double* h2, double* v, double* v2, int b, int m,
                                    long long* prof = nullptr) {
  static_assert(kBlockCap <= 64, "one rotation per lane");
  static_assert(kActiveWarps * 32 <= kThreads, "active warps are warps of the CTA");
  const int half = m / 2;
  constexpr int kRowPasses = (kBlockCap + 31) / 32;
  constexpr int kMaxPairs = (kBlockCap / 2 + kActiveWarps - 1) / kActiveWarps;  // column pairs of a warp
  __shared__ double red[2 * kActiveWarps];
  __shared__ int sweeps_used;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto team_barrier = [] { asm volatile("bar.sync 1, %0;\n" ::"n"(kActiveWarps * 32) : "memory"); };
  // where the content of position x goes in a step
  auto moved = [&](int x) {
    if (x != 0 && half > 1) x = (x & 1) ? (x == 1 ? 2 : x - 2) : (x == m - 2 ? m - 1 : x + 2);
    return x;
  };

  if (warp < kActiveWarps) {
    double* hc = h;
    double* hn = h2;
    double* vc = v;
    double* vn = v2;
    long long mark = prof ? clock64() : 0;
    auto lap = [&](int which) {
      if (prof && tid == 0) {
        const long long now = clock64();
        prof[which] += now - mark;
        mark = now;
      }
    };
    // this lane's row pair (2 lane, 2 lane + 1): offsets of its diagonal block and where its rows go
    const bool rot_on = lane < half;
    const int my = rot_on ? lane : 0;
    const int diag_off = 2 * my * m + 2 * my;
    const int to_p = moved(2 * my), to_q = moved(2 * my + 1);
    // this warp's column pairs: read offsets and write offsets
    int col_off[kMaxPairs], to_pc[kMaxPairs], to_qc[kMaxPairs];
#pragma unroll
    for (int u = 0; u < kMaxPairs; ++u) {
      const int tj = warp + u * kActiveWarps;
      const int j = tj < half ? tj : 0;
      col_off[u] = 2 * j * m;
      to_pc[u] = moved(2 * j) * m;
      to_qc[u] = moved(2 * j + 1) * m;
    }
    int sweep = 0;
    for (; sweep < kJacobiMaxSweeps; ++sweep) {
      double off = 0.0, all = 0.0;
      for (int col = warp; col < m; col += kActiveWarps)
        for (int row = lane; row < m; row += 32) {
          const double x = hc[col * m + row] * hc[col * m + row];
          all += x;
          if (row != col) off += x;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
      }
      if (lane == 0) {
        red[warp] = off;
        red[kActiveWarps + warp] = all;
      }
      team_barrier();
      off = 0.0;
      all = 0.0;
      for (int i = 0; i < kActiveWarps; ++i) {
        off += red[i];
        all += red[kActiveWarps + i];
      }
      team_barrier();
      lap(0);
      if (off <= (b * DBL_EPSILON) * (b * DBL_EPSILON) * all) break;  // uniform: same sums in every thread
      if (!(all <= DBL_MAX)) {  // NaN / Inf input (a failed factorisation upstream): nothing to converge to
        sweep = kJacobiMaxSweeps;
        break;
      }

      for (int step = 0; step < m - 1; ++step) {
        // operands first (they do not depend on the rotations): all loads of a step are in flight before its first
        // store, and the column pairs of a warp are not serialised behind one another
        double2 top[kMaxPairs], bot[kMaxPairs];  // (row p_i, row q_i) of column p_j, of column q_j
        double vx[kMaxPairs][kRowPasses], vy[kMaxPairs][kRowPasses];
#pragma unroll
        for (int u = 0; u < kMaxPairs; ++u) {
          if (warp + u * kActiveWarps >= half) break;  // uniform in the warp
          const double* const cp = hc + col_off[u] + 2 * my;
          top[u] = *reinterpret_cast<const double2*>(cp);
          bot[u] = *reinterpret_cast<const double2*>(cp + m);
#pragma unroll
          for (int r = 0; r < kRowPasses; ++r) {
            const int row = lane + 32 * r;
            vx[u][r] = row < m ? vc[col_off[u] + row] : 0.0;
            vy[u][r] = row < m ? vc[col_off[u] + m + row] : 0.0;
          }
        }
        double ci = 1.0, si = 0.0;
        {
          const double2 pq = *reinterpret_cast<const double2*>(hc + diag_off);  // h_pp, h_qp
          const double a = hc[diag_off + m + 1] - pq.x, b2 = 2.0 * pq.y;
          const double n2 = fma(a, a, b2 * b2);
          if (rot_on && n2 > 1e-290) {
            double y = rsqrt_seed(n2);
            const double hn2 = 0.5 * n2;
            y = fma(y, fma(-hn2 * y, y, 0.5), y);
            y = fma(y, fma(-hn2 * y, y, 0.5), y);           // 1 / r
            const double x = fma(0.5 * fabs(a), y, 0.5);    // cos^2: in [1/2, 1]
            double w = rsqrt_seed(x);
            const double hx = 0.5 * x;
            w = fma(w, fma(-hx * w, w, 0.5), w);
            w = fma(w, fma(-hx * w, w, 0.5), w);            // 1 / c
            ci = x * w;
            si = (a >= 0.0 ? 0.5 : -0.5) * (b2 * y) * w;
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxPairs; ++u) {
          const int tj = warp + u * kActiveWarps;
          if (tj >= half) break;  // uniform in the warp
          const double cj = __shfl_sync(0xffffffffu, ci, tj), sj = __shfl_sync(0xffffffffu, si, tj);
          if (rot_on) {
            // columns (H J_j), then rows (J_i^T ...)
            const double a1 = cj * top[u].x - sj * bot[u].x, b1 = sj * top[u].x + cj * bot[u].x;
            const double c1 = cj * top[u].y - sj * bot[u].y, d1 = sj * top[u].y + cj * bot[u].y;
            hn[to_pc[u] + to_p] = ci * a1 - si * c1;
            hn[to_pc[u] + to_q] = si * a1 + ci * c1;
            hn[to_qc[u] + to_p] = ci * b1 - si * d1;
            hn[to_qc[u] + to_q] = si * b1 + ci * d1;
          }
#pragma unroll
          for (int r = 0; r < kRowPasses; ++r) {
            const int row = lane + 32 * r;
            if (row < m) {
              vn[to_pc[u] + row] = cj * vx[u][r] - sj * vy[u][r];
              vn[to_qc[u] + row] = sj * vx[u][r] + cj * vy[u][r];
            }
          }
        }
        team_barrier();
        double* t = hc;
        hc = hn;
        hn = t;
        t = vc;
        vc = vn;
        vn = t;
      }
      lap(2);
    }
    if (hc != h) {  // uniform: an odd number of steps in all
      for (int e = tid; e < m * m; e += kActiveWarps * 32) {
        h[e] = hc[e];
        v[e] = vc[e];
      }
    }
    if (tid == 0) sweeps_used = sweep;
  }
  __syncthreads();
  return sweeps_used;
}

}  // namespace tpb
