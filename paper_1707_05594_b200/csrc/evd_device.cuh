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

}  // namespace tpb
