// Device-side pieces of the small dense eigen-solve shared by evd_kernels.cu (one launch per step, any leaf size) and
// leaf_solve_kernels.cu (the whole top-k solve of a small leaf in one launch).
#pragma once

#include <cuda_runtime.h>

#include <cfloat>

namespace tpb {

constexpr int kEvdMaxBlock = 112;     // largest block the single-CTA kernels take (2 b^2 doubles of shared memory)
constexpr int kJacobiMaxSweeps = 30;

// Parallel cyclic Jacobi on the symmetric matrix h (m x m in shared memory, m even, entries beyond b zero) with the
// rotations accumulated into v (m x m, identity on entry).  Round-robin pairing gives m/2 disjoint rotations per
// step; the step's update H <- J^T H J touches every 2 x 2 block (row pair, column pair) exactly once, so it needs
// no barrier between the column and the row half.  All kThreads threads of the CTA must call it together; on return
// (after a barrier) the eigenvalues sit on the diagonal of h, the eigenvectors in the columns of v, unsorted.
// Returns the number of sweeps used; kJacobiMaxSweeps means the off-diagonal mass never fell below (b eps ||H||_F)^2
// (or the input held NaN / Inf).  kBlockCap >= b sizes the per-lane register passes.
template <int kThreads, int kBlockCap>
__device__ int jacobi_sweeps_smem(double* __restrict__ h, double* __restrict__ v, int b, int m) {
  const int half = m / 2;
  __shared__ double rot_c[kEvdMaxBlock / 2], rot_s[kEvdMaxBlock / 2];
  __shared__ int rot_p[kEvdMaxBlock / 2], rot_q[kEvdMaxBlock / 2];
  constexpr int kWarps = kThreads / 32;
  __shared__ double red[2 * kWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

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
    if (off <= (b * DBL_EPSILON) * (b * DBL_EPSILON) * all) break;  // uniform: same sums in every thread
    if (!(all <= DBL_MAX)) {  // NaN / Inf input (a failed factorisation upstream): nothing to converge to
      sweep = kJacobiMaxSweeps;
      break;
    }

    for (int step = 0; step < m - 1; ++step) {
      if (tid < half) {
        const int p = (step + tid) % (m - 1);
        const int q = (tid == 0) ? (m - 1) : (step + m - 1 - tid) % (m - 1);
        double c = 1.0, s = 0.0;
        const double hpq = h[q * m + p];
        if (q < b && hpq != 0.0) {
          // angle |theta| <= pi/4 with tan(2 theta) = 2 h_pq / (h_qq - h_pp), from cos(2 theta) without tangents
          const double a = h[q * m + q] - h[p * m + p], b2 = 2.0 * hpq;
          const double rinv = rsqrt(a * a + b2 * b2);
          const double c2 = 0.5 + 0.5 * fabs(a) * rinv;  // cos^2(theta)
          const double cinv = rsqrt(c2);
          c = c2 * cinv;
          s = (a >= 0.0 ? 0.5 : -0.5) * b2 * rinv * cinv;
        }
        rot_p[tid] = p;
        rot_q[tid] = q;
        rot_c[tid] = c;
        rot_s[tid] = s;
      }
      __syncthreads();
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
          const bool diag = ti == tj;
          hp[pi[a]] = ci[a] * a1 - si[a] * c1;
          hp[qi[a]] = diag ? 0.0 : si[a] * a1 + ci[a] * c1;
          hq[pi[a]] = diag ? 0.0 : ci[a] * b1 - si[a] * d1;
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
    }
  }
  return sweep;
}

}  // namespace tpb
