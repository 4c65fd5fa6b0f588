// Cycles per step of the shared-memory Jacobi iterations of csrc/evd_device.cuh on a warm-start-like matrix
// (diagonal plus a small symmetric perturbation), one CTA of 512 threads as inside the fused leaf solve.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1707_05594_b200/csrc -o jacobi_step jacobi_step.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#include "evd_device.cuh"

template <int kCap, int kWarps, int kVariant>
__global__ void __launch_bounds__(512, 1) run(const double* in, double* out, long long* prof, int* sweeps, int b) {
  extern __shared__ __align__(16) double sm[];
  const int m = (b + 1) & ~1;
  double* h = sm;
  double* h2 = h + m * m;
  double* v = h2 + m * m;
  double* v2 = v + m * m;
  __shared__ long long p[4];
  if (threadIdx.x < 4) p[threadIdx.x] = 0;
  for (int e = threadIdx.x; e < m * m; e += 512) {
    const int c = e / m, r = e - c * m;
    h[e] = (r < b && c < b) ? in[c * b + r] : 0.0;
    v[e] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  int s;
  if (kVariant == 0)
    s = tpb::jacobi_sweeps_smem<512, kCap>(h, v, b, m, p);
  else
    s = tpb::jacobi_pingpong_smem<512, kCap, kWarps>(h, h2, v, v2, b, m, p);
  __syncthreads();
  if (threadIdx.x == 0) {
    *sweeps = s;
    for (int i = 0; i < 4; ++i) prof[i] = p[i];
  }
  for (int e = threadIdx.x; e < b; e += 512) out[e] = h[e * m + e];
}

template <int kCap, int kWarps, int kVariant>
void bench(const char* name, int b, double eps) {
  std::vector<double> a(b * b);
  srand(7);
  for (int c = 0; c < b; ++c)
    for (int r = 0; r <= c; ++r) {
      const double x = (rand() / double(RAND_MAX) - 0.5);
      a[c * b + r] = a[r * b + c] = r == c ? 1.0 + c + x : eps * x;
    }
  double *din, *dout;
  long long* dprof;
  int* dsw;
  cudaMalloc(&din, b * b * 8);
  cudaMalloc(&dout, b * 8);
  cudaMalloc(&dprof, 32);
  cudaMalloc(&dsw, 4);
  cudaMemcpy(din, a.data(), b * b * 8, cudaMemcpyHostToDevice);
  const int m = (b + 1) & ~1;
  const size_t smem = 4 * m * m * 8;
  cudaFuncSetAttribute(run<kCap, kWarps, kVariant>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    run<kCap, kWarps, kVariant><<<1, 512, smem>>>(din, dout, dprof, dsw, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  long long prof[4];
  int sw;
  cudaMemcpy(prof, dprof, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
  std::vector<double> ev(b);
  cudaMemcpy(ev.data(), dout, b * 8, cudaMemcpyDeviceToHost);
  double tr = 0, tr0 = 0;
  for (int i = 0; i < b; ++i) tr += ev[i], tr0 += a[i * b + i];
  const int steps = sw * (m - 1);
  const long long step_cycles = prof[1] + prof[2] + prof[3];
  double ev_err = 0;  // against the diagonal: the perturbation moves an eigenvalue by O(eps^2)
  { std::vector<double> d0(b), d1(ev); for (int i = 0; i < b; ++i) d0[i] = a[i * b + i]; std::sort(d0.begin(), d0.end()); std::sort(d1.begin(), d1.end()); for (int i = 0; i < b; ++i) ev_err = std::max(ev_err, std::fabs(d0[i] - d1[i])); }
  std::printf("{\"variant\": \"%s\", \"b\": %d, \"eps\": %g, \"sweeps\": %d, \"us\": %.1f, \"cycles_per_step\": %.0f, "
              "\"rot_upd_bar\": [%.0f, %.0f, %.0f], \"check_cycles_per_sweep\": %.0f, \"trace_err\": %.2e, \"err\": \"%s\"}\n",
              name, b, eps, sw, ms * 1e3, steps ? double(step_cycles) / steps : 0.0, double(prof[1]) / steps,
              double(prof[2]) / steps, double(prof[3]) / steps, double(prof[0]) / (sw + 1),
              std::fabs(tr - tr0) / tr0, ev_err, cudaGetErrorString(cudaGetLastError()));
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dprof);
  cudaFree(dsw);
}

int main() {
  for (double eps : {1e-3}) {
    bench<32, 16, 0>("two_barriers_16_warps", 28, eps);
    bench<32, 16, 1>("pingpong_16_warps", 28, eps);
    bench<32, 8, 1>("pingpong_8_warps", 28, eps);
    bench<32, 4, 1>("pingpong_4_warps", 28, eps);
    bench<32, 2, 1>("pingpong_2_warps", 28, eps);
    bench<32, 4, 1>("pingpong_4_warps", 18, eps);
    bench<32, 8, 1>("pingpong_8_warps", 18, eps);
    bench<32, 4, 1>("pingpong_4_warps", 13, eps);
    bench<64, 8, 1>("pingpong_8_warps", 48, eps);
    bench<64, 16, 1>("pingpong_16_warps", 48, eps);
  }
  return 0;
}
