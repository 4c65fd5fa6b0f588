// Microbenchmark: FP64 pipe ceilings on B200 (sm_100a).
//   - DMMA.8x8x4 issue throughput per SM vs warps/SM and independent accumulators
//   - DFMA throughput
//   - cuBLAS DGEMM ceiling (the roofline denominator P_fp64 used by bench.py)
//   - HBM copy bandwidth (sanity vs MEASURED_PEAKS.json)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o fp64_peaks fp64_peaks.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, p.clockRate);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  const int iters = 20000;
  int warps_list[] = {4, 8, 16, 32};
  for (int wi = 0; wi < 4; ++wi) {
    int warps = warps_list[wi];
    auto report = [&](const char* name, int nacc, float ms, double flops_per_thread_iter_warp) {
      double flops = (double)sms * warps * iters * nacc * flops_per_thread_iter_warp;
      printf("{\"bench\": \"%s\", \"warps_per_sm\": %d, \"nacc\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", name, warps, nacc, ms, flops / ms * 1e-9);
    };
    float ms;
    ms = time_ms([&] { dmma_loop<1><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dmma884", 1, ms, 512.0);
    ms = time_ms([&] { dmma_loop<2><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dmma884", 2, ms, 512.0);
    ms = time_ms([&] { dmma_loop<4><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dmma884", 4, ms, 512.0);
    ms = time_ms([&] { dmma_loop<8><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dmma884", 8, ms, 512.0);
    ms = time_ms([&] { dmma_loop<16><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dmma884", 16, ms, 512.0);
    ms = time_ms([&] { dfma_loop<8><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dfma", 8, ms, 64.0);
    ms = time_ms([&] { dfma_loop<16><<<sms, warps * 32>>>(out, iters, 1.0); }); report("dfma", 16, ms, 64.0);
  }
  // cuBLAS DGEMM ceilings: square, and the HOOI-shaped tall-skinny products
  cublasHandle_t h; cublasCreate(&h);
  struct Shape { int m, n, k; const char* name; } shapes[] = {
    {8192, 8192, 8192, "square8192"}, {4096, 4096, 4096, "square4096"},
    {100, 2560000/4, 1600, "c5_root_quarter(M=100,N=640000,K=1600)"},
    {1600, 100, 1600, "c5_slab(M=1600,N=100,K=1600)"},
    {1600, 1600, 10000, "c5_gram(1600x1600x10000)"}};
  for (auto& s : shapes) {
    double *A, *B, *C;
    CK(cudaMalloc(&A, sizeof(double) * (size_t)s.m * s.k)); CK(cudaMalloc(&B, sizeof(double) * (size_t)s.k * s.n)); CK(cudaMalloc(&C, sizeof(double) * (size_t)s.m * s.n));
    CK(cudaMemset(A, 0, sizeof(double) * (size_t)s.m * s.k)); CK(cudaMemset(B, 0, sizeof(double) * (size_t)s.k * s.n));
    double one = 1, zero = 0;
    float ms = time_ms([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, s.m, s.n, s.k, &one, A, s.m, B, s.k, &zero, C, s.m); }, 5);
    printf("{\"bench\": \"cublas_dgemm\", \"shape\": \"%s\", \"ms\": %.4f, \"tflops\": %.3f}\n", s.name, ms, 2.0 * s.m * s.n * s.k / ms * 1e-9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // sustained DGEMM (2 s) for the power-capped figure
  {
    int n = 8192; double *A, *B, *C; size_t bytes = sizeof(double) * (size_t)n * n;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes)); cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes);
    double one = 1, zero = 0;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = 60; cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\": \"cublas_dgemm_sustained\", \"shape\": \"square8192x%d\", \"ms\": %.3f, \"tflops\": %.3f}\n", reps, ms, 2.0 * n * n * n * reps / ms * 1e-9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // HBM copy
  {
    size_t n = (size_t)1 << 30; // 1 Gi doubles/2 => 8 GiB read + 8 GiB write
    double2 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); cudaMemset(a, 1, n * 8);
    float ms = time_ms([&] { copy_kernel<<<sms * 16, 512>>>(a, b, n / 2); }, 5);
    printf("{\"bench\": \"hbm_copy_kernel\", \"gbytes\": %.2f, \"ms\": %.4f, \"gbs\": %.1f}\n", 2.0 * n * 8 / 1e9, ms, 2.0 * n * 8 / ms * 1e-6);
    ms = time_ms([&] { cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice); }, 5);
    printf("{\"bench\": \"hbm_memcpy_d2d\", \"gbytes\": %.2f, \"ms\": %.4f, \"gbs\": %.1f}\n", 2.0 * n * 8 / 1e9, ms, 2.0 * n * 8 / ms * 1e-6);
  }
  return 0;
}
