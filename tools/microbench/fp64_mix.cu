// Do DMMA.8x8x4 (tensor pipe) and DFMA (fp64 pipe) share one execution resource on B200?
// Runs DMMA-only, DFMA-only and mixed loops (same warp / different warps) and prints combined TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NMMA, int NFMA>
__global__ void mix_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double c[8][2]; double f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = i * 0.25;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NMMA; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i % 8][0]), "+d"(c[i % 8][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NFMA; ++i) f[i % 16] = fma(a, f[i % 16], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// even warps DMMA, odd warps DFMA
__global__ void split_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double s = 0;
  if ((threadIdx.x >> 5) & 1) {
    double f[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = i * 0.25;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = fma(a, f[i], b);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F> float time_ms(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize(); float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 1024));
  const int iters = 20000, warps = 16;
  auto rep = [&](const char* name, int nmma, int nfma, float ms, int w_mma, int w_fma) {
    double fl = (double)sms * iters * ((double)w_mma * nmma * 512.0 + (double)w_fma * nfma * 64.0);
    printf("{\"bench\": \"%s\", \"nmma\": %d, \"nfma\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", name, nmma, nfma, ms, fl / ms * 1e-9);
  };
  float ms;
  ms = time_ms([&] { mix_loop<8, 0><<<sms, warps * 32>>>(out, iters, 1.0); }); rep("dmma_only", 8, 0, ms, warps, warps);
  ms = time_ms([&] { mix_loop<0, 16><<<sms, warps * 32>>>(out, iters, 1.0); }); rep("dfma_only", 0, 16, ms, warps, warps);
  ms = time_ms([&] { mix_loop<8, 16><<<sms, warps * 32>>>(out, iters, 1.0); }); rep("mixed_same_warp_8mma_16fma", 8, 16, ms, warps, warps);
  ms = time_ms([&] { mix_loop<8, 64><<<sms, warps * 32>>>(out, iters, 1.0); }); rep("mixed_same_warp_8mma_64fma", 8, 64, ms, warps, warps);
  ms = time_ms([&] { mix_loop<8, 8><<<sms, warps * 32>>>(out, iters, 1.0); }); rep("mixed_same_warp_8mma_8fma", 8, 8, ms, warps, warps);
  ms = time_ms([&] { split_loop<<<sms, warps * 32>>>(out, iters, 1.0); }); rep("split_warps_8mma|16fma", 8, 16, ms, warps / 2, warps / 2);
  return 0;
}
