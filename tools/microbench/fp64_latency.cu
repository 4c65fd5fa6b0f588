// Dependent-issue latencies that bound the single-CTA small dense kernels (Cholesky, Jacobi, triangular solves):
// cycles per dependent DFMA / DMUL / double rsqrt / division / float MUFU chain / shared-memory round trip /
// __syncthreads at 512 threads.  One warp (or one CTA for the barrier), clock64 around an unrolled dependent chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu && ./fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChain = 512;

template <int OP>
__global__ void chain(double seed, double* out, long long* cycles, int threads_active) {
  __shared__ double sm[1024];
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  sm[threadIdx.x] = x;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kChain; ++i) {
    if (OP == 0) x = fma(x, y, 1e-9);
    if (OP == 1) x = x * y;
    if (OP == 2) x = rsqrt(x + 1.5);
    if (OP == 3) x = 1.0 / (x + 1.5);
    if (OP == 4) x = sqrt(x + 1.5);
    if (OP == 5) { float f = static_cast<float>(x); f = rsqrtf(f + 1.5f); x = static_cast<double>(f); }
    if (OP == 6) { sm[threadIdx.x] = x; x = sm[threadIdx.x ^ 1] + 1e-9; }        // STS -> LDS round trip (same warp)
    if (OP == 7) { __syncthreads(); x += 1e-9; }
    if (OP == 8) { sm[threadIdx.x] = x; __syncthreads(); x = sm[(threadIdx.x + 32) % blockDim.x] + 1e-9; __syncthreads(); }
    if (OP == 9) x = x + y;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  out[threadIdx.x] = x;
  (void)threads_active;
}

template <int OP>
void run(const char* name, int threads) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  chain<OP><<<1, threads>>>(0.5, out, cyc, threads);
  chain<OP><<<1, threads>>>(0.5, out, cyc, threads);
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("{\"op\": \"%s\", \"threads\": %d, \"cycles_per_op\": %.1f}\n", name, threads, double(h) / kChain);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("dfma_dependent", 32);
  run<9>("dadd_dependent", 32);
  run<1>("dmul_dependent", 32);
  run<2>("double_rsqrt_dependent", 32);
  run<3>("double_div_dependent", 32);
  run<4>("double_sqrt_dependent", 32);
  run<5>("cvt_f32_rsqrtf_cvt_f64", 32);
  run<6>("sts_lds_roundtrip", 32);
  run<7>("syncthreads_512", 512);
  run<7>("syncthreads_1024", 1024);
  run<8>("sts_sync_lds_sync_512", 512);
  run<0>("dfma_dependent_16warps", 512);
  return 0;
}
