// Probe: FP64 DFMA throughput per SM as a function of warps per SM and independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void chain(double* out, int iters) {
  double a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K>
void run(double* out, int warps) {
  const int iters = 2000;
  chain<K><<<148, warps * 32>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); chain<K><<<148, warps * 32>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double n = 16.0 * K * iters * 148 * warps * 32;
  printf("K=%2d warps/SM=%2d: %.1f DFMA/clk/SM  (%.1f cycles per dependent DFMA per warp)\n", K, warps,
         n / (ms * 1e-3) / 148 / 1.965e9, (ms * 1e-3) * 1.965e9 / (16.0 * iters));
}
int main() {
  double* out; cudaMalloc(&out, 8 * 148 * 1024);
  for (int w : {4, 8, 16, 32}) { run<1>(out, w); run<2>(out, w); run<4>(out, w); run<8>(out, w); run<16>(out, w); }
  return 0;
}
