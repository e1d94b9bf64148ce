// Throwaway probe: FP64 DFMA throughput, DADD throughput, smem 16B bandwidth on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void smem_loop(double* out, int iters) {
  __shared__ double2 buf[2048];
  int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { double2 v = buf[(t + k * 256 + i) & 2047]; acc.x += v.x; acc.y += v.y; }
  }
  out[blockIdx.x * blockDim.x + t] = acc.x + acc.y;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  for (int bs : {256, 512, 1024}) {
    int grid = sms * (2048 / bs);
    dfma_loop<<<grid, bs>>>(out, 10);
    cudaEventRecord(e0); dfma_loop<<<grid, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)grid * bs;
    printf("dfma bs=%d: %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM at 1.965GHz)\n", bs, ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  {
    int grid = sms * 4, bs = 256;
    smem_loop<<<grid, bs>>>(out, 10);
    cudaEventRecord(e0); smem_loop<<<grid, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 16 * iters * (double)grid * bs;
    printf("smem 16B loads: %.3f ms  %.1f B/clk/SM at 1.965GHz\n", ms, bytes / (ms * 1e-3) / sms / 1.965e9);
  }
  {
    size_t n = (size_t)1 << 27; double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    copy_kernel<<<sms * 8, 256>>>(a, b, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_kernel<<<sms * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2GiB: %.1f GB/s\n", 5 * 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  cudaError_t err = cudaGetLastError(); printf("err=%s sms=%d\n", cudaGetErrorString(err), sms);
}
