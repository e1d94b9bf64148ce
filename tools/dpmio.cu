// Probe: do FP64 instructions and shared-memory instructions overlap on B200?
// Times a loop of NF independent DFMAs and NL shared loads (64- or 128-bit) per iteration,
// each alone and together, at 16 warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int NF, int NL, int WIDE>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  __shared__ double2 buf[2048];
  const int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = t * 1e-3 + q;
  unsigned long long acc = 0;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int f = 0; f < NF; ++f) a[f & 7] = fma(a[f & 7], b, c);
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int idx = (t + 256 * l + 64 * u + i) & 2047;
        if (WIDE) {
          double2 v = buf[idx];
          acc ^= __double_as_longlong(v.x) + __double_as_longlong(v.y);
        } else {
          double v = reinterpret_cast<double*>(buf)[idx * 2];
          acc ^= __double_as_longlong(v);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + t] = s + (double)acc;
}
template <int NF, int NL, int WIDE>
float run(double* out) {
  const int iters = 2000;
  k<NF, NL, WIDE><<<296, 256>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<NF, NL, WIDE><<<296, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // cycles per iteration-unit (one u step) per SM
  const double cyc = (ms * 1e-3) * 1.965e9 / (iters * 4.0);
  printf("NF=%2d NL=%d wide=%d: %.3f ms  %.1f cycles per step per SM (16 warps): DFMA alone would be %.1f, LDS alone %.1f\n", NF, NL, WIDE, ms, cyc,
         NF * 16 * 2 / 4.0, NL * 16 * (WIDE ? 4.0 : 2.0));
  return ms;
}
int main() {
  double* out; cudaMalloc(&out, 8 * 296 * 256);
  run<16, 0, 0>(out); run<0, 2, 0>(out); run<16, 2, 0>(out);
  run<0, 2, 1>(out); run<16, 2, 1>(out);
  run<16, 4, 0>(out); run<0, 4, 0>(out);
  run<32, 2, 0>(out); run<32, 0, 0>(out);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
