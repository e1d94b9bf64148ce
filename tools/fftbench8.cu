// Experiment: 4096-point FFT with 8 values per thread (512 threads, radix 8^4)
// against the 16-per-thread (256 threads, radix 16^3) block of fft.cuh.
#include <cstdio>
#include "../paper_1905_09071_b200/csrc/fft.cuh"
using namespace ttagg;

constexpr int M = 4096, E8 = 8, T8 = M / E8;

__device__ __forceinline__ void twiddle8(cplx* x, cplx w1, cplx w4) {
  const cplx w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  x[1] = cmul(x[1], w1); x[2] = cmul(x[2], w2); x[3] = cmul(x[3], w3); x[4] = cmul(x[4], w4);
  x[5] = cmul(x[5], cmul(w4, w1)); x[6] = cmul(x[6], cmul(w4, w2)); x[7] = cmul(x[7], cmul(w4, w3));
}

template <int NS, bool LAST>
__device__ __forceinline__ void stage8(cplx (&v)[8], int t, double2* sm, const double2* __restrict__ tw) {
  cplx x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = v[i];
  if constexpr (NS > 1) {
    const int qm = t & (NS - 1);
    const int e = qm * (TW_BASE / (NS * 8));
    twiddle8(x, ld_c(tw + e), ld_c(tw + 4 * e));
  }
  DFT<8>::run(x);
  if constexpr (LAST) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = x[i];
  } else {
    const int base = (t / NS) * NS * 8 + (t & (NS - 1));
#pragma unroll
    for (int i = 0; i < 8; ++i) sts_c(sm + pad16(base + i * NS), x[i]);
  }
}
__device__ __forceinline__ void load8(cplx (&v)[8], int t, const double2* sm) {
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = lds_c(sm + pad16(t + T8 * r));
}
__device__ __forceinline__ void fft8(cplx (&v)[8], int t, double2* sm, const double2* tw) {
  stage8<1, false>(v, t, sm, tw); __syncthreads(); load8(v, t, sm); __syncthreads();
  stage8<8, false>(v, t, sm, tw); __syncthreads(); load8(v, t, sm); __syncthreads();
  stage8<64, false>(v, t, sm, tw); __syncthreads(); load8(v, t, sm); __syncthreads();
  stage8<512, true>(v, t, sm, tw);
}

__global__ void __launch_bounds__(512, 2) bench8(double2* out, const double2* tw, int iters) {
  extern __shared__ double2 sm[];
  const int t = threadIdx.x;
  cplx v[8];
  for (int r = 0; r < 8; ++r) v[r] = mk(1e-3 * (t + r), 1e-3 * (t - r));
  for (int it = 0; it < iters; ++it) {
    fft8(v, t, sm, tw);
    for (int r = 0; r < 8; ++r) v[r] = cscale(v[r], 1.0 / 64);
  }
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < 8; ++r) { acc.x += v[r].x; acc.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256, 2) bench16(double2* out, const double2* tw, int iters) {
  extern __shared__ double2 sm[];
  const int t = threadIdx.x;
  cplx v[16];
  for (int r = 0; r < 16; ++r) v[r] = mk(1e-3 * (t + r), 1e-3 * (t - r));
  for (int it = 0; it < iters; ++it) {
    fft_fwd<M>(v, t, sm, tw);
    for (int r = 0; r < 16; ++r) v[r] = cscale(v[r], 1.0 / 64);
  }
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < 16; ++r) { acc.x += v[r].x; acc.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename K>
void run(const char* name, K kern, int threads, double2* out, double2* tw) {
  const size_t smem = (size_t)fft_smem_elems(M) * sizeof(double2);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * 2 * 8, iters = 100;
  kern<<<grid, threads, smem>>>(out, tw, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, threads, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pts = (double)grid * M * iters;
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
  printf("%-10s occ=%d/SM %.3f ms  %.3f clk/pt/SM  %s\n", name, nb, ms, 148 * 1.965e9 * (ms * 1e-3) / pts,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2 *out, *tw;
  cudaMalloc(&out, 64 << 20); cudaMalloc(&tw, 4096 * 16);
  double2 h[4096];
  for (int m = 0; m < 4096; ++m) h[m] = make_double2(cos(2 * M_PI * m / 4096), -sin(2 * M_PI * m / 4096));
  cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    run("16x256", bench16, 256, out, tw);
    run("8x512", bench8, 512, out, tw);
  }
  return 0;
}
