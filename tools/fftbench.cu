// Microbenchmark of the in-register/smem Stockham FFT building block (fft.cuh).
#include <cstdio>
#include "../paper_1905_09071_b200/csrc/fft.cuh"
using namespace ttagg;

template <int M, int GROUPS, bool WARP>
__global__ void bench(double2* out, const double2* tw, int iters) {
  constexpr int E = fft_e(M), T = fft_t(M), SE = fft_smem_elems(M);
  extern __shared__ double2 sm[];
  const int tr = threadIdx.x / T, t = threadIdx.x % T;   // transform index in CTA
  double2* ex = sm + tr * SE;
  cplx v[E];
  for (int r = 0; r < E; ++r) v[r] = mk(1e-3 * (t + r), 1e-3 * (t - r));
  for (int it = 0; it < iters; ++it) {
    if constexpr (WARP) fft_fwd<M, WarpSync>(v, t, ex, tw, WarpSync());
    else if constexpr (GROUPS == 1) fft_fwd<M>(v, t, ex, tw);
    else fft_fwd<M, GroupSync>(v, t, ex, tw, GroupSync{1 + tr, T});
    for (int r = 0; r < E; ++r) v[r] = cscale(v[r], 1.0 / 64);
  }
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < E; ++r) { acc.x += v[r].x; acc.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int M, int NT, int GROUPS, bool WARP>
void run(const char* name, double2* out, double2* tw, int ctas_per_sm) {
  constexpr int T = fft_t(M);
  const int threads = T * NT;
  const size_t smem = (size_t)NT * fft_smem_elems(M) * sizeof(double2);
  cudaFuncSetAttribute(bench<M, GROUPS, WARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 148 * ctas_per_sm * 8;
  int iters = 200;
  bench<M, GROUPS, WARP><<<grid, threads, smem>>>(out, tw, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<M, GROUPS, WARP><<<grid, threads, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double pts = (double)grid * NT * M * iters;
  double flops = pts * 5 * __builtin_log2(M);
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench<M, GROUPS, WARP>, threads, smem);
  printf("%-28s M=%5d thr=%4d smem=%6zu occ=%d/SM: %.3f ms  %.2f Gpts/s  %.1f TFLOP/s(5NlogN)  %.2f clk/pt/SM  err=%s\n", name, M, threads, smem, nb,
         ms, pts / ms / 1e6, flops / ms / 1e9, 148 * 1.965e9 * (ms * 1e-3) / pts, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2 *out, *tw;
  cudaMalloc(&out, 64 << 20); cudaMalloc(&tw, 4096 * 16);
  double2 h[4096];
  for (int m = 0; m < 4096; ++m) h[m] = make_double2(cos(2 * M_PI * m / 4096), -sin(2 * M_PI * m / 4096));
  cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
  run<4096, 1, 1, false>("4096 cta", out, tw, 1);
  run<4096, 2, 2, false>("4096 2groups", out, tw, 1);
  run<2048, 1, 1, false>("2048 cta", out, tw, 2);
  run<2048, 2, 2, false>("2048 2groups", out, tw, 1);
  run<1024, 4, 1, false>("1024 x4 cta", out, tw, 2);
  run<512, 4, 1, true>("512 warp x4", out, tw, 3);
  run<512, 8, 1, true>("512 warp x8", out, tw, 2);
  run<256, 8, 1, true>("256 warp x8", out, tw, 3);
  run<256, 16, 1, true>("256 warp x16", out, tw, 2);
  run<16, 128, 1, true>("16 regs x128", out, tw, 4);
  return 0;
}
