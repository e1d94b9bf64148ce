// Microbenchmark + check of the wide FFT block (fft64.cuh: 4096 points on 64
// threads x 64 values, one exchange) against the [16,16,16] block of fft.cuh.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/fftbench64 tools/fftbench64.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include "fft64.cuh"
using namespace ttagg;

template <int G>
__global__ void __launch_bounds__(64 * G, 1) bench_wide(double2* out, const double2* tw, int iters) {
  extern __shared__ double smd[];
  const int g = threadIdx.x / 64, t = threadIdx.x % 64;
  double* ex = smd + g * FFT64_EX_DOUBLES;
  cplx v[64];
#pragma unroll
  for (int r = 0; r < 64; ++r) v[r] = mk(1e-3 * (t + r), 1e-3 * (t - r));
  const GroupSync sync{1 + g, 64};
  for (int it = 0; it < iters; ++it) {
    fft4096_wide_raw(v, t, ex, tw, sync);
    cplx o[64];
#pragma unroll
    for (int r = 0; r < 64; ++r) o[r] = cscale(v[perm64(r)], 1.0 / 64);
#pragma unroll
    for (int r = 0; r < 64; ++r) v[r] = o[r];
  }
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < 64; ++r) { acc.x += v[r].x; acc.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(64) check_wide(const double2* in, double2* out, const double2* tw) {
  extern __shared__ double smd[];
  const int t = threadIdx.x;
  cplx v[64];
#pragma unroll
  for (int r = 0; r < 64; ++r) v[r] = ld_c(in + t + 64 * r);
  fft4096_wide_raw(v, t, smd, tw, GroupSync{1, 64});
#pragma unroll
  for (int r = 0; r < 64; ++r) out[t + 64 * r] = make_double2(v[perm64(r)].x, v[perm64(r)].y);
}

__global__ void __launch_bounds__(256) check_old(const double2* in, double2* out, const double2* tw) {
  extern __shared__ double2 sm2[];
  const int t = threadIdx.x;
  cplx v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = ld_c(in + t + 256 * r);
  fft_fwd<4096>(v, t, sm2, tw);
#pragma unroll
  for (int r = 0; r < 16; ++r) out[t + 256 * r] = make_double2(v[r].x, v[r].y);
}

__global__ void __launch_bounds__(256, 2) bench_old(double2* out, const double2* tw, int iters) {
  extern __shared__ double2 sm2[];
  const int t = threadIdx.x;
  cplx v[16];
  for (int r = 0; r < 16; ++r) v[r] = mk(1e-3 * (t + r), 1e-3 * (t - r));
  for (int it = 0; it < iters; ++it) {
    fft_fwd<4096>(v, t, sm2, tw);
    for (int r = 0; r < 16; ++r) v[r] = cscale(v[r], 1.0 / 64);
  }
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < 16; ++r) { acc.x += v[r].x; acc.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// Closer to pass A's inner loop: per iteration one residue = read z (shared,
// 64 KB), twist by a per-register constant, transform, scale every output by a
// per-register twiddle and store it (to a per-CTA global region that stays in L2).
template <int G>
__global__ void __launch_bounds__(64 * G, 1) bench_res(double2* out, const double2* tw, int iters) {
  extern __shared__ double smd[];
  const int g = threadIdx.x / 64, t = threadIdx.x % 64;
  double* ex = smd + g * FFT64_EX_DOUBLES;
  double2* zs = reinterpret_cast<double2*>(smd + G * FFT64_EX_DOUBLES);
  __shared__ double2 Kst[64], Pst[64];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) zs[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  if (threadIdx.x < 64) {
    Kst[threadIdx.x] = tw[threadIdx.x * 3];
    Pst[threadIdx.x] = tw[threadIdx.x * 5];
  }
  __syncthreads();
  const GroupSync sync{1 + g, 64};
  double2* o = out + ((size_t)blockIdx.x * G + g) * 4096 * 2;
  const cplx tb = ld_c(tw + t);
  for (int it = 0; it < iters; ++it) {
    cplx v[64];
#pragma unroll
    for (int r = 0; r < 64; ++r) v[r] = cmul(lds_c(zs + t + 64 * r), cmul(tb, lds_c(Kst + r)));
    fft4096_wide_raw(v, t, ex, tw, sync);
    double2* oo = o + (it & 1) * 4096;
#pragma unroll
    for (int r = 0; r < 64; ++r) sts_c(oo + t + 64 * r, cmul(v[perm64(r)], cmul(tb, lds_c(Pst + r))));
  }
}

template <int G>
void run_res(double2* out, double2* tw) {
  const size_t smem = (size_t)G * FFT64_EX_DOUBLES * sizeof(double) + 65536;
  cudaFuncSetAttribute(bench_res<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench_res<G>, 64 * G, smem);
  const int grid = 148, iters = 400;
  bench_res<G><<<grid, 64 * G, smem>>>(out, tw, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench_res<G><<<grid, 64 * G, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pts = (double)grid * G * 4096 * iters;
  printf("res  G=%d thr=%d smem=%zu occ=%d/SM: %.3f ms %.2f clk/pt/SM err=%s\n", G, 64 * G, smem, nb, ms,
         148 * 1.965e9 * (ms * 1e-3) / pts, cudaGetErrorString(cudaGetLastError()));
}


// The same loop on the [16,16,16] block as pass A uses it today: 256 threads,
// two CTAs per SM, z in shared memory, split exchanges.
__constant__ double2 cK[8][16];
template <bool TM, bool CK = false>
__global__ void __launch_bounds__(256, 2) bench_res_old(double2* out, const double2* tw, int iters) {
  extern __shared__ __align__(16) double2 sm2[];
  const int t = threadIdx.x;
  __shared__ uint32_t tm_base;
  uint32_t tmw = TMW_NONE;
  if constexpr (TM) {
    if ((t >> 5) == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&tm_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int w = t >> 5;
    tmw = tm_base + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (w >> 2);
    tmem_store_twiddles16(tmw, tw, (t & 15) * 16);
    tmem_store_twiddles16(tmw + 64, tw, t);
  }
  double2* zs = sm2;
  double* ex = reinterpret_cast<double*>(sm2 + 4096);
  __shared__ double2 Kst[16], Pst[16];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) zs[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  if (threadIdx.x < 16) {
    Kst[threadIdx.x] = tw[threadIdx.x * 3];
    Pst[threadIdx.x] = tw[threadIdx.x * 5];
  }
  __syncthreads();
  double2* o = out + (size_t)blockIdx.x * 4096 * 2;
  const cplx tb = ld_c(tw + t);
  for (int it = 0; it < iters; ++it) {
    cplx v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double2 kc = CK ? cK[it % 5][r] : Kst[r];
      v[r] = cmul(lds_c(zs + t + 256 * r), cmul(tb, mk(kc.x, kc.y)));
    }
    fft_fwd_split<4096>(v, t, ex, tw, CtaSync(), nullptr, tmw);
    double2* oo = o + (it & 1) * 4096;
#pragma unroll
    for (int r = 0; r < 16; ++r) sts_c(oo + t + 256 * r, cmul(v[r], cmul(tb, lds_c(Pst + r))));
  }
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if ((t >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm_base) : "memory");
  }
}
template <bool TM, bool CK = false>
void run_res_old(double2* out, double2* tw, int per_sm) {
  const size_t smem = per_sm == 1 ? 120 * 1024 : 65536 + (fft_smem_elems(4096) + 1) * 8;
  cudaFuncSetAttribute(bench_res_old<TM, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench_res_old<TM, CK>, 256, smem);
  const int grid = 148 * per_sm, iters = 400;
  bench_res_old<TM, CK><<<grid, 256, smem>>>(out, tw, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench_res_old<TM, CK><<<grid, 256, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pts = (double)grid * 4096 * iters;
  printf("res_old constK=%d tmem_tw=%d 256thr smem=%zu occ=%d/SM: %.3f ms %.2f clk/pt/SM err=%s\n", (int)CK, (int)TM, smem, nb, ms,
         148 * 1.965e9 * (ms * 1e-3) / pts, cudaGetErrorString(cudaGetLastError()));
}

template <int G>
void run_wide(double2* out, double2* tw) {
  const size_t smem = (size_t)G * FFT64_EX_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(bench_wide<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench_wide<G>, 64 * G, smem);
  const int grid = 148 * 8, iters = 100;
  bench_wide<G><<<grid, 64 * G, smem>>>(out, tw, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench_wide<G><<<grid, 64 * G, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pts = (double)grid * G * 4096 * iters;
  printf("wide G=%d thr=%d smem=%zu occ=%d/SM: %.3f ms %.2f clk/pt/SM err=%s\n", G, 64 * G, smem, nb, ms,
         148 * 1.965e9 * (ms * 1e-3) / pts, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2 *out, *tw, *in, *o1, *o2;
  cudaMalloc(&out, 128 << 20); cudaMalloc(&tw, 4096 * 16);
  cudaMalloc(&in, 4096 * 16); cudaMalloc(&o1, 4096 * 16); cudaMalloc(&o2, 4096 * 16);
  std::vector<double2> h(4096), x(4096), r1(4096), r2(4096);
  for (int m = 0; m < 4096; ++m) h[m] = make_double2(cos(2 * M_PI * m / 4096), -sin(2 * M_PI * m / 4096));
  cudaMemcpy(tw, h.data(), 4096 * 16, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(cK, h.data(), sizeof(double2) * 8 * 16);
  unsigned s = 12345;
  for (int m = 0; m < 4096; ++m) {
    s = s * 1664525u + 1013904223u; double a = (s >> 8) / 16777216.0 - 0.5;
    s = s * 1664525u + 1013904223u; double b = (s >> 8) / 16777216.0 - 0.5;
    x[m] = make_double2(a, b);
  }
  cudaMemcpy(in, x.data(), 4096 * 16, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(check_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, FFT64_EX_DOUBLES * 8);
  cudaFuncSetAttribute(check_old, cudaFuncAttributeMaxDynamicSharedMemorySize, fft_smem_elems(4096) * 16);
  cudaFuncSetAttribute(bench_old, cudaFuncAttributeMaxDynamicSharedMemorySize, fft_smem_elems(4096) * 16);
  check_wide<<<1, 64, FFT64_EX_DOUBLES * 8>>>(in, o1, tw);
  check_old<<<1, 256, fft_smem_elems(4096) * 16>>>(in, o2, tw);
  cudaMemcpy(r1.data(), o1, 4096 * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), o2, 4096 * 16, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int m = 0; m < 4096; ++m) {
    md = fmax(md, fmax(fabs(r1[m].x - r2[m].x), fabs(r1[m].y - r2[m].y)));
    mx = fmax(mx, fmax(fabs(r2[m].x), fabs(r2[m].y)));
  }
  // reference DFT of a few bins on the host
  double mh = 0;
  for (int k : {0, 1, 63, 64, 65, 1000, 2048, 4095}) {
    long double sr = 0, si = 0;
    for (int n = 0; n < 4096; ++n) {
      long double ang = -2.0L * M_PIl * ((long long)n * k % 4096) / 4096.0L;
      sr += x[n].x * cosl(ang) - x[n].y * sinl(ang);
      si += x[n].x * sinl(ang) + x[n].y * cosl(ang);
    }
    mh = fmax(mh, fmax(fabs((double)sr - r1[k].x), fabs((double)si - r1[k].y)));
  }
  printf("check: max|wide-old| = %.3e, max|wide-host| = %.3e (scale %.3e) err=%s\n", md, mh, mx,
         cudaGetErrorString(cudaGetLastError()));
  {
    const size_t smem = fft_smem_elems(4096) * 16;
    const int grid = 148 * 16, iters = 100;
    bench_old<<<grid, 256, smem>>>(out, tw, 2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    bench_old<<<grid, 256, smem>>>(out, tw, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double pts = (double)grid * 4096 * iters;
    printf("old 256thr x2/SM: %.3f ms %.2f clk/pt/SM\n", ms, 148 * 1.965e9 * (ms * 1e-3) / pts);
  }
  run_wide<1>(out, tw);
  run_wide<2>(out, tw);
  run_wide<3>(out, tw);
  run_wide<4>(out, tw);
  run_res_old<true>(out, tw, 2);
  run_res_old<true, true>(out, tw, 2);
  run_res_old<true>(out, tw, 2);
  run_res_old<true, true>(out, tw, 2);
  run_res_old<false>(out, tw, 1);
  run_res_old<true>(out, tw, 1);
  run_res<2>(out, tw);
  run_res<3>(out, tw);
  run_res<4>(out, tw);
  return 0;
}
