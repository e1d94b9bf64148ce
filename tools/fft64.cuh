// EXPERIMENT (measured slower, not used by the library).
// Wide fp64 FFT block for sm_100a: one length-4096 transform owned by 64
// threads (two warps), 64 complex values per thread, radix plan [64, 64] —
// one exchange per transform instead of the two of the [16,16,16] block in
// fft.cuh, and a two-warp barrier domain, so four transforms per SM run
// independently of one another.  Layout contract on entry and exit: register
// r of thread t holds element / frequency t + 64 r.
#pragma once
#include "../paper_1905_09071_b200/csrc/fft.cuh"

namespace ttagg {

// cos(2 pi m / 64), m = 0..16
__device__ constexpr double C64T[17] = {1.0,
                                        0.99518472667219692873,
                                        0.98078528040323043058,
                                        0.95694033573220882438,
                                        0.92387953251128673848,
                                        0.88192126434835504956,
                                        0.83146961230254523567,
                                        0.77301045336273699338,
                                        0.70710678118654757274,
                                        0.63439328416364548779,
                                        0.55557023301960228867,
                                        0.47139673682599780857,
                                        0.38268343236508983729,
                                        0.29028467725446233105,
                                        0.19509032201612833135,
                                        0.09801714032956077016,
                                        0.0};
__host__ __device__ constexpr double cos64(int m) {
  m = ((m % 64) + 64) % 64;
  if (m > 32) m = 64 - m;
  return m > 16 ? -C64T[32 - m] : C64T[m];
}
__host__ __device__ constexpr double sin64(int m) { return cos64(m - 16); }

// a * W_64^m (W = exp(-2 pi i / 64)), m compile-time
template <int m>
__device__ __forceinline__ cplx w64(cplx a) {
  constexpr int k = m & 63;
  if constexpr (k == 0) return a;
  else if constexpr (k == 16) return mul_mi(a);
  else if constexpr (k == 32) return cplx{-a.x, -a.y};
  else if constexpr (k == 48) return mul_pi(a);
  else if constexpr (k == 8) return cplx{TTAGG_SQRT1_2 * (a.x + a.y), TTAGG_SQRT1_2 * (a.y - a.x)};
  else if constexpr (k == 24) return cplx{TTAGG_SQRT1_2 * (a.y - a.x), -TTAGG_SQRT1_2 * (a.x + a.y)};
  else if constexpr (k == 40) return cplx{-TTAGG_SQRT1_2 * (a.x + a.y), TTAGG_SQRT1_2 * (a.x - a.y)};
  else if constexpr (k == 56) return cplx{TTAGG_SQRT1_2 * (a.x - a.y), TTAGG_SQRT1_2 * (a.x + a.y)};
  else {
    constexpr double wr = cos64(k), wi = -sin64(k);
    return cplx{fma(a.x, wr, -a.y * wi), fma(a.x, wi, a.y * wr)};
  }
}

// DFT-8 in place on eight named values, natural order out
__device__ __forceinline__ void dft8(cplx& v0, cplx& v1, cplx& v2, cplx& v3, cplx& v4, cplx& v5, cplx& v6, cplx& v7) {
  cplx e0 = v0, e1 = v2, e2 = v4, e3 = v6;
  cplx o0 = v1, o1 = v3, o2 = v5, o3 = v7;
  dft4(e0, e1, e2, e3);
  dft4(o0, o1, o2, o3);
  o1 = w16<2>(o1);
  o2 = w16<4>(o2);
  o3 = w16<6>(o3);
  v0 = cadd(e0, o0); v4 = csub(e0, o0);
  v1 = cadd(e1, o1); v5 = csub(e1, o1);
  v2 = cadd(e2, o2); v6 = csub(e2, o2);
  v3 = cadd(e3, o3); v7 = csub(e3, o3);
}

template <int N2, int K1>
__device__ __forceinline__ void tw64_row(cplx (&x)[64]) {
  if constexpr (K1 < 8) {
    x[8 * K1 + N2] = w64<N2 * K1>(x[8 * K1 + N2]);
    tw64_row<N2, K1 + 1>(x);
  }
}
template <int N2>
__device__ __forceinline__ void tw64_all(cplx (&x)[64]) {
  if constexpr (N2 < 8) {
    tw64_row<N2, 1>(x);
    tw64_all<N2 + 1>(x);
  }
}

// position of output frequency k of dft64 in the register array
__host__ __device__ constexpr int perm64(int k) { return 8 * (k & 7) + (k >> 3); }

// DFT-64 in place: n = 8 n1 + n2, k = k1 + 8 k2; X[k] ends up in x[perm64(k)]
__device__ __forceinline__ void dft64(cplx (&x)[64]) {
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2)
    dft8(x[n2], x[8 + n2], x[16 + n2], x[24 + n2], x[32 + n2], x[40 + n2], x[48 + n2], x[56 + n2]);
  // x[8 k1 + n2] = B[n2][k1]; twiddle W_64^(n2 k1)
  tw64_all<1>(x);
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1)
    dft8(x[8 * k1], x[8 * k1 + 1], x[8 * k1 + 2], x[8 * k1 + 3], x[8 * k1 + 4], x[8 * k1 + 5], x[8 * k1 + 6],
         x[8 * k1 + 7]);
}

constexpr int FFT64_PITCH = 65;                       // doubles per exchange row (conflict-free transposed reads)
constexpr int FFT64_EX_DOUBLES = 64 * FFT64_PITCH;    // split (re / im) exchange buffer of one transform

// compiler-only fence: keeps ptxas from hoisting later loads over this point
// (the 64-value transforms leave no registers for early loads)
__device__ __forceinline__ void sched_fence() { asm volatile("" ::: "memory"); }

// v[i] *= w^i, i = 1..63, from w^1..w^7 and w^8, w^16, .., w^56 (table loads)
__device__ __forceinline__ void twiddle64(cplx (&v)[64], const double2* __restrict__ tw, int q) {
  cplx lo[8];
#pragma unroll
  for (int b = 1; b < 8; ++b) lo[b] = ld_c(tw + q * b);
#pragma unroll
  for (int b = 1; b < 8; ++b) v[b] = cmul(v[b], lo[b]);
#pragma unroll
  for (int a = 1; a < 8; ++a) {
    sched_fence();
    const cplx hi = ld_c(tw + ((q * 8 * a) & (TW_BASE - 1)));
    v[8 * a] = cmul(v[8 * a], hi);
#pragma unroll
    for (int b = 1; b < 8; ++b) v[8 * a + b] = cmul(v[8 * a + b], cmul(hi, lo[b]));
  }
  sched_fence();
}

// Forward length-4096 transform by 64 threads (t = 0..63), exchanges in two
// rounds (real parts, then imaginary parts) through `ex` (FFT64_EX_DOUBLES
// doubles, private to this transform); `sync` is a barrier over the 64 threads.
// in: v[r] = x[t + 64 r]; out: v[perm64(r)] = X[t + 64 r].
template <class Sync>
__device__ __forceinline__ void fft4096_wide_raw(cplx (&v)[64], int t, double* ex, const double2* __restrict__ tw,
                                                 const Sync& sync) {
  dft64(v);  // Y[t][ka] in v[perm64(ka)]
#pragma unroll
  for (int ka = 0; ka < 64; ++ka) ex[ka * FFT64_PITCH + t] = v[perm64(ka)].x;
  sync();
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i].x = ex[t * FFT64_PITCH + i];
  sync();
  // imaginary parts: the old ones still sit where stage 1 left them
  // (v[perm64(ka)].y), the new real part of slot i is already in v[i].x
#pragma unroll
  for (int ka = 0; ka < 64; ++ka) ex[ka * FFT64_PITCH + t] = v[perm64(ka)].y;
  sync();
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i].y = ex[t * FFT64_PITCH + i];
  sync();
  twiddle64(v, tw, t);
  dft64(v);  // X[t + 64 kb] in v[perm64(kb)]
}

}  // namespace ttagg
