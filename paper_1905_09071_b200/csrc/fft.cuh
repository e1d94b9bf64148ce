// fp64 complex FFT building blocks for sm_100a.
//
// One transform of length M (power of two, 1..4096) is owned by T = M/E
// threads, each holding E = min(16, M) complex values in registers.  The
// transform is a Stockham auto-sort DIT with radix plan [b, 16, 16, ...]
// (b = M / 16^a in {1,2,4,8}); every exchange between stages goes through a
// padded shared-memory buffer (one pad slot per 16 elements keeps the
// 16-byte accesses conflict-free).  Layout contract, identical on entry and
// exit: register r of thread t holds element / frequency  t + T*r.
//
// Twiddles come from one table W_4096^m (m < 4096) in global memory (L1
// resident); W_M^m = W_4096^(m * 4096/M).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ttagg {

struct cplx {
  double x, y;
};

__device__ __forceinline__ cplx mk(double x, double y) { return cplx{x, y}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cplx{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ cplx cmulc(cplx a, cplx b) {  // a * conj(b)
  return cplx{fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)};
}
__device__ __forceinline__ cplx cconj(cplx a) { return cplx{a.x, -a.y}; }
__device__ __forceinline__ cplx cscale(cplx a, double s) { return cplx{a.x * s, a.y * s}; }
__device__ __forceinline__ cplx mul_mi(cplx a) { return cplx{a.y, -a.x}; }  // * (-i)
__device__ __forceinline__ cplx mul_pi(cplx a) { return cplx{-a.y, a.x}; }  // * (+i)

__device__ __forceinline__ cplx ld_c(const double2* p) {
  double2 v = __ldg(p);
  return cplx{v.x, v.y};
}
__device__ __forceinline__ cplx lds_c(const double2* p) {
  double2 v = *p;
  return cplx{v.x, v.y};
}
__device__ __forceinline__ void sts_c(double2* p, cplx v) { *p = make_double2(v.x, v.y); }
// streaming (evict-first) global store: data written once and read by a later kernel
__device__ __forceinline__ void stg_cs(double2* p, cplx v) { __stcs(p, make_double2(v.x, v.y)); }

// ---------------------------------------------------------------------------
// small DFTs (forward, W = exp(-2 pi i / R)), in place on v[0..R)
// ---------------------------------------------------------------------------
template <int R>
struct DFT;

template <>
struct DFT<1> {
  __device__ __forceinline__ static void run(cplx*) {}
};

template <>
struct DFT<2> {
  __device__ __forceinline__ static void run(cplx* v) {
    cplx a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

__device__ __forceinline__ void dft4(cplx& a0, cplx& a1, cplx& a2, cplx& a3) {
  cplx s02 = cadd(a0, a2), d02 = csub(a0, a2);
  cplx s13 = cadd(a1, a3), d13 = mul_mi(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

template <>
struct DFT<4> {
  __device__ __forceinline__ static void run(cplx* v) { dft4(v[0], v[1], v[2], v[3]); }
};

#define TTAGG_SQRT1_2 0.70710678118654752440
#define TTAGG_COS_PI8 0.92387953251128675613
#define TTAGG_SIN_PI8 0.38268343236508977173

// multiply by W_16^m, m compile-time in [0, 16)
template <int m>
__device__ __forceinline__ cplx w16(cplx a) {
  constexpr int k = m & 15;
  if constexpr (k == 0) return a;
  else if constexpr (k == 4) return mul_mi(a);
  else if constexpr (k == 8) return cplx{-a.x, -a.y};
  else if constexpr (k == 12) return mul_pi(a);
  else if constexpr (k == 2) return cplx{TTAGG_SQRT1_2 * (a.x + a.y), TTAGG_SQRT1_2 * (a.y - a.x)};
  else if constexpr (k == 6) return cplx{TTAGG_SQRT1_2 * (a.y - a.x), -TTAGG_SQRT1_2 * (a.x + a.y)};
  else if constexpr (k == 10) return cplx{-TTAGG_SQRT1_2 * (a.x + a.y), TTAGG_SQRT1_2 * (a.x - a.y)};
  else if constexpr (k == 14) return cplx{TTAGG_SQRT1_2 * (a.x - a.y), TTAGG_SQRT1_2 * (a.x + a.y)};
  else {
    // general: cos(2 pi k/16) - i sin(2 pi k/16)
    constexpr double c[16] = {1.0, TTAGG_COS_PI8, TTAGG_SQRT1_2, TTAGG_SIN_PI8, 0.0, -TTAGG_SIN_PI8,
                              -TTAGG_SQRT1_2, -TTAGG_COS_PI8, -1.0, -TTAGG_COS_PI8, -TTAGG_SQRT1_2,
                              -TTAGG_SIN_PI8, 0.0, TTAGG_SIN_PI8, TTAGG_SQRT1_2, TTAGG_COS_PI8};
    constexpr double wr = c[k];
    constexpr double wi = -c[(k + 12) & 15];  // -sin(2 pi k / 16) = -cos(2 pi (k - 4)/16)
    return cplx{fma(a.x, wr, -a.y * wi), fma(a.x, wi, a.y * wr)};
  }
}

template <>
struct DFT<8> {
  __device__ __forceinline__ static void run(cplx* v) {
    // split n = 2 n1 + n2: DFT4 over evens and odds, then W_8 twiddles
    cplx e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    cplx o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    o1 = w16<2>(o1);
    o2 = w16<4>(o2);
    o3 = w16<6>(o3);
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
  }
};

template <>
struct DFT<16> {
  __device__ __forceinline__ static void run(cplx* v) {
    // n = 4 n1 + n2 ; k = k1 + 4 k2
    // step 1: for each n2, DFT4 over n1 of v[4 n1 + n2]
    dft4(v[0], v[4], v[8], v[12]);
    dft4(v[1], v[5], v[9], v[13]);
    dft4(v[2], v[6], v[10], v[14]);
    dft4(v[3], v[7], v[11], v[15]);
    // now v[4 k1 + n2] = B[n2][k1]; twiddle W16^(n2 k1)
    v[5] = w16<1>(v[5]);
    v[6] = w16<2>(v[6]);
    v[7] = w16<3>(v[7]);
    v[9] = w16<2>(v[9]);
    v[10] = w16<4>(v[10]);
    v[11] = w16<6>(v[11]);
    v[13] = w16<3>(v[13]);
    v[14] = w16<6>(v[14]);
    v[15] = w16<9>(v[15]);
    // step 3: for each k1, DFT4 over n2 of B[n2][k1] = v[4 k1 + n2] -> X[k1 + 4 k2]
    dft4(v[0], v[1], v[2], v[3]);
    dft4(v[4], v[5], v[6], v[7]);
    dft4(v[8], v[9], v[10], v[11]);
    dft4(v[12], v[13], v[14], v[15]);
    // v[4 k1 + k2] = X[k1 + 4 k2]: transpose 4x4 to natural order
    cplx t;
    t = v[1]; v[1] = v[4]; v[4] = t;
    t = v[2]; v[2] = v[8]; v[8] = t;
    t = v[3]; v[3] = v[12]; v[12] = t;
    t = v[6]; v[6] = v[9]; v[9] = t;
    t = v[7]; v[7] = v[13]; v[13] = t;
    t = v[11]; v[11] = v[14]; v[14] = t;
  }
};

// ---------------------------------------------------------------------------
// Stockham transform of length M
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }
__host__ __device__ constexpr int fft_e(int M) { return M >= 16 ? 16 : M; }
__host__ __device__ constexpr int fft_t(int M) { return M / fft_e(M); }
// first-stage radix b = M / 16^a
__host__ __device__ constexpr int fft_first_radix(int M) {
  return M >= 16 ? (1 << (ilog2c(M) % 4)) : M;
}
__host__ __device__ constexpr int fft_smem_elems(int M) { return M + (M >> 4) + 1; }
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

constexpr int TW_BASE = 4096;  // twiddle table W_4096^m

// Barrier used between FFT stages: the whole CTA, or a named barrier over
// one thread group (bar.sync id, nthreads; id 0 is __syncthreads).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct WarpSync {  // all threads of one transform live in one warp (T <= 32)
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct GroupSync {
  int id, n;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};

// x[i] *= w^i for i = 1..15 with w^1, w^4 loaded: the other powers need at
// most two multiplications from a table value (keeps twiddles within ~2 ulp)
__device__ __forceinline__ void twiddle16(cplx* x, cplx w1, cplx w4) {
  const cplx w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  const cplx w8 = cmul(w4, w4), w12 = cmul(w8, w4);
  x[1] = cmul(x[1], w1);
  x[2] = cmul(x[2], w2);
  x[3] = cmul(x[3], w3);
  x[4] = cmul(x[4], w4);
  x[5] = cmul(x[5], cmul(w4, w1));
  x[6] = cmul(x[6], cmul(w4, w2));
  x[7] = cmul(x[7], cmul(w4, w3));
  x[8] = cmul(x[8], w8);
  x[9] = cmul(x[9], cmul(w8, w1));
  x[10] = cmul(x[10], cmul(w8, w2));
  x[11] = cmul(x[11], cmul(w8, w3));
  x[12] = cmul(x[12], w12);
  x[13] = cmul(x[13], cmul(w12, w1));
  x[14] = cmul(x[14], cmul(w12, w2));
  x[15] = cmul(x[15], cmul(w12, w3));
}

// ---- tensor memory (TMEM) as per-thread storage (tcgen05.alloc / st / ld,
// 32x32b shape: a thread reads and writes the columns of its own lane; warp w
// of a CTA owns lanes 32 (w % 4) .. +31)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Stage twiddles kept in tensor memory: the 15 powers w^1..w^15 of a
// twiddled radix-16 stage depend on the thread only (w = W_{16 NS}^(t mod NS)),
// so a persistent CTA stores them once (64 TMEM columns per stage: slot i =
// w^i, slot 0 unused) and every transform reads them back instead of
// rebuilding them from w^1 and w^4 (13 complex products per stage).
constexpr uint32_t TMW_NONE = 0xffffffffu;
__device__ __forceinline__ void tmem_store_twiddles16(uint32_t taddr, const double2* __restrict__ tw, int e) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t r[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 w = tw[((4 * q + u) * e) & (4096 - 1)];
      r[4 * u + 0] = (uint32_t)__double2loint(w.x);
      r[4 * u + 1] = (uint32_t)__double2hiint(w.x);
      r[4 * u + 2] = (uint32_t)__double2loint(w.y);
      r[4 * u + 3] = (uint32_t)__double2hiint(w.y);
    }
    tmem_st16(taddr + 16 * q, r);
  }
  tmem_wait_st();
}
__device__ __forceinline__ void twiddle16_tmem(cplx* x, uint32_t taddr) {
  uint32_t r[4][16];
#pragma unroll
  for (int q = 0; q < 4; ++q) tmem_ld16(taddr + 16 * q, r[q]);
  tmem_wait_ld();
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    const int q = i >> 2, u = i & 3;
    const cplx w = mk(__hiloint2double((int)r[q][4 * u + 1], (int)r[q][4 * u]),
                      __hiloint2double((int)r[q][4 * u + 3], (int)r[q][4 * u + 2]));
    x[i] = cmul(x[i], w);
  }
}

// One stage.  Registers: element t + T*r in v[r] on entry (read pattern).
template <int M, int R, int NS, bool LAST>
__device__ __forceinline__ void fft_stage(cplx (&v)[fft_e(M)], int t, double2* sm, const double2* __restrict__ tw,
                                          const double2* stw = nullptr, uint32_t tmw = TMW_NONE) {
  constexpr int E = fft_e(M);
  constexpr int T = fft_t(M);
  constexpr int G = E / R;  // butterflies per thread
#pragma unroll
  for (int u = 0; u < G; ++u) {
    const int q = t + T * u;
    cplx x[R];
#pragma unroll
    for (int i = 0; i < R; ++i) x[i] = v[u + i * G];
    if constexpr (NS > 1) {
      // W_{NS R}^{i qm} = W_4096^{i qm 4096/(NS R)}
      const int qm = q & (NS - 1);
      const int e = qm * (TW_BASE / (NS * R));
#ifndef TTAGG_TW_MODE
#define TTAGG_TW_MODE 0
#endif
      if constexpr (R == 16 && TTAGG_TW_MODE == 0) {
        if (tmw != TMW_NONE) twiddle16_tmem(x, tmw);
        else if (stw) twiddle16(x, lds_c(stw + qm), lds_c(stw + NS + qm));
        else twiddle16(x, ld_c(tw + e), ld_c(tw + 4 * e));
      } else if constexpr (R == 16 && TTAGG_TW_MODE == 2) {
        // w1..w3 and w4, w8, w12 loaded; 9 products
        const cplx w1 = ld_c(tw + e), w2 = ld_c(tw + 2 * e), w3 = ld_c(tw + 3 * e);
        const cplx w4 = ld_c(tw + 4 * e), w8 = ld_c(tw + 8 * e), w12 = ld_c(tw + 12 * e);
        x[1] = cmul(x[1], w1); x[2] = cmul(x[2], w2); x[3] = cmul(x[3], w3);
        x[4] = cmul(x[4], w4); x[8] = cmul(x[8], w8); x[12] = cmul(x[12], w12);
        x[5] = cmul(x[5], cmul(w4, w1)); x[6] = cmul(x[6], cmul(w4, w2)); x[7] = cmul(x[7], cmul(w4, w3));
        x[9] = cmul(x[9], cmul(w8, w1)); x[10] = cmul(x[10], cmul(w8, w2)); x[11] = cmul(x[11], cmul(w8, w3));
        x[13] = cmul(x[13], cmul(w12, w1)); x[14] = cmul(x[14], cmul(w12, w2)); x[15] = cmul(x[15], cmul(w12, w3));
      } else {
#pragma unroll
        for (int i = 1; i < R; ++i) x[i] = cmul(x[i], ld_c(tw + i * e));
      }
    }
    DFT<R>::run(x);
    if constexpr (LAST) {
#pragma unroll
      for (int i = 0; i < R; ++i) v[u + i * G] = x[i];
    } else {
      const int base = (q / NS) * NS * R + (q & (NS - 1));
#pragma unroll
      for (int i = 0; i < R; ++i) sts_c(sm + pad16(base + i * NS), x[i]);
    }
  }
}

template <int M>
__device__ __forceinline__ void fft_load_regs(cplx (&v)[fft_e(M)], int t, const double2* sm) {
  constexpr int E = fft_e(M);
  constexpr int T = fft_t(M);
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = lds_c(sm + pad16(t + T * r));
}

// Forward FFT of length M (no normalisation).  All threads of the CTA must
// call it (it contains __syncthreads when M > 16); `sm` is this transform's
// private buffer of fft_smem_elems(M) slots.
template <int M>
__host__ __device__ constexpr int fft_stage_ns(int which);

template <int M, class Sync = CtaSync>
__device__ __forceinline__ void fft_fwd(cplx (&v)[fft_e(M)], int t, double2* sm, const double2* __restrict__ tw,
                                        const Sync& sync = Sync(), const double2* stw = nullptr,
                                        uint32_t tmw = TMW_NONE) {
  if constexpr (M <= 16) {
    DFT<M>::run(v);
    // DFT<R> leaves natural order, and with T == 1 register r == frequency r
  } else {
    constexpr int b = fft_first_radix(M);
    constexpr int a = (ilog2c(M) - ilog2c(b)) / 4;  // number of radix-16 stages
    static_assert(a >= 1, "M >= 16");
    int ns_done;
    if constexpr (b > 1) {
      fft_stage<M, b, 1, false>(v, t, sm, tw);
      sync();
      fft_load_regs<M>(v, t, sm);
      sync();
    }
    constexpr int NS1 = b;
    // radix-16 stages: NS = b, 16 b, 256 b, ...
    if constexpr (a == 1) {
      fft_stage<M, 16, NS1, true>(v, t, sm, tw);
    } else if constexpr (a == 2) {
      fft_stage<M, 16, NS1, false>(v, t, sm, tw, stw);
      sync();
      fft_load_regs<M>(v, t, sm);
      sync();
      // tmw (b == 1 only): the one twiddled stage reads its twiddles from tensor memory
      fft_stage<M, 16, NS1 * 16, true>(v, t, sm, tw, stw ? stw + 2 * fft_stage_ns<M>(0) : nullptr,
                                       b == 1 ? tmw : TMW_NONE);
    } else {
      static_assert(a == 3, "M <= 4096");
      fft_stage<M, 16, NS1, false>(v, t, sm, tw);
      sync();
      fft_load_regs<M>(v, t, sm);
      sync();
      fft_stage<M, 16, NS1 * 16, false>(v, t, sm, tw, stw);
      sync();
      fft_load_regs<M>(v, t, sm);
      sync();
      fft_stage<M, 16, NS1 * 256, true>(v, t, sm, tw, stw ? stw + 2 * fft_stage_ns<M>(0) : nullptr);
    }
    (void)ns_done;
  }
}

// Two independent forward transforms of length M interleaved stage by stage
// (twice the independent work between barriers, half the barriers); each has
// its own exchange buffer.
template <int M, class Sync = CtaSync>
__device__ __forceinline__ void fft_fwd2(cplx (&v1)[fft_e(M)], cplx (&v2)[fft_e(M)], int t, double2* sm1, double2* sm2,
                                         const double2* __restrict__ tw, const Sync& sync = Sync()) {
  constexpr int b = fft_first_radix(M);
  constexpr int a = (ilog2c(M) - ilog2c(b)) / 4;
  static_assert(M >= 256 && a >= 2 && a <= 3, "256 <= M <= 4096");
  auto xchg = [&]() {
    sync();
    fft_load_regs<M>(v1, t, sm1);
    fft_load_regs<M>(v2, t, sm2);
    sync();
  };
  if constexpr (b > 1) {
    fft_stage<M, b, 1, false>(v1, t, sm1, tw);
    fft_stage<M, b, 1, false>(v2, t, sm2, tw);
    xchg();
  }
  constexpr int NS1 = b;
  if constexpr (a == 2) {
    fft_stage<M, 16, NS1, false>(v1, t, sm1, tw);
    fft_stage<M, 16, NS1, false>(v2, t, sm2, tw);
    xchg();
    fft_stage<M, 16, NS1 * 16, true>(v1, t, sm1, tw);
    fft_stage<M, 16, NS1 * 16, true>(v2, t, sm2, tw);
  } else {
    fft_stage<M, 16, NS1, false>(v1, t, sm1, tw);
    fft_stage<M, 16, NS1, false>(v2, t, sm2, tw);
    xchg();
    fft_stage<M, 16, NS1 * 16, false>(v1, t, sm1, tw);
    fft_stage<M, 16, NS1 * 16, false>(v2, t, sm2, tw);
    xchg();
    fft_stage<M, 16, NS1 * 256, true>(v1, t, sm1, tw);
    fft_stage<M, 16, NS1 * 256, true>(v2, t, sm2, tw);
  }
}

// ---------------------------------------------------------------------------
// Half-footprint exchanges: the same transform with every exchange done in
// two rounds (real parts, then imaginary parts) through a buffer of
// fft_smem_elems(M) doubles — half the shared memory of fft_fwd, two more
// barriers per exchange, no extra registers (a value's real and imaginary
// halves live in separate registers, so the new real parts can land while
// the old imaginary parts still wait to be written).
// ---------------------------------------------------------------------------
template <int M, int R, int NS, class Sync>
__device__ __forceinline__ void fft_stage_split(cplx (&v)[fft_e(M)], int t, double* sm, const double2* __restrict__ tw,
                                                const Sync& sync, const double2* stw = nullptr,
                                                uint32_t tmw = TMW_NONE) {
  constexpr int E = fft_e(M);
  constexpr int T = fft_t(M);
  constexpr int G = E / R;
  int dst[E];
#pragma unroll
  for (int u = 0; u < G; ++u) {
    const int q = t + T * u;
    cplx x[R];
#pragma unroll
    for (int i = 0; i < R; ++i) x[i] = v[u + i * G];
    if constexpr (NS > 1) {
      const int qm = q & (NS - 1);
      const int e = qm * (TW_BASE / (NS * R));
      if constexpr (R == 16) {
        if (tmw != TMW_NONE) twiddle16_tmem(x, tmw);
        else if (stw) twiddle16(x, lds_c(stw + qm), lds_c(stw + NS + qm));
        else twiddle16(x, ld_c(tw + e), ld_c(tw + 4 * e));
      } else {
#pragma unroll
        for (int i = 1; i < R; ++i) x[i] = cmul(x[i], ld_c(tw + i * e));
      }
    }
    DFT<R>::run(x);
    const int base = (q / NS) * NS * R + (q & (NS - 1));
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[u + i * G] = x[i];
      dst[u + i * G] = pad16(base + i * NS);
    }
  }
#pragma unroll
  for (int r = 0; r < E; ++r) sm[dst[r]] = v[r].x;
  sync();
#pragma unroll
  for (int r = 0; r < E; ++r) v[r].x = sm[pad16(t + T * r)];
  sync();
#pragma unroll
  for (int r = 0; r < E; ++r) sm[dst[r]] = v[r].y;
  sync();
#pragma unroll
  for (int r = 0; r < E; ++r) v[r].y = sm[pad16(t + T * r)];
  sync();
}

// Stage-twiddle table for the twiddled radix-16 stages of a length-M
// transform (shared memory, filled once per CTA by fft_stage_table): for each
// such stage with NS sub-transforms, w1[NS] then w4[NS] (w = W_{16 NS}^qm).
// Its reads are unit-stride across the warp, where the W_4096 table gathers
// touch up to 16 lines per warp load.
template <int M>
__host__ __device__ constexpr int fft_stage_ns(int which) {  // NS of the two twiddled radix-16 stages
  return M >= 4096 ? (which ? 256 : 16) : (which ? 16 * fft_first_radix(M) : fft_first_radix(M));
}
template <int M>
__host__ __device__ constexpr int fft_stage_table_elems() {
  return 2 * (fft_stage_ns<M>(0) + fft_stage_ns<M>(1));
}
template <int M>
__device__ __forceinline__ void fft_stage_table(double2* stw, const double2* __restrict__ tw, int t, int nthreads) {
  constexpr int NSa = fft_stage_ns<M>(0), NSb = fft_stage_ns<M>(1);
  for (int i = t; i < 2 * (NSa + NSb); i += nthreads) {
    const bool second = i >= 2 * NSa;
    const int NS = second ? NSb : NSa;
    const int k = second ? i - 2 * NSa : i;
    const int qm = k % NS, pw = k < NS ? 1 : 4;
    stw[i] = tw[pw * qm * (TW_BASE / (NS * 16))];
  }
}

// Length-4096 transform (16 values per thread, 256 threads), split exchanges,
// tensor-memory stage twiddles with the first half of each stage's twiddles
// (w^1..w^7) requested before the exchange's last round, so their latency
// hides behind that round's loads and barrier; the second half is requested
// while the first is being applied.
#ifndef TTAGG_TW_HALFPRE
#define TTAGG_TW_HALFPRE 1
#endif
__device__ __forceinline__ cplx tw_slot(const uint32_t (&r)[16], int u) {
  return mk(__hiloint2double((int)r[4 * u + 1], (int)r[4 * u]), __hiloint2double((int)r[4 * u + 3], (int)r[4 * u + 2]));
}
template <class Sync>
__device__ __forceinline__ void split_exchange16_pre(cplx (&v)[16], const int (&dst)[16], int t, double* sm,
                                                     const Sync& sync, uint32_t tnext, uint32_t (&w0)[16],
                                                     uint32_t (&w1)[16]) {
  constexpr int T = 256;
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[dst[r]] = v[r].x;
  sync();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r].x = sm[pad16(t + T * r)];
  sync();
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[dst[r]] = v[r].y;
  sync();
  tmem_ld16(tnext, w0);
  tmem_ld16(tnext + 16, w1);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r].y = sm[pad16(t + T * r)];
  sync();
}
__device__ __forceinline__ void tw_apply_halves(cplx (&v)[16], uint32_t taddr, uint32_t (&w0)[16], uint32_t (&w1)[16]) {
  tmem_wait_ld();
#pragma unroll
  for (int u = 1; u < 4; ++u) v[u] = cmul(v[u], tw_slot(w0, u));
#pragma unroll
  for (int u = 0; u < 4; ++u) v[4 + u] = cmul(v[4 + u], tw_slot(w1, u));
  tmem_ld16(taddr + 32, w0);
  tmem_ld16(taddr + 48, w1);
  tmem_wait_ld();
#pragma unroll
  for (int u = 0; u < 4; ++u) v[8 + u] = cmul(v[8 + u], tw_slot(w0, u));
#pragma unroll
  for (int u = 0; u < 4; ++u) v[12 + u] = cmul(v[12 + u], tw_slot(w1, u));
}
template <class Sync>
__device__ __forceinline__ void fft4096_split_tm(cplx (&v)[16], int t, double* sm, const Sync& sync, uint32_t tmw) {
  uint32_t w0[16], w1[16];
  int dst[16];
  DFT<16>::run(v);  // stage 1: NS = 1, no twiddles; output i of butterfly q = t goes to 16 q + i
#pragma unroll
  for (int i = 0; i < 16; ++i) dst[i] = pad16(t * 16 + i);
  split_exchange16_pre(v, dst, t, sm, sync, tmw, w0, w1);
  tw_apply_halves(v, tmw, w0, w1);  // stage 2: NS = 16
  DFT<16>::run(v);
  {
    const int base = (t / 16) * 256 + (t & 15);
#pragma unroll
    for (int i = 0; i < 16; ++i) dst[i] = pad16(base + i * 16);
  }
  split_exchange16_pre(v, dst, t, sm, sync, tmw + 64, w0, w1);
  tw_apply_halves(v, tmw + 64, w0, w1);  // stage 3: NS = 256 (last): natural order in the registers
  DFT<16>::run(v);
}

template <int M, class Sync = CtaSync>
__device__ __forceinline__ void fft_fwd_split(cplx (&v)[fft_e(M)], int t, double* sm, const double2* __restrict__ tw,
                                              const Sync& sync = Sync(), const double2* stw = nullptr,
                                              uint32_t tmw = TMW_NONE) {
  static_assert(M >= 256 && M <= 4096, "block transforms");
  if constexpr (M == 4096 && TTAGG_TW_HALFPRE) {
    if (tmw != TMW_NONE) {
      fft4096_split_tm(v, t, sm, sync, tmw);
      return;
    }
  }
  constexpr int b = fft_first_radix(M);
  constexpr int a = (ilog2c(M) - ilog2c(b)) / 4;
  constexpr int off = 2 * fft_stage_ns<M>(0);
  if constexpr (b > 1) fft_stage_split<M, b, 1>(v, t, sm, tw, sync);
  constexpr int NS1 = b;
  if constexpr (a == 2) {
    // tmw (M >= 256 with b == 1 only): stage NS = 16 at tmw, nothing else twiddled
    fft_stage_split<M, 16, NS1>(v, t, sm, tw, sync, stw, b == 1 ? TMW_NONE : tmw);
    fft_stage<M, 16, NS1 * 16, true>(v, t, nullptr, tw, stw ? stw + off : nullptr,
                                     tmw == TMW_NONE ? TMW_NONE : tmw + (b == 1 ? 0 : 64));
  } else {
    static_assert(a == 3, "M <= 4096");
    // tmw: the two twiddled stages (NS = 16 b, 256 b) read their per-thread
    // twiddles from tensor memory columns tmw + 0 and tmw + 64
    fft_stage_split<M, 16, NS1>(v, t, sm, tw, sync);
    fft_stage_split<M, 16, NS1 * 16>(v, t, sm, tw, sync, stw, tmw);
    fft_stage<M, 16, NS1 * 256, true>(v, t, nullptr, tw, stw ? stw + off : nullptr,
                                      tmw == TMW_NONE ? TMW_NONE : tmw + 64);
  }
}

// Inverse (unnormalised) via conj(FFT(conj(x))).
template <int M, class Sync = CtaSync>
__device__ __forceinline__ void fft_inv(cplx (&v)[fft_e(M)], int t, double2* sm, const double2* __restrict__ tw,
                                        const Sync& sync = Sync(), uint32_t tmw = TMW_NONE) {
  constexpr int E = fft_e(M);
#pragma unroll
  for (int r = 0; r < E; ++r) v[r].y = -v[r].y;
  fft_fwd<M, Sync>(v, t, sm, tw, sync, nullptr, tmw);
#pragma unroll
  for (int r = 0; r < E; ++r) v[r].y = -v[r].y;
}

}  // namespace ttagg
