// B200-native RHS evaluator for the multi-particle Smoluchowski equations.
//
// Gain P^(d) (rhs.py:234-302 TT, rhs.py:345-391 CP) is an fp64 FFT
// convolution of length L = d*Np (alias-free since L >= d*N - d + 1, SURVEY
// §7), evaluated as a four-step transform L = (d*N1) x N2 over the size
// index viewed as o = n1*N2 + n2:
//
//   pass A  (per column pair, per n2): the column transform over n1 — a
//           length-d*N1 DFT with only N1 nonzero inputs, done as d twisted
//           length-N1 FFTs ("residues"); two real columns ride in one
//           complex FFT and are separated through the Hermitian mirror;
//           only a half set of rows is kept; rows are twiddled by
//           W_L^(n2*kappa) and written to the exchange buffer T.  The
//           column sums needed by the loss (<F[:,r], n>) fall out of the
//           same read.
//   pass B  (per block of 8 rows kappa, streaming over all columns): the
//           length-N2 row FFTs, then the per-frequency product over modes
//           and sum over ranks (CP) or the spectral matrix chain (TT); then
//           the (d-1)-position shift, the inverse row FFT and the inverse
//           twiddle, written to U.
//   pass C  (per n2): the inverse column transform, pruned to the N1
//           outputs that land on sizes 1..N, scaled by 1/(L d!).
//
// Loss Q^(d) (rhs.py:305-338, 394-414): qcoef reduces the pass-A column
// sums to the per-rank scalars (CP) / contracted chain (TT); the combine
// kernel applies the tail GEMV, adds all orders and writes p, q, s (or the
// fused RK2 stage update, integrator.py:153-157).
//
// Data layout in HBM: every length-N vector of the hot loop lives in the
// "perm" layout (element o = n1*N2 + n2 at n2*N1 + n1), so pass A reads each
// column with unit stride; factor columns / TT fibers are stored once, at
// upload, in that layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fft.cuh"
#include "ttagg_b200.h"

using namespace ttagg;

namespace {

constexpr int MAXD = 8;
constexpr int MAXRES = MAXD;  // one residue class per order
constexpr int MAXORD = 8;
constexpr int LSPLIT = 11;
constexpr int LLO = 1 << LSPLIT;
#ifndef TTAGG_RB
#define TTAGG_RB 8
#endif
// residue row blocks are padded to multiples of RB rows (8 x 16 B: every n2 row of the
// exchange starts on a 128-byte line, so pass B's 8-row warp loads are whole lines)
constexpr int RB = TTAGG_RB;

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(TTAGG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(x)            \
  do {                    \
    int rc_ = (x);        \
    if (rc_) return rc_;  \
  } while (0)

struct Geom {
  int64_t N = 0, Np = 0;
  int N1 = 0, N2 = 0;
};

int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

int make_geom(int64_t N, Geom* g) {
  if (N < 2) return fail(TTAGG_ERR_ARG, "concentration state must be a vector of length >= 2");
  int64_t Np = std::max<int64_t>(64, next_pow2(N));
  // N = N1 x N2 with N2 <= 256 = 16^2 (row transforms: two radix-16 stages,
  // 16 threads per row, warp-resident) and N1 <= 4096 = 16^3
  int64_t N1 = std::max<int64_t>(4, Np / 256);
  if (N1 > 4096)
    return fail(TTAGG_ERR_UNSUPPORTED, "N = " + std::to_string(N) + " exceeds the supported 2^20 size classes");
  g->N = N;
  g->Np = Np;
  g->N1 = (int)N1;
  g->N2 = (int)(Np / N1);
  return TTAGG_OK;
}

// ---------------------------------------------------------------------------
// per-order transform plan (tables live in device memory)
// ---------------------------------------------------------------------------
struct OrderPlan {
  int d = 0;
  Geom g;
  int64_t L = 0;  // d * Np
  int K = 0;      // d * N1
  int nres = 0;
  int res_base[MAXRES] = {0};
  int res_cnt[MAXRES] = {0};
  int K_rows = 0;
  double2* tabK = nullptr;    // W_K^m, m < K
  double2* tabLlo = nullptr;  // W_L^m, m < 2048
  double2* tabLhi = nullptr;  // W_L^(m*2048), m < ceil(L/2048)
  int* rowkappa = nullptr;    // kappa of every exchange row (-1: pad)
};

void host_twiddles(std::vector<double2>& out, int64_t L, int64_t count, int64_t stride) {
  // W_L^(m*stride) = exp(-2 pi i m stride / L), long double then rounded
  out.resize(count);
  const long double twopi = 6.283185307179586476925286766559005768L;
  for (int64_t m = 0; m < count; ++m) {
    int64_t e = (m * stride) % L;
    long double ang = twopi * (long double)e / (long double)L;
    out[m] = make_double2((double)cosl(ang), (double)(-sinl(ang)));
  }
}

}  // namespace

struct ttagg_ctx {
  int device = 0;
  std::mutex mu;
  double2* tw4096 = nullptr;
  std::map<std::pair<int, int64_t>, OrderPlan*> plans;
  // workspaces: one per order slot of a kernel set (exchange T, inverse rows U,
  // TT chain scratch), so the orders' passes can run concurrently
  struct Work {
    double2* T = nullptr;
    size_t T_bytes = 0;
    double2* U = nullptr;
    size_t U_bytes = 0;
    double2* scratch = nullptr;
    size_t scratch_bytes = 0;
  } work[MAXORD];
  static constexpr int NFILL = 3;  // cheaper orders' pass B/C, one stream each (least priority)
  cudaStream_t s_main = nullptr, s_fill[NFILL] = {nullptr, nullptr, nullptr};  // mid / least priority
  cudaEvent_t ev_fork = nullptr, ev_a = nullptr, ev_fill[NFILL] = {nullptr, nullptr, nullptr};
  int num_sms = 0;
  double* pbuf = nullptr;
  size_t pbuf_bytes = 0;
  double* vec = nullptr;  // general vectors (natural/perm state, outputs)
  size_t vec_bytes = 0;
  double* diagp = nullptr;  // per-block diag partials
  size_t diagp_bytes = 0;
  double* diag = nullptr;  // 2 x 8 finalized diag
  int64_t* book = nullptr; // device step bookkeeping
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Rec { int cls, d; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  double prof_acc[5] = {0, 0, 0, 0, 0};
  long long launches = 0;  // kernel launches issued by this context
  bool poison = false;     // debug: NaN-fill every scratch buffer before use
  // the workspaces above are shared by every call: the GPU work of a call
  // issued on one stream waits for the previous call's (on any other stream)
  cudaEvent_t ev_last = nullptr;
  cudaStream_t last_stream = nullptr;
  bool last_valid = false;
  // page-locked staging for host-pointer calls whose buffers are pageable
  double* pin = nullptr;
  size_t pin_bytes = 0;
};

struct ttagg_kernel {
  ttagg_ctx* ctx = nullptr;
  int kind = 0, d = 0;
  int64_t N = 0;
  Geom g;
  int C = 0, C_pad = 0;
  double* X = nullptr;   // column pairs interleaved: pair p, element e -> double2 at X[(p Np + e) 2]
  double* Xt = nullptr;  // tail columns (the loss's last factor), one per row: [ntail][Np]
  int R = 0;            // CP: local ranks
  int ranks[MAXD + 1] = {0};
  int core_off[MAXD + 1] = {0};
  int Rmax = 0;
  int ntail = 0;
  int* tail_cols = nullptr;
  int nblk = 0;  // pass-A blocks per column (dot partials)
  double* V = nullptr;     // dense: N^d coefficients, row-major (natural sizes)
  double* nat = nullptr;   // dense: the state in natural order (scratch, N)
  double* part = nullptr;  // dense: loss partial sums [chunks][N]
  int chunks = 0;          // dense: loss chunks over the first d-1 modes
  int* fdesc = nullptr;  // TT: descriptors of the uploaded (live) fibers
  int* cidx = nullptr;   // TT: full fiber index -> uploaded column or -1
  int C_full = 0;        // TT: fibers before dropping
  int live_cols = 0;     // TT: uploaded live fibers (C less the no-op alignment slots)
  double* dots = nullptr;
  double* coef = nullptr;
  OrderPlan* plan = nullptr;
  // column pairs stored in X (pass A transforms these); without deduplication
  // xpairs = C_pad / 2 and pair p lives at p.  Deduplicated CP uploads store
  // each distinct (ordered) pair of columns once: pmap[p] is the stored pair
  // of original pair p, dslot[c] the column-sum slot of original column c.
  int xpairs = 0;
  int* pmap = nullptr;
  int* dslot = nullptr;
};

namespace {

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ cplx twL(const double2* __restrict__ lo, const double2* __restrict__ hi, long long m) {
  return cmul(ld_c(hi + (m >> LSPLIT)), ld_c(lo + (m & (LLO - 1))));
}

// state value at perm index e: n + alpha*k rounded as numpy does (no fma)
__device__ __forceinline__ double state_at(const double* __restrict__ nv, const double* __restrict__ kv, double alpha,
                                           size_t e) {
  double w = __ldg(nv + e);
  if (kv) w = __dadd_rn(w, __dmul_rn(alpha, __ldg(kv + e)));
  return w;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// pass A: column transforms (+ column sums for the loss)
// ---------------------------------------------------------------------------
struct PassAArgs {
  const double* X;
  const double* nv;
  const double* kv;
  double alpha;
  double2* T;
  double* dots;
  const double2* tw;
  const double2* tabK;
  const double2* tabLlo;
  const double2* tabLhi;
  int d, N2, K_rows, nblk, want_T;
  int pair0;  // first column pair of this launch (pass-A chunk)
  int raw;    // exchange rows leave without the four-step twiddle (pass B applies it; raw_exchange())
  int res_base[MAXRES], res_cnt[MAXRES];
};

// Emit one column-transform output of the packed pair z = a + i b
// (Y = Zcol[kappa], kappa = j + d k1, w = W_L^(n2 kappa)) into the exchange:
//   P plane, row kappa (kappa <= K/2):      Y w
//   M plane, row kappa' = K - kappa (kappa >= K/2, or kappa = 0):
//       conj(Y w) W_L^(n2 K)  (= conj(Zcol[K-kappa']) W_L^(n2 kappa'); kappa = 0: conj(Y))
// Pass B's row FFT of M_kappa' yields conj(Z[-k]) at the same frequencies as
// the P row, so the two real columns are separated in pass B's registers.
struct PMOut {
  double2* TP;  // P plane of this pair at this n2 (+ rho)
  double2* TM;  // M plane
  cplx cn2;     // W_L^(n2 K) = W_N2^(n2)
};

#ifndef TTAGG_A_TBPRE
#define TTAGG_A_TBPRE 1
#endif
#ifndef TTAGG_A_TMEMTW
#define TTAGG_A_TMEMTW 1
#endif
#ifndef TTAGG_B_JOINT
#define TTAGG_B_JOINT 1
#endif
__device__ __forceinline__ void emit_pm(const PassAArgs& a, const PMOut& o, int N1, int d, int j, int k1, cplx Y,
                                        cplx w) {
  const cplx Yw = cmul(Y, w);
  const cplx Mv = cmul(cconj(Yw), o.cn2);
  if (k1 < a.res_cnt[j]) sts_c(o.TP + a.res_base[j] + k1, Yw);
  if (j == 0) {
    if (k1 == 0) {
      sts_c(o.TM + a.res_base[0], cconj(Y));
    } else if (2 * k1 >= N1) {
      sts_c(o.TM + a.res_base[0] + (N1 - k1), Mv);
    }
  } else if (2 * k1 >= N1) {
    sts_c(o.TM + a.res_base[d - j] + (N1 - 1 - k1), Mv);
  }
}

// emit_pm with the plane known per register (block transforms, E = 16): the
// outputs k1 = t + T r with r < 8 (k1 < N1/2) are P rows only, r >= 8 M rows
// only, except k1 = 0 (also M, as conj(Y)) and, for residue 0, k1 = N1/2
// (also P) — both held by thread 0.  The M value is formed as conj(Y) times
// conj(w) cn2 = conj(b) PMst[r] (PMst[r] = conj(Pst[r]) cn2): two complex
// multiplies per output instead of three.  Assumes res_cnt[0] = N1/2 + 1 and
// res_cnt[j>0] = N1/2 (checked on the host).
// rbase: the residues' first exchange rows (res_base, staged in shared memory
// by the caller: a dynamically indexed kernel-parameter array costs constant-
// cache round trips)
template <int N1>
__device__ __forceinline__ void emit_split(const int* rbase, const PMOut& o, int d, int j, int t, const cplx (&v)[16],
                                           cplx b, const double2* Pst, const double2* PMst) {
  constexpr int T = N1 / 16;
  double2* TP = o.TP + rbase[j];
#pragma unroll
  for (int r = 0; r < 8; ++r) sts_c(TP + t + T * r, cmul(v[r], cmul(b, lds_c(Pst + r))));
  const cplx bc = cconj(b);
  double2* TM = j == 0 ? o.TM + rbase[0] + N1 - t : o.TM + rbase[d - j] + (N1 - 1 - t);
#pragma unroll
  for (int r = 8; r < 16; ++r) sts_c(TM - T * r, cmul(cconj(v[r]), cmul(bc, lds_c(PMst + r))));
  if (t == 0 && j == 0) {
    sts_c(o.TM + rbase[0], cconj(v[0]));
    sts_c(TP + T * 8, cmul(v[8], cmul(b, lds_c(Pst + 8))));
  }
}

#ifndef TTAGG_EMIT_CS
#define TTAGG_EMIT_CS 1
#endif
#if TTAGG_EMIT_CS
#define EMIT_ST stg_cs
#else
#define EMIT_ST sts_c
#endif
// emit_split for a raw exchange (raw_exchange()): the four-step twiddle
// W_L^(n2 kappa) is the same for the P row kappa and the M row kappa (see
// emit_pm), depends on (row, n2) only and not on the column pair, so pass B
// applies it from per-thread constants and pass A stores Y resp. conj(Y).
template <int N1>
__device__ __forceinline__ void emit_raw(const int* rbase, const PMOut& o, int d, int j, int t, const cplx (&v)[16]) {
  constexpr int T = N1 / 16;
  double2* TP = o.TP + rbase[j];
#pragma unroll
  for (int r = 0; r < 8; ++r) EMIT_ST(TP + t + T * r, v[r]);
  double2* TM = j == 0 ? o.TM + rbase[0] + N1 - t : o.TM + rbase[d - j] + (N1 - 1 - t);
#pragma unroll
  for (int r = 8; r < 16; ++r) EMIT_ST(TM - T * r, cconj(v[r]));
  if (t == 0 && j == 0) {
    EMIT_ST(o.TM + rbase[0], cconj(v[0]));
    EMIT_ST(TP + T * 8, v[8]);
  }
}

// Small column transforms (T < 32 threads per column): one CTA = one column
// pair x G adjacent columns; residues transformed in sequence.
template <int N1>
__global__ void __launch_bounds__(256) passA_kernel(const PassAArgs a) {
  constexpr int E = fft_e(N1), T = fft_t(N1), SE = fft_smem_elems(N1);
  extern __shared__ double2 smem[];
  __shared__ double red[2][256];
  const int G = blockDim.x / T;
  const int tid = threadIdx.x, g = tid / T, t = tid - g * T;
  const int n2 = blockIdx.x * G + g;
  const int pair = a.pair0 + blockIdx.y;
  const int d = a.d;
  const size_t Np = (size_t)N1 * a.N2;
  double2* zbuf = smem;
  double2* exch = smem + G * N1 + g * SE;
  const double2* zc = zbuf + g * N1;
  {
    const size_t e0 = (size_t)blockIdx.x * G * N1;
    const double2* xp = reinterpret_cast<const double2*>(a.X) + (size_t)pair * Np + e0;
    double sa = 0.0, sb = 0.0;
    for (int i = tid; i < G * N1; i += blockDim.x) {
      const double w = state_at(a.nv, a.kv, a.alpha, e0 + i);
      const double2 x = __ldg(xp + i);
      const double va = x.x * w, vb = x.y * w;
      zbuf[i] = make_double2(va, vb);
      sa += va;
      sb += vb;
    }
    red[0][tid] = sa;
    red[1][tid] = sb;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (tid < w && tid + w < (int)blockDim.x) {
        red[0][tid] += red[0][tid + w];
        red[1][tid] += red[1][tid + w];
      }
      __syncthreads();
    }
    if (tid == 0) {
      a.dots[(size_t)(2 * pair) * a.nblk + blockIdx.x] = red[0][0];
      a.dots[(size_t)(2 * pair + 1) * a.nblk + blockIdx.x] = red[1][0];
    }
  }
  if (!a.want_T) return;
  const size_t plane = (size_t)a.K_rows * a.N2;
  PMOut o;
  o.TP = a.T + (size_t)pair * 2 * plane + (size_t)n2 * a.K_rows;
  o.TM = o.TP + plane;
  o.cn2 = twL(a.tabLlo, a.tabLhi, (long long)n2 * (d * N1));
  for (int j = 0; j < d; ++j) {
    cplx v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int n1 = t + T * r;
      v[r] = cmul(lds_c(zc + n1), ld_c(a.tabK + j * n1));
    }
    fft_fwd<N1>(v, t, exch, a.tw);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int k1 = t + T * r;
      emit_pm(a, o, N1, d, j, k1, v[r], twL(a.tabLlo, a.tabLhi, (long long)n2 * (j + d * k1)));
    }
  }
}


// Pass A for column transforms of >= 32 threads (N1 >= 512): one CTA (one
// thread group, T threads) = one work item (column pair, n2), 70 KB of shared
// memory, two CTAs per SM so one CTA's memory phases overlap the other's
// FFTs.  The weighted input z = (a + i b) n is re-read from L2 for every
// residue (first touch from DRAM); outputs leave as P/M exchange rows.
template <int N1>
__global__ void __launch_bounds__(fft_t(N1), 2) passA_big_kernel(const PassAArgs a) {
  constexpr int E = fft_e(N1), T = fft_t(N1), SE = fft_smem_elems(N1);
  constexpr int NW = T / 32;
  static_assert(T >= 32, "warp-multiple groups");
  extern __shared__ double2 smem[];
  __shared__ double red[2][NW];
  __shared__ double2 Pst[16];
  __shared__ double2 Kst[MAXRES][16];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int d = a.d;
  const int N2 = a.N2;
  const int K = d * N1;
  const int item = blockIdx.x;
  const int pair = a.pair0 + item / N2, n2 = item % N2;
  const size_t Np = (size_t)N1 * N2;
  const size_t e0 = (size_t)n2 * N1;
  const double2* xp = reinterpret_cast<const double2*>(a.X) + (size_t)pair * Np + e0;
  const double* nv = a.nv + e0;
  const double* kv = a.kv ? a.kv + e0 : nullptr;
  double2* exch = smem;
  for (int i = t; i < d * 16; i += T) {
    const int j = i / 16, r = i % 16;
    const cplx w = ld_c(a.tabK + (j * T * r) % K);
    Kst[j][r] = make_double2(w.x, w.y);
  }
  if (t < 16) {
    const cplx w = twL(a.tabLlo, a.tabLhi, (long long)n2 * d * T * t);
    Pst[t] = make_double2(w.x, w.y);
  }
  const size_t plane = (size_t)a.K_rows * N2;
  PMOut o;
  o.TP = a.T + (size_t)pair * 2 * plane + (size_t)n2 * a.K_rows;
  o.TM = o.TP + plane;
  o.cn2 = twL(a.tabLlo, a.tabLhi, (long long)n2 * K);
  // z in the FFT's register layout (element t + T r)
  auto load_z = [&](cplx (&z)[E]) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int n1 = t + T * r;
      double w = __ldg(nv + n1);
      if (kv) w = __dadd_rn(w, __dmul_rn(a.alpha, __ldg(kv + n1)));
      const double2 x = __ldg(xp + n1);
      z[r] = mk(x.x * w, x.y * w);
    }
  };
  {
    cplx z[E];
    load_z(z);
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      sa += z[r].x;
      sb += z[r].y;
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      red[0][wid] = sa;
      red[1][wid] = sb;
    }
    __syncthreads();
    if (t == 0) {
      double ta = 0.0, tb = 0.0;
      for (int w = 0; w < NW; ++w) {
        ta += red[0][w];
        tb += red[1][w];
      }
      a.dots[(size_t)(2 * pair) * a.nblk + n2] = ta;
      a.dots[(size_t)(2 * pair + 1) * a.nblk + n2] = tb;
    }
    if (!a.want_T) return;
    // residue 0 straight from these registers
    fft_fwd<N1>(z, t, exch, a.tw);
    const cplx b = twL(a.tabLlo, a.tabLhi, (long long)n2 * (d * t));
#pragma unroll
    for (int r = 0; r < E; ++r) emit_pm(a, o, N1, d, 0, t + T * r, z[r], cmul(b, lds_c(Pst + r)));
  }
  for (int j = 1; j < d; ++j) {
    cplx v[E];
    load_z(v);
    const cplx tb = ld_c(a.tabK + j * t);
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = cmul(v[r], cmul(tb, lds_c(&Kst[j][r])));
    fft_fwd<N1>(v, t, exch, a.tw);
    const cplx b = twL(a.tabLlo, a.tabLhi, (long long)n2 * (j + d * t));
#pragma unroll
    for (int r = 0; r < E; ++r) emit_pm(a, o, N1, d, j, t + T * r, v[r], cmul(b, lds_c(Pst + r)));
  }
}

// ---- bulk-copy (TMA) and mbarrier helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on mbarrier m
#ifndef TTAGG_L2_HINT
#define TTAGG_L2_HINT 1
#endif
// L2 policy for data read exactly once per RHS (pass A's factor-column rows: -0.03 ms on A5; the same hint on
// pass B's exchange reads measured +0.05 ms and is not used)
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
#if TTAGG_L2_HINT
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m)), "l"(l2_evict_first())
      : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TTAGG_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TTAGG_WAIT_%=;\n}" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}

// Pass A, TMA-fed (N1 >= 1024): persistent CTAs (two per SM) walk the work
// items (column pair, n2).  The pair's raw row x = (a, b) (N1 x 16 B,
// contiguous in the perm layout) arrives in shared memory by one bulk copy
// issued while the previous item's last residue is still transforming; the
// weighted input z = x n is formed in place once per item (the loss column
// sums fall out of that pass) and every residue reads it from shared memory
// instead of re-reading the columns through L1/L2.  To fit z (N1 x 16 B) and
// the transform's exchange in two CTAs per SM, exchanges go through a
// half-size buffer in two rounds (fft_fwd_split).
// stage twiddles in tensor memory: CTAs of 4 or 8 warps (N1 = 2048, 4096); the
// column budget (512 per SM) holds for their 4 resp. 2 resident CTAs
__host__ __device__ constexpr bool passA_tmem_twiddles(int N1) { return TTAGG_A_TMEMTW && fft_t(N1) >= 128; }
__host__ __device__ constexpr unsigned passA_tmem_cols(int N1) { return fft_t(N1) >= 256 ? 256u : 128u; }

// resident CTAs per SM the register budget is sized for: 16 warps per SM
#ifndef TTAGG_A_WARPS
#define TTAGG_A_WARPS 16
#endif
__host__ __device__ constexpr int passA_min_ctas(int N1) {
  return fft_t(N1) >= 256 ? 2 : (TTAGG_A_WARPS * 32) / fft_t(N1);
}

template <int N1, bool RAW>
__global__ void __launch_bounds__(fft_t(N1), passA_min_ctas(N1)) passA_tma_kernel(const PassAArgs a, int nitems) {
  constexpr int E = fft_e(N1), T = fft_t(N1);
  constexpr int NW = T / 32;
  constexpr unsigned ROW_BYTES = N1 * sizeof(double2);
  constexpr int NCHUNK = ROW_BYTES > 32768 ? ROW_BYTES / 32768 : 1;
  static_assert(T >= 64, "block transforms");
  extern __shared__ __align__(128) double2 smem[];
  double2* zs = smem;                                  // N1 slots: the item's x, then z
  double* ex = reinterpret_cast<double*>(smem + N1);  // fft_smem_elems(N1) doubles
  double2* stw = reinterpret_cast<double2*>(ex + ((fft_smem_elems(N1) + 1) & ~1));  // stage twiddles
  __shared__ double red[2][NW];
  __shared__ double2 Pst[2][16], PMst[2][16];
  __shared__ double2 Ust[2][MAXRES];
  __shared__ double2 Kst[MAXRES][16];
  __shared__ int rbase[MAXRES];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tm_base;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int d = a.d;
  const int N2 = a.N2;
  const int K = d * N1;
  const size_t Np = (size_t)N1 * N2;
  const double2* X2 = reinterpret_cast<const double2*>(a.X);
  for (int i = t; i < d * 16; i += T) {
    const int j = i / 16, r = i % 16;
    const cplx w = ld_c(a.tabK + (j * T * r) % K);
    Kst[j][r] = make_double2(w.x, w.y);
  }
  if (t < MAXRES) rbase[t] = a.res_base[t];
  // Stage twiddles: the 15 powers a thread needs in each of the two twiddled
  // radix-16 stages never change, so CTAs of >= 4 warps park them in tensor
  // memory once (128 columns per thread: 64 per stage; warps w and w + 4
  // share a lane quadrant and take different column halves) and every
  // transform reads them back (tcgen05.ld) instead of rebuilding them from
  // two table values; smaller CTAs keep the shared stage table.
  uint32_t tmw = TMW_NONE;
  if constexpr (passA_tmem_twiddles(N1)) {
    constexpr unsigned TCOLS = passA_tmem_cols(N1);
    if (wid == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm_base)),
                   "n"(TCOLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmw = tm_base + ((uint32_t)(32 * (wid & 3)) << 16) + 128u * (uint32_t)(wid >> 2);
    constexpr int NSa = fft_stage_ns<N1>(0), NSb = fft_stage_ns<N1>(1);
    tmem_store_twiddles16(tmw, a.tw, (t & (NSa - 1)) * (TW_BASE / (NSa * 16)));
    tmem_store_twiddles16(tmw + 64, a.tw, (t & (NSb - 1)) * (TW_BASE / (NSb * 16)));
  } else {
    fft_stage_table<N1>(stw, a.tw, t, T);
  }
  auto issue = [&](int it) {  // one thread: bulk-copy item it's row into zs
    const int pair = a.pair0 + it / N2, n2 = it % N2;
    const double2* src = X2 + (size_t)pair * Np + (size_t)n2 * N1;
    fence_proxy_async();
    mbar_expect_tx(&mbar, ROW_BYTES);
#pragma unroll
    for (int c = 0; c < NCHUNK; ++c)
      bulk_g2s(zs + c * (N1 / NCHUNK), src + c * (N1 / NCHUNK), ROW_BYTES / NCHUNK, &mbar);
  };
  if (t == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && (int)blockIdx.x < nitems) issue(blockIdx.x);
  unsigned parity = 0;
  const size_t plane = (size_t)a.K_rows * N2;
  for (int item = blockIdx.x, it_n = 0; item < nitems; item += gridDim.x, ++it_n) {
    const int pair = a.pair0 + item / N2, n2 = item % N2;
    const size_t e0 = (size_t)n2 * N1;
    const double* nv = a.nv + e0;
    const double* kv = a.kv ? a.kv + e0 : nullptr;
    const int pb = it_n & 1;
    PMOut o;
    o.TP = a.T + (size_t)pair * 2 * plane + (size_t)n2 * a.K_rows;
    o.TM = o.TP + plane;
    cplx ct = mk(1.0, 0.0);
    if constexpr (!RAW) {
      if (t < 16) {
        const cplx w = twL(a.tabLlo, a.tabLhi, (long long)n2 * d * T * t);
        Pst[pb][t] = make_double2(w.x, w.y);
      } else if (t < 16 + d) {
        const cplx w = twL(a.tabLlo, a.tabLhi, (long long)n2 * (t - 16));
        Ust[pb][t - 16] = make_double2(w.x, w.y);
      }
      // emit twiddle W_L^(n2 (j + d t)) = W_L^(n2 d t) W_L^(n2 j)
      ct = twL(a.tabLlo, a.tabLhi, (long long)n2 * (d * t));
      o.cn2 = twL(a.tabLlo, a.tabLhi, (long long)n2 * K);
      if (t >= 32 && t < 48) {
        const cplx w = twL(a.tabLlo, a.tabLhi, (long long)n2 * d * T * (t - 32));
        const cplx pm = cmul(cconj(w), o.cn2);
        PMst[pb][t - 32] = make_double2(pm.x, pm.y);
      }
    }
    // the state weights of this n2 row (through L1; shared by every pair)
    double wv[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int n1 = t + T * r;
      double w = __ldg(nv + n1);
      if (kv) w = __dadd_rn(w, __dmul_rn(a.alpha, __ldg(kv + n1)));
      wv[r] = w;
    }
    mbar_wait(&mbar, parity);
    parity ^= 1;
    cplx z[E];
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int n1 = t + T * r;
      const double2 x = zs[n1];
      z[r] = mk(x.x * wv[r], x.y * wv[r]);
      zs[n1] = make_double2(z[r].x, z[r].y);
      sa += z[r].x;
      sb += z[r].y;
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      red[0][wid] = sa;
      red[1][wid] = sb;
    }
    __syncthreads();  // z complete in zs, red and Pst[pb] visible
    if (t == 0) {
      double ta = 0.0, tb = 0.0;
      for (int w = 0; w < NW; ++w) {
        ta += red[0][w];
        tb += red[1][w];
      }
      a.dots[(size_t)(2 * pair) * a.nblk + n2] = ta;
      a.dots[(size_t)(2 * pair + 1) * a.nblk + n2] = tb;
    }
    const int next = item + gridDim.x;
    if (!a.want_T) {
      __syncthreads();  // every thread is done with zs (and red)
      if (t == 0 && next < nitems) issue(next);
      continue;
    }
    // residue 0 straight from the registers
    fft_fwd_split<N1>(z, t, ex, a.tw, CtaSync(), stw, tmw);
    if constexpr (RAW) emit_raw<N1>(rbase, o, d, 0, t, z);
    else emit_split<N1>(rbase, o, d, 0, t, z, ct, Pst[pb], PMst[pb]);
#if TTAGG_A_TBPRE
    cplx tbn = ld_c(a.tabK + t);  // residue 1's per-thread twist, requested a transform ahead
#endif
    for (int j = 1; j < d; ++j) {
      cplx v[E];
#if TTAGG_A_TBPRE
      const cplx tb = tbn;
      if (j + 1 < d) tbn = ld_c(a.tabK + (j + 1) * t);
#else
      const cplx tb = ld_c(a.tabK + j * t);
#endif
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = cmul(lds_c(zs + t + T * r), cmul(tb, lds_c(&Kst[j][r])));
      if (j == d - 1) {
        __syncthreads();  // zs free: the next item's row can land while this residue transforms
        if (t == 0 && next < nitems) issue(next);
      }
      fft_fwd_split<N1>(v, t, ex, a.tw, CtaSync(), stw, tmw);
      if constexpr (RAW) emit_raw<N1>(rbase, o, d, j, t, v);
      else emit_split<N1>(rbase, o, d, j, t, v, cmul(ct, lds_c(&Ust[pb][j])), Pst[pb], PMst[pb]);
    }
  }
  if constexpr (passA_tmem_twiddles(N1)) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(passA_tmem_cols(N1))
                   : "memory");
  }
}

// (tensor-memory helpers tmem_st16 / tmem_ld16 live in fft.cuh)
// ---------------------------------------------------------------------------
// pass B: row FFTs, spectral product / chain, inverse row FFTs
// ---------------------------------------------------------------------------
struct PassBArgs {
  const double2* T;
  double2* U;
  const double2* tw;
  const double2* tabLlo;
  const double2* tabLhi;
  const int* rowkappa;
  double2* scratch;
  long long L;
  int d, K, K_rows, C, kind, Rmax;
  int p0, p1;        // column pairs of this launch
  int nrb;           // row blocks (CTAs loop over them)
  int ranks[MAXD + 1];
  const int* fdesc;  // TT: per uploaded fiber, packed (core, rn, rp, first, last, noop)
  const int* pmap;   // deduplicated CP: stored exchange pair of each pair (null: identity)
  int raw;           // the exchange holds untwiddled column outputs: multiply by W_L^(n2 kappa) here
};

// TT fiber descriptor: the uploaded columns are the live fibers only (all-zero
// fibers and fibers on a chain path that is zero are dropped at upload), in
// core-major, rn-major, rp-inner order; first/last mark the first and last
// live fiber that feeds chain state (core, rn).
constexpr int FD_FIRST = 1 << 20, FD_LAST = 1 << 21, FD_NOOP = 1 << 22;
// the column accumulates into the chain's second accumulator (tensor memory):
// cores with several output states pair their fibers by output state (rn, rn+1)
// at the same input state rp, so both halves of a pair read one chain state
constexpr int FD_ACC1 = 1 << 23;
__host__ __device__ constexpr int fd_pack(int lam, int rn, int rp, bool first, bool last) {
  return lam | (rn << 4) | (rp << 12) | (first ? FD_FIRST : 0) | (last ? FD_LAST : 0);
}
__device__ __forceinline__ int fd_lam(int f) { return f & 15; }
__device__ __forceinline__ int fd_rn(int f) { return (f >> 4) & 255; }
__device__ __forceinline__ int fd_rp(int f) { return (f >> 12) & 255; }

// ---- per-thread asynchronous 16-byte copies (global -> shared), zero-fill when !ok
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA = 8 exchange rows x T threads per row (128 threads).  Lanes run
// over the 8 rows fastest so every warp load reads whole 128-byte segments
// of the P and M planes T[pair][plane][n2][rho]; the row transforms exchange
// through shared memory.  Per column pair: FFT(P row), FFT(M row), then the
// two real columns separate in registers: 2A = P + M, 2B = -i (P - M).
// The next pair's planes stream in with cp.async while this pair computes:
// every thread copies exactly the elements it later reads, into two staging
// regions that double as the row FFTs' exchange buffers (P stage for FFT(P),
// M stage for FFT(M)); a plane is re-armed as soon as its FFT has passed the
// transform's last barrier.
template <int N2, bool TT, bool TMA>
__global__ void __launch_bounds__(128) passB_kernel(const PassBArgs a, const __grid_constant__ CUtensorMap tmT) {
  constexpr int E = fft_e(N2), T = fft_t(N2), SE = fft_smem_elems(N2);
  constexpr int ROWS = 128 / T;
  constexpr int STG = (ROWS * SE > E * 128) ? ROWS * SE : E * 128;
  static_assert(!TMA || (N2 == 256 && ROWS == 8 && STG % 8 == 0), "TMA staging: 8 rows x 256, 128-byte aligned");
  extern __shared__ __align__(128) double2 smem[];
  __shared__ __align__(8) uint64_t mbar;  // TMA: both planes of the next pair landed
  __shared__ uint32_t tm_base;            // TT: the second chain accumulator (64 TMEM columns)
  unsigned parity = 0;
  // tensor memory: the TT chain's second accumulator (columns 0..63) and, with
  // a raw exchange (TMA kernels), the row's four-step twiddles (columns 64..127)
  constexpr bool TMEM = TT || TMA;
  constexpr unsigned TCOLS = TMA ? 128u : 64u;
  if constexpr (TMEM) {
    if ((threadIdx.x >> 5) == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm_base)),
                   "n"(TCOLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  const int tid = threadIdx.x;
  const int rl8 = tid & 7, t = (tid >> 3) % T, sub = (tid >> 3) / T;
  const int rloc = sub * 8 + rl8;
  double2* stP = smem;
  double2* stM = smem + STG;
  double2* Sb = smem + 2 * STG;  // CP rank sum, [k2][row] (conflict-free across the rows of a warp)
  const size_t plane = (size_t)a.K_rows * N2;
  const int d = a.d;
  const int C = a.C;
  // TT: per-CTA chain scratch (reused by every row block of this CTA)
  const size_t slot = (size_t)blockIdx.x * 2 * a.Rmax;
  const uint32_t tacc = TMEM ? tm_base + ((uint32_t)(32 * (tid >> 5)) << 16) : 0u;
  const uint32_t tfs = tacc + 64;
  auto st = [&](int b, int r, int i) -> double2* {
    return a.scratch + ((slot + (size_t)b * a.Rmax + r) * E + i) * blockDim.x + tid;
  };

  for (int rb = blockIdx.x; rb < a.nrb; rb += gridDim.x) {
    const int rho = rb * ROWS + rloc;
    const bool valid = rho < a.K_rows;
    const double2* Tb = a.T + (valid ? rho : 0);  // + pair*2*plane + {0, plane} + n2*K_rows
    auto xp = [&](int p) { return a.pmap ? __ldg(a.pmap + p) : p; };
    auto fetch = [&](double2* stage, int p, int pl) {
      const double2* src = Tb + ((size_t)xp(p) * 2 + pl) * plane;
#pragma unroll
      for (int i = 0; i < E; ++i) cp_async16(stage + i * 128 + tid, src + (size_t)(t + T * i) * a.K_rows, valid);
      cp_async_commit();
    };
    // TMA: one thread moves both planes of pair p (8 rows x 256 n2 x 16 B
    // each, the [n2][row] staging layout; rows past K_rows arrive as zeros)
    auto fetch_tma = [&](int p) {
      if (tid == 0) {
        fence_proxy_async();
        mbar_expect_tx(&mbar, 2u * ROWS * N2 * sizeof(double2));
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
          double2* dst = pl ? stM : stP;
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  smem_u32(dst)),
              "l"(&tmT), "r"(2 * rb * ROWS), "r"(0), "r"(2 * xp(p) + pl), "r"(smem_u32(&mbar))
              : "memory");
        }
      }
    };
    // CP: running product over the modes of one rank term.  TT: chain
    // accumulator of the current state (core, rn); the last group processed
    // is the last core's, so after the loop it holds the chain result.
    if constexpr (TMA) {
      if (a.raw) {  // this row's four-step twiddles W_L^(n2 kappa), n2 = t + T i (as passB_pipe_kernel)
        const int kap0 = valid ? max(a.rowkappa[rho], 0) : 0;
#pragma unroll
        for (int q = 0; q < E / 4; ++q) {
          uint32_t r[16];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const cplx w = twL(a.tabLlo, a.tabLhi, (long long)(t + T * (4 * q + u)) * kap0);
            r[4 * u + 0] = (uint32_t)__double2loint(w.x);
            r[4 * u + 1] = (uint32_t)__double2hiint(w.x);
            r[4 * u + 2] = (uint32_t)__double2loint(w.y);
            r[4 * u + 3] = (uint32_t)__double2hiint(w.y);
          }
          tmem_st16(tfs + 16 * q, r);
        }
        tmem_wait_st();
      }
    }
    cplx acc[E];
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = mk(0.0, 0.0);
    if constexpr (!TT) {
#pragma unroll
      for (int i = 0; i < E; ++i) Sb[(t + T * i) * ROWS + rloc] = make_double2(0.0, 0.0);
    }
    auto row_fft = [&](cplx (&v)[E], double2* stage) { fft_fwd<N2>(v, t, stage + rloc * SE, a.tw); };

    // TT: the chain state of the pair's first column is prefetched into the
    // (otherwise unused) rank-sum region Sb with cp.async before the row FFTs
    bool pre = false;
    auto process = [&](cplx (&X)[E], int c, bool from_sb) {
      if constexpr (!TT) {
        const int m = c % d;  // rank-major columns: c = r d + m
        if (m == 0) {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = X[i];
        } else {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = cmul(acc[i], X[i]);
        }
        if (m == d - 1) {
#pragma unroll
          for (int i = 0; i < E; ++i) {
            double2* sp = Sb + (t + T * i) * ROWS + rloc;
            sts_c(sp, cadd(lds_c(sp), acc[i]));
          }
        }
      } else {
        const int f = __ldg(a.fdesc + c);
        if (f & FD_NOOP) return;
        const int lam = fd_lam(f), rn = fd_rn(f), rp = fd_rp(f);
        if (lam == 0) {
#pragma unroll
          for (int i = 0; i < E; ++i) sts_c(st(0, rn, i), X[i]);
        } else if (f & FD_ACC1) {
          // second accumulator: four values at a time through tensor memory
          // (rn-paired cores are never the last core, so a finished state
          // always goes to the chain scratch)
#pragma unroll
          for (int q = 0; q < E / 4; ++q) {
            uint32_t r[16];
            if (!(f & FD_FIRST)) {
              tmem_ld16(tacc + 16 * q, r);
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = 4 * q + u;
              cplx v = (f & FD_FIRST) ? mk(0.0, 0.0)
                                      : mk(__hiloint2double((int)r[4 * u + 1], (int)r[4 * u]),
                                           __hiloint2double((int)r[4 * u + 3], (int)r[4 * u + 2]));
              v = cadd(v, cmul(from_sb ? lds_c(Sb + i * 128 + tid) : lds_c(st((lam - 1) & 1, rp, i)), X[i]));
              if (f & FD_LAST) {
                sts_c(st(lam & 1, rn, i), v);
              } else {
                r[4 * u + 0] = (uint32_t)__double2loint(v.x);
                r[4 * u + 1] = (uint32_t)__double2hiint(v.x);
                r[4 * u + 2] = (uint32_t)__double2loint(v.y);
                r[4 * u + 3] = (uint32_t)__double2hiint(v.y);
              }
            }
            if (!(f & FD_LAST)) tmem_st16(tacc + 16 * q, r);
          }
          if (!(f & FD_LAST)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else {
          if (f & FD_FIRST) {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = mk(0.0, 0.0);
          }
#pragma unroll
          for (int i = 0; i < E; ++i)
            acc[i] = cadd(acc[i], cmul(from_sb ? lds_c(Sb + i * 128 + tid) : lds_c(st((lam - 1) & 1, rp, i)), X[i]));
          if ((f & FD_LAST) && lam < d - 1) {
#pragma unroll
            for (int i = 0; i < E; ++i) sts_c(st(lam & 1, rn, i), acc[i]);
          }
        }
      }
    };

    if constexpr (TMA) {
      fetch_tma(a.p0);
    } else {
      fetch(stP, a.p0, 0);
      fetch(stM, a.p0, 1);
    }
    for (int p = a.p0; p < a.p1; ++p) {
      const bool more = p + 1 < a.p1;
      cplx vp[E], vm[E];
#if TTAGG_B_JOINT
      if constexpr (N2 == 256) {
        if constexpr (TMA) {
          mbar_wait(&mbar, parity);
          parity ^= 1;
        } else {
          cp_async_wait<0>();
        }
        bool twiddled = false;
        if constexpr (TMA) {
          if (a.raw) {
            twiddled = true;
#pragma unroll
            for (int q = 0; q < E / 4; ++q) {
              uint32_t r[16];
              tmem_ld16(tfs + 16 * q, r);
              tmem_wait_ld();
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = 4 * q + u;
                const cplx w = mk(__hiloint2double((int)r[4 * u + 1], (int)r[4 * u]),
                                  __hiloint2double((int)r[4 * u + 3], (int)r[4 * u + 2]));
                vp[i] = cmul(lds_c(stP + i * 128 + tid), w);
                vm[i] = cmul(lds_c(stM + i * 128 + tid), w);
              }
            }
          }
        }
        if (!twiddled) {
#pragma unroll
          for (int i = 0; i < E; ++i) {
            vp[i] = lds_c(stP + i * 128 + tid);
            vm[i] = lds_c(stM + i * 128 + tid);
          }
        }
        if constexpr (TT) {
          const int f = __ldg(a.fdesc + 2 * p);
          pre = !(f & FD_NOOP) && fd_lam(f) >= 1;
          if (pre) {  // state of column 2p: written (if at all) by earlier columns of this thread
            __threadfence_block();
#pragma unroll
            for (int i = 0; i < E; ++i) cp_async16(Sb + i * 128 + tid, st((fd_lam(f) - 1) & 1, fd_rp(f), i), true);
          }
          cp_async_commit();
        }
        __syncthreads();
        fft_fwd2<N2>(vp, vm, t, stP + rloc * SE, stM + rloc * SE, a.tw);
        if constexpr (TMA) {
          if (more) fetch_tma(p + 1);  // every thread is past the transforms' last barrier
          if constexpr (TT) cp_async_wait<0>();  // the state group
        } else {
          if (more) {
            fetch(stP, p + 1, 0);
            fetch(stM, p + 1, 1);
          } else {
            cp_async_commit();
            cp_async_commit();
          }
          if constexpr (TT) cp_async_wait<2>();  // the state group (P/M of p+1 may fly on)
        }
      } else
#endif
      {
      cp_async_wait<1>();  // P(p) landed (M(p) may still be in flight)
#pragma unroll
      for (int i = 0; i < E; ++i) vp[i] = lds_c(stP + i * 128 + tid);
      __syncthreads();  // every thread holds its P slots before the stage turns into exchange space
      row_fft(vp, stP);  // ends past its last barrier: stage free again
      if (more) fetch(stP, p + 1, 0); else cp_async_commit();
      cp_async_wait<1>();  // M(p) landed
#pragma unroll
      for (int i = 0; i < E; ++i) vm[i] = lds_c(stM + i * 128 + tid);
      __syncthreads();
      row_fft(vm, stM);
      if (more) fetch(stM, p + 1, 1); else cp_async_commit();
      }
#pragma unroll
      for (int i = 0; i < E; ++i) {
        // 2A = P + M, 2B = -i (P - M); the 2^d this leaves on every order-d
        // product is removed exactly in pass C's scale
        const cplx P = vp[i];
        vp[i] = cadd(P, vm[i]);
        vm[i] = mul_mi(csub(P, vm[i]));
      }
      bool pre1 = false;  // TT: the pair's second fiber reads the same (prefetched) chain state
      if constexpr (TT) {
        if (pre && 2 * p + 1 < C) {
          const int f0 = __ldg(a.fdesc + 2 * p), f1 = __ldg(a.fdesc + 2 * p + 1);
          pre1 = !(f1 & FD_NOOP) && fd_lam(f1) == fd_lam(f0) && fd_rp(f1) == fd_rp(f0);
        }
      }
      process(vp, 2 * p, pre);
      if (2 * p + 1 < C) process(vm, 2 * p + 1, pre1);
      pre = false;
    }
    cp_async_wait<0>();
    __syncthreads();
    cplx S[E];
#pragma unroll
    for (int i = 0; i < E; ++i) S[i] = TT ? acc[i] : lds_c(Sb + (t + T * i) * ROWS + rloc);

    // (d-1)-position shift (s'[t] = s[t-(d-1)] <=> S'[k] = S[k] W_L^{(d-1)k}), inverse row FFT, inverse twiddle, Hermitian weight
    const int kap = valid ? max(a.rowkappa[rho], 0) : 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const long long k = (long long)kap + (long long)a.K * (t + T * i);
      const long long m = ((long long)(d - 1) * k) % a.L;
      S[i] = cmul(S[i], twL(a.tabLlo, a.tabLhi, m));  // shift by d-1: * W_L^{+(d-1)k}
    }
    fft_inv<N2>(S, t, stP + rloc * SE, a.tw);
    const double wgt = (kap == 0 || 2 * kap == a.K) ? 1.0 : 2.0;
    if (valid) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int n2 = t + T * i;
        const cplx u = cscale(cmulc(S[i], twL(a.tabLlo, a.tabLhi, (long long)n2 * kap)), wgt);
        sts_c(a.U + (size_t)n2 * a.K_rows + rho, u);
      }
    }
  }
  if constexpr (TMEM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(TCOLS) : "memory");
  }
}

// Pass B for CP kernels with a full pair of prefetch window (N2 = 256, TMA).
// passB_kernel lands each pair's planes in the row FFTs' exchange buffers, so
// the next pair can only be requested once both transforms are done (about a
// quarter of a pair's compute ahead of its use).  Here the staging regions
// (P and M of one pair, 2 x 32 KB) are separate from the exchange buffer
// (one 8-row buffer, the two row FFTs run one after the other), and the rank
// sum lives in tensor memory (64 TMEM columns per CTA: thread = lane, its 16
// complex sums in its own columns) instead of shared memory, so two CTAs
// still fit per SM: as soon as every thread holds pair p in registers, pair
// p+1 is requested and streams in during the whole of pair p's transforms
// and products.  Same arithmetic in the same order as passB_kernel<256,
// false, true> (bitwise equal results).
constexpr int PIPE_STG = 8 * 256;                       // one plane of one row block (double2)
constexpr int PIPE_EX = 8 * fft_smem_elems(256);        // row FFT exchange (double2)
constexpr size_t PIPE_SMEM = (size_t)(2 * PIPE_STG + PIPE_EX) * sizeof(double2);

#ifndef TTAGG_B_TMEMTW
#define TTAGG_B_TMEMTW 1
#endif
constexpr unsigned PIPE_TCOLS = TTAGG_B_TMEMTW ? 256u : 128u;

template <bool RAW>
__global__ void __launch_bounds__(128, 2) passB_pipe_kernel(const PassBArgs a, const __grid_constant__ CUtensorMap tmT) {
  constexpr int N2 = 256, E = 16, T = 16, SE = fft_smem_elems(N2), ROWS = 8;
  extern __shared__ __align__(128) double2 smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tm_base;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm_base)), "n"(PIPE_TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int tid = threadIdx.x;
  const int rloc = tid & 7, t = tid >> 3;
  double2* stP = smem;
  double2* stM = smem + PIPE_STG;
  double2* ex = smem + 2 * PIPE_STG + rloc * SE;
  const uint32_t tsum = tm_base + ((uint32_t)(32 * (tid >> 5)) << 16);
  const uint32_t tfs = tsum + 64;  // raw exchange: this thread's four-step twiddles W_L^(n2 kappa), n2 = t + 16 i
  // the row transforms' stage twiddles W_256^(t i) (per thread, as in pass A)
  const uint32_t tmw = TTAGG_B_TMEMTW ? tsum + 128 : TMW_NONE;
  if (TTAGG_B_TMEMTW) tmem_store_twiddles16(tmw, a.tw, t * (TW_BASE / 256));
  const int d = a.d, C = a.C;
  unsigned parity = 0;
  auto fetch = [&](int rb, int p) {  // one thread: both planes of pair p of row block rb
    if (tid == 0) {
      const int xp = a.pmap ? __ldg(a.pmap + p) : p;
      fence_proxy_async();
      mbar_expect_tx(&mbar, 2u * ROWS * N2 * sizeof(double2));
#pragma unroll
      for (int pl = 0; pl < 2; ++pl)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(smem_u32(pl ? stM : stP)),
            "l"(&tmT), "r"(2 * rb * ROWS), "r"(0), "r"(2 * xp + pl), "r"(smem_u32(&mbar))
            : "memory");
    }
  };
  if (blockIdx.x < a.nrb && a.p0 < a.p1) fetch(blockIdx.x, a.p0);
  for (int rb = blockIdx.x; rb < a.nrb; rb += gridDim.x) {
    const int rho = rb * ROWS + rloc;
    const bool valid = rho < a.K_rows;
    const int kap = valid ? max(a.rowkappa[rho], 0) : 0;
    if constexpr (RAW) {
      // the row's four-step twiddles are the same for every pair: built once
      // per row block, parked in tensor memory (16 complex = 64 columns)
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        uint32_t r[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const cplx w = twL(a.tabLlo, a.tabLhi, (long long)(t + T * (4 * q + u)) * kap);
          r[4 * u + 0] = (uint32_t)__double2loint(w.x);
          r[4 * u + 1] = (uint32_t)__double2hiint(w.x);
          r[4 * u + 2] = (uint32_t)__double2loint(w.y);
          r[4 * u + 3] = (uint32_t)__double2hiint(w.y);
        }
        tmem_st16(tfs + 16 * q, r);
      }
      tmem_wait_st();
    }
    cplx acc[E];
    bool have_sum = false;  // the first finished rank term stores, later ones add
    for (int p = a.p0; p < a.p1; ++p) {
      cplx vp[E], vm[E];
      // raw exchange: the row's four-step twiddles come back from tensor memory
      // (two 4-value chunks in flight) while the pair's planes are still landing,
      // and multiply the values as they leave the staging regions
      uint32_t fs[2][16];
      if constexpr (RAW) {
        tmem_ld16(tfs, fs[0]);
        tmem_ld16(tfs + 16, fs[1]);
      }
      mbar_wait(&mbar, parity);
      parity ^= 1;
      if constexpr (RAW) {
#pragma unroll
        for (int q = 0; q < E / 4; ++q) {
          if (q == 0 || q == 2) tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = 4 * q + u;
            const cplx w = mk(__hiloint2double((int)fs[q & 1][4 * u + 1], (int)fs[q & 1][4 * u]),
                              __hiloint2double((int)fs[q & 1][4 * u + 3], (int)fs[q & 1][4 * u + 2]));
            vp[i] = cmul(lds_c(stP + i * 128 + tid), w);
            vm[i] = cmul(lds_c(stM + i * 128 + tid), w);
          }
          if (q < 2) tmem_ld16(tfs + 32 + 16 * q, fs[q]);  // chunk q + 2 follows into the buffer just used
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          vp[i] = lds_c(stP + i * 128 + tid);
          vm[i] = lds_c(stM + i * 128 + tid);
        }
      }
      __syncthreads();  // every thread holds pair p: the staging regions are free
      {
        const int nrb = rb + (int)gridDim.x;
        if (p + 1 < a.p1) fetch(rb, p + 1);
        else if (nrb < a.nrb) fetch(nrb, a.p0);
      }
      fft_fwd<N2>(vp, t, ex, a.tw, CtaSync(), nullptr, tmw);
      fft_fwd<N2>(vm, t, ex, a.tw, CtaSync(), nullptr, tmw);
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const cplx P = vp[i];
        vp[i] = cadd(P, vm[i]);
        vm[i] = mul_mi(csub(P, vm[i]));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * p + h;
        if (c >= C) break;
        const cplx(&X)[E] = h ? vm : vp;
        const int m = c % d;  // rank-major columns: c = r d + m
        if (m == 0) {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = X[i];
        } else {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = cmul(acc[i], X[i]);
        }
        if (m == d - 1) {
          // rank sum += acc, four complex values (16 TMEM columns) at a time
#pragma unroll
          for (int q = 0; q < E / 4; ++q) {
            uint32_t r[16];
            if (have_sum) {
              tmem_ld16(tsum + 16 * q, r);
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = 4 * q + u;
              // running sum from exact zero like passB_kernel's Sb (sign of zero included)
              const cplx old = have_sum ? mk(__hiloint2double((int)r[4 * u + 1], (int)r[4 * u]),
                                             __hiloint2double((int)r[4 * u + 3], (int)r[4 * u + 2]))
                                        : mk(0.0, 0.0);
              const cplx v = cadd(old, acc[i]);
              r[4 * u + 0] = (uint32_t)__double2loint(v.x);
              r[4 * u + 1] = (uint32_t)__double2hiint(v.x);
              r[4 * u + 2] = (uint32_t)__double2loint(v.y);
              r[4 * u + 3] = (uint32_t)__double2hiint(v.y);
            }
            tmem_st16(tsum + 16 * q, r);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          have_sum = true;
        }
      }
    }
    cplx S[E];
#pragma unroll
    for (int q = 0; q < E / 4; ++q) {
      uint32_t r[16];
      tmem_ld16(tsum + 16 * q, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < 4; ++u)
        S[4 * q + u] = have_sum ? mk(__hiloint2double((int)r[4 * u + 1], (int)r[4 * u]),
                                     __hiloint2double((int)r[4 * u + 3], (int)r[4 * u + 2]))
                                : mk(0.0, 0.0);
    }
    // (d-1)-position shift, inverse row FFT, inverse twiddle, Hermitian weight (as passB_kernel)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const long long k = (long long)kap + (long long)a.K * (t + T * i);
      const long long m = ((long long)(d - 1) * k) % a.L;
      S[i] = cmul(S[i], twL(a.tabLlo, a.tabLhi, m));
    }
    fft_inv<N2>(S, t, ex, a.tw, CtaSync(), tmw);
    const double wgt = (kap == 0 || 2 * kap == a.K) ? 1.0 : 2.0;
    if (valid) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int n2 = t + T * i;
        const cplx u = cscale(cmulc(S[i], twL(a.tabLlo, a.tabLhi, (long long)n2 * kap)), wgt);
        sts_c(a.U + (size_t)n2 * a.K_rows + rho, u);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(PIPE_TCOLS) : "memory");
}

// ---------------------------------------------------------------------------
// pass C: inverse column transforms, pruned to the sizes 1..N
// ---------------------------------------------------------------------------
struct PassCArgs {
  const double2* U;
  double* p;
  const double2* tw;
  const double2* tabK;
  long long N;
  double invL, fact;
  int d, N2, K_rows, nres;
  int res_base[MAXRES], res_cnt[MAXRES];
};

template <int N1>
__global__ void __launch_bounds__(256) passC_kernel(const PassCArgs a) {
  constexpr int E = fft_e(N1), T = fft_t(N1), SE = fft_smem_elems(N1);
  extern __shared__ double2 smem[];
  const int G = blockDim.x / T;
  const int tid = threadIdx.x, g = tid / T, t = tid - g * T;
  const int n2 = blockIdx.x * G + g;
  double2* exch = smem + g * SE;
  const double2* Ucol = a.U + (size_t)n2 * a.K_rows;
  double acc[E];
#pragma unroll
  for (int r = 0; r < E; ++r) acc[r] = 0.0;
  for (int j = 0; j < a.nres; ++j) {
    cplx v[E];
    const int cnt = a.res_cnt[j];
    const double2* src = Ucol + a.res_base[j];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int k1 = t + T * r;
      v[r] = k1 < cnt ? ld_c(src + k1) : mk(0.0, 0.0);
    }
    fft_inv<N1>(v, t, exch, a.tw);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const cplx w = ld_c(a.tabK + j * (t + T * r));
      acc[r] += w.x * v[r].x + w.y * v[r].y;  // Re(conj(W^(j n1)) v)
    }
  }
  double* dst = a.p + (size_t)n2 * N1;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int n1 = t + T * r;
    const long long o = (long long)n1 * a.N2 + n2;
    dst[n1] = (o >= a.d - 1 && o < a.N) ? (acc[r] * a.invL) / a.fact : 0.0;
  }
}

// ---------------------------------------------------------------------------
// loss coefficients: ordered reduction of the pass-A column sums
// ---------------------------------------------------------------------------
struct QArgs {
  const double* dots;
  double* coef;
  int nblk, C, kind, d, R;
  int ranks[MAXD + 1];
  int core_off[MAXD + 1];
  const int* cidx;  // TT: full fiber index -> uploaded column, -1 if dropped (contributes 0)
  const int* dslot; // deduplicated CP: column-sum slot of each column (null: identity)
};

__global__ void __launch_bounds__(1024) qcoef_kernel(const QArgs a) {
  extern __shared__ double sdot[];
  // one warp per column: coalesced partial loads, fixed-order lane sums then
  // a fixed shuffle tree (deterministic)
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = threadIdx.x >> 5; c < a.C; c += nw) {
    double s = 0.0;
    const double* p = a.dots + (size_t)(a.dslot ? __ldg(a.dslot + c) : c) * a.nblk;
    for (int b = lane; b < a.nblk; b += 32) s += p[b];
    s = warp_sum(s);
    if (lane == 0) sdot[c] = s;
  }
  __syncthreads();
  if (a.kind == TTAGG_KIND_CP) {
    // s_r = prod_{m < d-1} <F^(m)[:, r], n>   (rhs.py:401-412)
    for (int r = threadIdx.x; r < a.R; r += blockDim.x) {
      double s = 1.0;
      for (int m = 0; m < a.d - 1; ++m) s *= sdot[r * a.d + m];
      a.coef[r] = s;
    }
  } else if (threadIdx.x == 0) {
    // w = V1 V2 ... V_{d-1}, V_l[rp, rn] = sum_i H_l[rp, i, rn] n_i   (rhs.py:305-338)
    auto V = [&](int full) {
      const int c = a.cidx[full];
      return c < 0 ? 0.0 : sdot[c];
    };
    double w[64], wn[64];
    for (int rn = 0; rn < a.ranks[1]; ++rn) w[rn] = V(a.core_off[0] + rn);
    for (int lam = 1; lam < a.d - 1; ++lam) {
      const int rp_n = a.ranks[lam], rn_n = a.ranks[lam + 1];
      for (int rn = 0; rn < rn_n; ++rn) {
        double s = 0.0;
        for (int rp = 0; rp < rp_n; ++rp) s += w[rp] * V(a.core_off[lam] + rn * rp_n + rp);
        wn[rn] = s;
      }
      for (int rn = 0; rn < rn_n; ++rn) w[rn] = wn[rn];
    }
    for (int rp = 0; rp < a.ranks[a.d - 1]; ++rp) a.coef[rp] = w[rp];
  }
}

// ---------------------------------------------------------------------------
// combine: sum orders, loss tail, outputs / fused RK2 stage
// ---------------------------------------------------------------------------
struct CombineOrder {
  const double* p;     // perm-layout gain (nullable)
  const double* X;     // columns (perm layout)
  const int* tail;     // tail column indices
  const double* coef;  // tail coefficients (nullable -> no loss)
  int ntail;
  double qdiv;  // (d-1)!
};

struct CombineArgs {
  CombineOrder o[MAXORD];
  int nord;
  const double* nv;
  const double* kv;
  double alpha;
  long long N;
  int N1, N2;
  // natural outputs
  double* p;
  double* q;
  double* s;
  // perm outputs
  double* out_perm;     // s or base + a*s
  const double* base;   // stage base (nullable -> out = s)
  double a;
  double* diagp;        // per-block partials (nullable)
};

__device__ __forceinline__ void pq_at(const CombineArgs& A, size_t e, double nvv, double& P, double& Q) {
  const size_t Np = (size_t)A.N1 * A.N2;
  P = 0.0;
  Q = 0.0;
  for (int k = 0; k < A.nord; ++k) {
    const CombineOrder& o = A.o[k];
    if (o.p) P += __ldg(o.p + e);
    if (o.coef) {
      // loads batched 8 at a time, summed in rank order (deterministic)
      double tail = 0.0;
      constexpr int BT = 24;
      for (int r0 = 0; r0 < o.ntail; r0 += BT) {
        double xv[BT];
#pragma unroll
        for (int u = 0; u < BT; ++u) {
          const int r = r0 + u;
          xv[u] = r < o.ntail ? __ldg(o.X + (size_t)__ldg(o.tail + r) * Np + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < BT; ++u)
          if (r0 + u < o.ntail) tail += xv[u] * __ldg(o.coef + r0 + u);
      }
      Q += -(nvv * tail) / o.qdiv;
    }
  }
}

__global__ void __launch_bounds__(1024) combine_natural_kernel(const CombineArgs A) {
  __shared__ double tp[32][33], tq[32][33];
  const int TN1 = min(32, A.N1), TN2 = min(32, A.N2);
  const int n1_0 = blockIdx.y * TN1, n2_0 = blockIdx.x * TN2;
  for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
    const int i1 = idx % TN1, i2 = idx / TN1;
    const size_t e = (size_t)(n2_0 + i2) * A.N1 + (n1_0 + i1);
    double P, Q;
    pq_at(A, e, state_at(A.nv, A.kv, A.alpha, e), P, Q);
    tp[i2][i1] = P;
    tq[i2][i1] = Q;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
    const int i2 = idx % TN2, i1 = idx / TN2;
    const long long o = (long long)(n1_0 + i1) * A.N2 + (n2_0 + i2);
    if (o < A.N) {
      const double P = tp[i2][i1], Q = tq[i2][i1];
      if (A.p) A.p[o] = P;
      if (A.q) A.q[o] = Q;
      if (A.s) A.s[o] = P + Q;
    }
  }
}

// diag partial layout per block: [0] nonfinite count, [1] min, [2] max|.|, [3..5] M0..M2
constexpr int DIAGW = 8;

__global__ void __launch_bounds__(256) combine_perm_kernel(const CombineArgs A) {
  __shared__ double red[6][8];
  const size_t Np = (size_t)A.N1 * A.N2;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nf = 0.0, mn = INFINITY, mx = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
  if (e < Np) {
    const int n1 = (int)(e % A.N1), n2 = (int)(e / A.N1);
    const long long o = (long long)n1 * A.N2 + n2;
    double out = 0.0;
    if (o < A.N) {
      const double nvv = state_at(A.nv, A.kv, A.alpha, e);
      double P, Q;
      pq_at(A, e, nvv, P, Q);
      const double s = P + Q;
      out = A.base ? __dadd_rn(__ldg(A.base + e), __dmul_rn(A.a, s)) : s;
      if (A.diagp) {
        nf = isfinite(out) ? 0.0 : 1.0;
        mn = out;
        mx = fabs(out);
        const double k = (double)(o + 1);
        m0 = out;
        m1 = k * out;
        m2 = k * k * out;
      }
    }
    A.out_perm[e] = out;
  }
  if (!A.diagp) return;
  // deterministic block reduction
  nf = warp_sum(nf);
  m0 = warp_sum(m0);
  m1 = warp_sum(m1);
  m2 = warp_sum(m2);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = nf; red[1][wid] = mn; red[2][wid] = mx;
    red[3][wid] = m0; red[4][wid] = m1; red[5][wid] = m2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v[6] = {0.0, INFINITY, 0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      v[0] += red[0][w]; v[1] = fmin(v[1], red[1][w]); v[2] = fmax(v[2], red[2][w]);
      v[3] += red[3][w]; v[4] += red[4][w]; v[5] += red[5][w];
    }
    double* dst = A.diagp + (size_t)blockIdx.x * DIAGW;
    for (int i = 0; i < 6; ++i) dst[i] = v[i];
  }
}

// elementwise stage out = base + a*s with diagnostics (multi-GPU path, after the all-reduce)
__global__ void __launch_bounds__(256) stage_kernel(const double* base, const double* s, double a, double* out,
                                                    long long N, int N1, int N2, double* diagp) {
  __shared__ double red[6][8];
  const size_t Np = (size_t)N1 * N2;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nf = 0.0, mn = INFINITY, mx = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
  if (e < Np) {
    const int n1 = (int)(e % N1), n2 = (int)(e / N1);
    const long long o = (long long)n1 * N2 + n2;
    double v = 0.0;
    if (o < N) {
      v = base ? __dadd_rn(base[e], __dmul_rn(a, s[e])) : s[e];
      nf = isfinite(v) ? 0.0 : 1.0;
      mn = v;
      mx = fabs(v);
      const double k = (double)(o + 1);
      m0 = v; m1 = k * v; m2 = k * k * v;
    }
    if (out) out[e] = v;
  }
  if (!diagp) return;
  nf = warp_sum(nf); m0 = warp_sum(m0); m1 = warp_sum(m1); m2 = warp_sum(m2);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = nf; red[1][wid] = mn; red[2][wid] = mx;
    red[3][wid] = m0; red[4][wid] = m1; red[5][wid] = m2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v[6] = {0.0, INFINITY, 0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      v[0] += red[0][w]; v[1] = fmin(v[1], red[1][w]); v[2] = fmax(v[2], red[2][w]);
      v[3] += red[3][w]; v[4] += red[4][w]; v[5] += red[5][w];
    }
    double* dst = diagp + (size_t)blockIdx.x * DIAGW;
    for (int i = 0; i < 6; ++i) dst[i] = v[i];
  }
}

// fixed-order reduction of the per-block partials -> diag[0..5]
__global__ void diag_finalize_kernel(const double* diagp, int nb, double* diag) {
  __shared__ double red[6][256];
  double v[6] = {0.0, INFINITY, 0.0, 0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const double* p = diagp + (size_t)b * DIAGW;
    v[0] += p[0]; v[1] = fmin(v[1], p[1]); v[2] = fmax(v[2], p[2]);
    v[3] += p[3]; v[4] += p[4]; v[5] += p[5];
  }
  for (int i = 0; i < 6; ++i) red[i][threadIdx.x] = v[i];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      red[0][threadIdx.x] += red[0][threadIdx.x + w];
      red[1][threadIdx.x] = fmin(red[1][threadIdx.x], red[1][threadIdx.x + w]);
      red[2][threadIdx.x] = fmax(red[2][threadIdx.x], red[2][threadIdx.x + w]);
      red[3][threadIdx.x] += red[3][threadIdx.x + w];
      red[4][threadIdx.x] += red[4][threadIdx.x + w];
      red[5][threadIdx.x] += red[5][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < 6; ++i) diag[i] = red[i][0];
}

// RK2 bookkeeping after one step (device-resident, integrator.py:207-227):
// book[0] = current step, [1] = fail step, [2] = negativity step, [3] = rows written
__global__ void rk2_book_kernel(const double* diag_mid, const double* diag_new, int64_t* book, long long record_every,
                                double* rec) {
  if (threadIdx.x != 0) return;
  const long long step = book[0] + 1;
  book[0] = step;
  if (book[1] != 0) return;
  if (diag_mid[0] != 0.0 || diag_new[0] != 0.0) {
    book[1] = step;
    return;
  }
  if (book[2] == 0 && diag_new[1] < -1e-9 * diag_new[2]) book[2] = step;
  if (step % record_every == 0) {
    const long long row = book[3];
    rec[row * 4 + 0] = diag_new[3];
    rec[row * 4 + 1] = diag_new[4];
    rec[row * 4 + 2] = diag_new[5];
    rec[row * 4 + 3] = diag_new[1];
    book[3] = row + 1;
  }
}

__global__ void rk2_book_init_kernel(const double* diag0, int64_t* book, double* rec) {
  if (threadIdx.x != 0) return;
  book[0] = 0; book[1] = 0; book[2] = 0; book[3] = 1;
  rec[0] = diag0[3]; rec[1] = diag0[4]; rec[2] = diag0[5]; rec[3] = diag0[1];
}

// ---------------------------------------------------------------------------
// layout kernels
// ---------------------------------------------------------------------------
// dir 0: natural (length N) -> perm (length Np, zero padded); dir 1: perm -> natural
__global__ void permute_kernel(const double* __restrict__ in, double* __restrict__ out, long long N, int N1, int N2,
                               int dir, int* nonfinite = nullptr) {
  __shared__ double tile[32][33];
  const int TN1 = min(32, N1), TN2 = min(32, N2);
  const int n1_0 = blockIdx.y * TN1, n2_0 = blockIdx.x * TN2;
  if (dir == 0) {
    // read natural: consecutive threads -> consecutive n2
    for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
      const int i2 = idx % TN2, i1 = idx / TN2;
      const long long o = (long long)(n1_0 + i1) * N2 + (n2_0 + i2);
      const double x = o < N ? in[o] : 0.0;
      if (nonfinite && !isfinite(x)) *nonfinite = 1;  // benign race: every writer stores 1
      tile[i2][i1] = x;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
      const int i1 = idx % TN1, i2 = idx / TN1;
      out[(size_t)(n2_0 + i2) * N1 + (n1_0 + i1)] = tile[i2][i1];
    }
  } else {
    for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
      const int i1 = idx % TN1, i2 = idx / TN1;
      tile[i2][i1] = in[(size_t)(n2_0 + i2) * N1 + (n1_0 + i1)];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < TN1 * TN2; idx += blockDim.x) {
      const int i2 = idx % TN2, i1 = idx / TN2;
      const long long o = (long long)(n1_0 + i1) * N2 + (n2_0 + i2);
      if (o < N) out[o] = tile[i2][i1];
    }
  }
}

// ---------------------------------------------------------------------------
// dense kernels: direct summation (rhs.py:202-227), O(N^d) with N^d <= 2^26
// ---------------------------------------------------------------------------
struct DenseArgs {
  const double* V;    // N^d, row-major
  const double* nat;  // state in natural order
  double* p_perm;     // gain (perm layout) or null
  double* part;       // loss partials [chunks][N]
  double* w_perm;     // loss contraction (perm layout)
  int N, d, N1, N2, chunks;
  long long head;     // N^(d-1)
  double fact;        // d!
};

__device__ __forceinline__ size_t perm_of(long long o, int N1, int N2) {
  return (size_t)(o % N2) * N1 + (size_t)(o / N2);
}

// state in natural order: n + alpha k rounded as numpy does (state_at)
__global__ void dense_state_kernel(const double* nv, const double* kv, double alpha, double* nat, int N, int N1,
                                   int N2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) nat[i] = state_at(nv, kv, alpha, perm_of(i, N1, N2));
}

__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
  // fixed-order block reduction (deterministic): warp trees, then warp 0
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// Gain at output position o (size o+1): the tuples (i_1..i_d), 0-based, with
// i_1 + ... + i_d = o - d + 1 (sizes summing to o + 1), weighted
// C[i] n_{i_1} ... n_{i_d} in axis order (rhs.py:205-216); divided by d!.
// One CTA per o; threads stride over the leading d-1 indices.
__global__ void __launch_bounds__(256) dense_gain_kernel(const DenseArgs a) {
  __shared__ double red[8];
  const int o = blockIdx.x;
  const int s = o - (a.d - 1);
  double acc = 0.0;
  if (s >= 0) {
    for (long long m = threadIdx.x; m < a.head; m += blockDim.x) {
      int idx[MAXD];
      long long rem = m;
      int sum = 0;
      for (int j = a.d - 2; j >= 0; --j) {
        idx[j] = (int)(rem % a.N);
        rem /= a.N;
        sum += idx[j];
      }
      const int last = s - sum;
      if (last < 0 || last >= a.N) continue;
      double w = __ldg(a.V + (size_t)m * a.N + last);
      for (int j = 0; j < a.d - 1; ++j) w *= __ldg(a.nat + idx[j]);
      w *= __ldg(a.nat + last);
      acc += w;
    }
  }
  const double tot = block_sum_fixed(acc, red);
  if (threadIdx.x == 0) a.p_perm[perm_of(o, a.N1, a.N2)] = s >= 0 ? tot / a.fact : 0.0;
}

// Loss contraction w[k] = sum over the first d-1 modes of C[i_1..i_{d-1}, k]
// n_{i_1}...n_{i_{d-1}} (rhs.py:219-227): per chunk of leading indices a
// partial per k (coalesced over k), then a fixed-order sum over chunks.
__global__ void __launch_bounds__(128) dense_loss_part_kernel(const DenseArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (a.head + a.chunks - 1) / a.chunks;
  const long long m0 = (long long)blockIdx.y * per, m1 = min(a.head, m0 + per);
  double acc = 0.0;
  if (k < a.N) {
    for (long long m = m0; m < m1; ++m) {
      double u = 1.0;
      long long rem = m;
      for (int j = a.d - 2; j >= 0; --j) {
        u *= __ldg(a.nat + (int)(rem % a.N));
        rem /= a.N;
      }
      acc += __ldg(a.V + (size_t)m * a.N + k) * u;
    }
    a.part[(size_t)blockIdx.y * a.N + k] = acc;
  }
}

__global__ void dense_loss_finish_kernel(const DenseArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.N) return;
  double w = 0.0;
  for (int c = 0; c < a.chunks; ++c) w += a.part[(size_t)c * a.N + k];
  a.w_perm[perm_of(k, a.N1, a.N2)] = w;
}

// scatter an N x R row-major factor (or a TT core slice) into perm-layout columns:
// column (rank index j) goes to column colmap[j] of X — pair-interleaved
// (`paired`, the pass-A operand: column c at X[((c/2) Np + e) 2 + c%2]) or one
// column per row (the combine's tail copy); src element (o, j) at src[o*ld + srcidx[j]]
__global__ void scatter_columns_kernel(const double* __restrict__ src, long long N, int ld, int ncols,
                                       const int* __restrict__ srcidx, const int* __restrict__ colmap, double* X,
                                       int N1, int N2, int paired) {
  const size_t Np = (size_t)N1 * N2;
  const int j = blockIdx.y;
  const int sj = srcidx[j];
  const int c = colmap[j];
  double* dst = paired ? X + (size_t)(c >> 1) * 2 * Np + (c & 1) : X + (size_t)c * Np;
  const int stride = paired ? 2 : 1;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < Np; e += (size_t)gridDim.x * blockDim.x) {
    const int n1 = (int)(e % N1), n2 = (int)(e / N1);
    const long long o = (long long)n1 * N2 + n2;
    dst[e * stride] = o < N ? src[o * ld + sj] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// host: plans, workspaces, launches
// ---------------------------------------------------------------------------
int ensure(void** p, size_t* have, size_t need, bool zero = false) {
  if (*have >= need) return TTAGG_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  size_t alloc = std::max<size_t>(need, 256);
  cudaError_t e = cudaMalloc(p, alloc);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(TTAGG_ERR_NOMEM, "device allocation of " + std::to_string(alloc) + " bytes failed: " + cudaGetErrorString(e));
  }
  if (zero) {
    // cudaMemset runs on the legacy default stream, which the context's
    // non-blocking streams do not wait for: complete it before any kernel can
    // touch the buffer
    CUDA_TRY(cudaMemset(*p, 0, alloc));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  *have = alloc;
  return TTAGG_OK;
}

int get_plan(ttagg_ctx* ctx, int d, const Geom& g, OrderPlan** out) {
  auto key = std::make_pair(d, g.Np);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) {
    *out = it->second;
    return TTAGG_OK;
  }
  OrderPlan* P = new OrderPlan();
  P->d = d;
  P->g = g;
  P->L = (int64_t)d * g.Np;
  P->K = d * g.N1;
  const int N1 = g.N1;
  int base = 0, nres = 0;
  auto add = [&](int cnt) {
    P->res_base[nres] = base;
    P->res_cnt[nres] = cnt;
    base += (cnt + RB - 1) & ~(RB - 1);
    ++nres;
  };
  // rows kappa in [0, K/2] grouped by residue j = kappa mod d (kappa = j + d k1)
  add(N1 / 2 + 1);
  for (int j = 1; j < d; ++j) add(N1 / 2);
  P->nres = nres;
  P->K_rows = base;
  std::vector<int> kap(P->K_rows, -1);
  for (int j = 0; j < nres; ++j)
    for (int k1 = 0; k1 < P->res_cnt[j]; ++k1) kap[P->res_base[j] + k1] = j + d * k1;
  std::vector<double2> tk, tlo, thi;
  host_twiddles(tk, P->K, P->K, 1);
  host_twiddles(tlo, P->L, LLO, 1);
  const int64_t nhi = (P->L + LLO - 1) / LLO;
  host_twiddles(thi, P->L, nhi, LLO);
  auto up = [&](void** dst, const void* src, size_t bytes) -> int {
    CUDA_TRY(cudaMalloc(dst, bytes));
    CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    return TTAGG_OK;
  };
  TRY(up((void**)&P->tabK, tk.data(), tk.size() * sizeof(double2)));
  TRY(up((void**)&P->tabLlo, tlo.data(), tlo.size() * sizeof(double2)));
  TRY(up((void**)&P->tabLhi, thi.data(), thi.size() * sizeof(double2)));
  TRY(up((void**)&P->rowkappa, kap.data(), kap.size() * sizeof(int)));
  ctx->plans[key] = P;
  *out = P;
  return TTAGG_OK;
}

// raise the dynamic shared-memory cap once per (device, kernel instantiation):
// cudaFuncSetAttribute applies to the current device only (never inside a
// stream capture: the first launch of every shape runs eagerly)
template <typename K>
int set_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[std::make_pair(dev, (const void*)kern)];
  if (bytes > 48 * 1024 && bytes > have) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
  return TTAGG_OK;
}

// ---- pass A
// 1: TMA-fed persistent pass A for N1 >= 1024 (default); 0: passA_big_kernel
// (TTAGG_PASSA=0, kept for A/B measurements)
int passA_mode() {
  static const int mode = [] {
    const char* e = getenv("TTAGG_PASSA");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

// columns per pass-A CTA: thread groups of <= 128 threads when the transform allows
constexpr int passA_G(int T, int N2) { return std::max(1, std::min(256 / T, N2)); }

template <int N1>
int launchA(const PassAArgs& a, int N2, int npairs, cudaStream_t st) {
  constexpr int T = fft_t(N1);
  if constexpr (T >= 64) {
    bool halves = true;  // emit_split's plane map (always true for the plans make_plan builds)
    for (int j = 0; j < a.d; ++j) halves = halves && a.res_cnt[j] == N1 / 2 + (j == 0);
    if (passA_mode() == 1 && halves) {
      const size_t smem = (size_t)N1 * sizeof(double2) + (size_t)((fft_smem_elems(N1) + 1) & ~1) * sizeof(double) +
                          (passA_tmem_twiddles(N1) ? 0 : (size_t)fft_stage_table_elems<N1>() * sizeof(double2));
      auto kern = a.raw ? passA_tma_kernel<N1, true> : passA_tma_kernel<N1, false>;
      TRY(set_smem(kern, smem));
      static int resident[64] = {0};  // CTAs per SM x SMs, per device
      int dev = 0;
      CUDA_TRY(cudaGetDevice(&dev));
      if (dev >= 64) return fail(TTAGG_ERR_UNSUPPORTED, "device ordinal >= 64");
      if (!resident[dev]) {
        int sms = 0, occ = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passA_tma_kernel<N1, false>, T, smem));
        if (passA_tmem_twiddles(N1)) {
          // the occupancy query answers 1 for a kernel that allocates tensor
          // memory; the CTAs the launch bounds and the shared memory allow do
          // become resident (their column requests sum to <= 512)
          cudaFuncAttributes fa;
          int smem_sm = 0;
          CUDA_TRY(cudaFuncGetAttributes(&fa, passA_tma_kernel<N1, false>));
          CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
          const int by_smem = (int)((size_t)smem_sm / (smem + fa.sharedSizeBytes + 1024));
          const int by_tmem = 512 / (int)passA_tmem_cols(N1);
          occ = std::max(occ, std::min(passA_min_ctas(N1), std::min(by_smem, by_tmem)));
        }
        resident[dev] = std::max(1, occ) * sms;
      }
      const int nitems = npairs * N2;
      const int grid = std::max(1, std::min(nitems, resident[dev]));
      kern<<<grid, T, smem, st>>>(a, nitems);
      CUDA_TRY(cudaGetLastError());
      return TTAGG_OK;
    }
  }
  if (a.raw) return fail(TTAGG_ERR_UNSUPPORTED, "raw exchange needs the TMA-fed pass A");
  if constexpr (T >= 32) {
    const size_t smem = (size_t)fft_smem_elems(N1) * sizeof(double2);
    TRY(set_smem(passA_big_kernel<N1>, smem));
    passA_big_kernel<N1><<<npairs * N2, T, smem, st>>>(a);
    CUDA_TRY(cudaGetLastError());
    return TTAGG_OK;
  }
  const int G = passA_G(T, N2);
  const size_t smem = ((size_t)G * N1 + (size_t)G * fft_smem_elems(N1)) * sizeof(double2);
  TRY(set_smem(passA_kernel<N1>, smem));
  dim3 grid(N2 / G, npairs);
  passA_kernel<N1><<<grid, T * G, smem, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  return TTAGG_OK;
}

int nblk_for(int N1, int N2) { return fft_t(N1) >= 32 ? N2 : N2 / passA_G(fft_t(N1), N2); }

int dispatchA(int N1, const PassAArgs& a, int N2, int npairs, cudaStream_t st) {
  switch (N1) {
    case 4: return launchA<4>(a, N2, npairs, st);
    case 8: return launchA<8>(a, N2, npairs, st);
    case 16: return launchA<16>(a, N2, npairs, st);
    case 32: return launchA<32>(a, N2, npairs, st);
    case 64: return launchA<64>(a, N2, npairs, st);
    case 128: return launchA<128>(a, N2, npairs, st);
    case 256: return launchA<256>(a, N2, npairs, st);
    case 512: return launchA<512>(a, N2, npairs, st);
    case 1024: return launchA<1024>(a, N2, npairs, st);
    case 2048: return launchA<2048>(a, N2, npairs, st);
    case 4096: return launchA<4096>(a, N2, npairs, st);
  }
  return fail(TTAGG_ERR_UNSUPPORTED, "unsupported N1");
}

// ---- pass B
template <int N2>
size_t smemB() {
  constexpr int T = fft_t(N2);
  constexpr int ROWS = 128 / T;
  constexpr size_t STG = std::max((size_t)ROWS * fft_smem_elems(N2), (size_t)fft_e(N2) * 128);
  return (2 * STG + (size_t)ROWS * N2) * sizeof(double2);
}

// 1: CP pass B with a full pair of prefetch window (passB_pipe_kernel, default);
// 0: passB_kernel (TTAGG_PASSB_PIPE=0, kept for A/B measurements)
int passB_pipe() {
  static const int mode = [] {
    const char* e = getenv("TTAGG_PASSB_PIPE");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

template <int N2, bool TT>
int launchB(const PassBArgs& a, const CUtensorMap* tm, int grid, cudaStream_t st) {
  const size_t smem = smemB<N2>();
  if constexpr (N2 == 256) {
    if (tm && !TT && passB_pipe()) {
      auto kern = a.raw ? passB_pipe_kernel<true> : passB_pipe_kernel<false>;
      TRY(set_smem(kern, PIPE_SMEM));
      kern<<<grid, 128, PIPE_SMEM, st>>>(a, *tm);
      CUDA_TRY(cudaGetLastError());
      return TTAGG_OK;
    }
    if (tm) {
      TRY(set_smem(passB_kernel<N2, TT, true>, smem));
      passB_kernel<N2, TT, true><<<grid, 128, smem, st>>>(a, *tm);
      CUDA_TRY(cudaGetLastError());
      return TTAGG_OK;
    }
  }
  CUtensorMap none;
  std::memset(&none, 0, sizeof(none));
  TRY(set_smem(passB_kernel<N2, TT, false>, smem));
  passB_kernel<N2, TT, false><<<grid, 128, smem, st>>>(a, none);
  CUDA_TRY(cudaGetLastError());
  return TTAGG_OK;
}

int rowsB(int N2) { return 128 / fft_t(N2); }

// 1: pass B streams the exchange with TMA tensor copies (N2 = 256, default);
// 0: per-thread cp.async (TTAGG_PASSB_TMA=0, kept for A/B measurements)
int passB_tma() {
  static const int mode = [] {
    const char* e = getenv("TTAGG_PASSB_TMA");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The exchange T[pair][plane][n2][rho] (double2) as a 3-D fp64 tensor
// {2 K_rows, N2, 2 npairs}; one box = 8 rows x all N2 of one plane.
int exchange_tensor_map(CUtensorMap* tm, const double2* T, int K_rows, int N2, int npairs) {
  static EncodeTiledFn encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = (EncodeTiledFn)fn;
  });
  if (!encode) return fail(TTAGG_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
  const cuuint64_t dims[3] = {(cuuint64_t)2 * K_rows, (cuuint64_t)N2, (cuuint64_t)2 * npairs};
  const cuuint64_t strides[2] = {(cuuint64_t)K_rows * sizeof(double2), (cuuint64_t)K_rows * N2 * sizeof(double2)};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * rowsB(N2)), (cuuint32_t)N2, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)T, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TTAGG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return TTAGG_OK;
}

// N2 <= 256 always (make_geom): the row block is 8 rows of one 16-thread
// row transform each (the lane map in passB_kernel assumes T <= 16)
int dispatchB(int N2, bool tt, const PassBArgs& a, const CUtensorMap* tm, int grid, cudaStream_t st) {
#define TTAGG_B(n) \
  case n: return tt ? launchB<n, true>(a, tm, grid, st) : launchB<n, false>(a, tm, grid, st);
  switch (N2) {
    TTAGG_B(16)
    TTAGG_B(32)
    TTAGG_B(64)
    TTAGG_B(128)
    TTAGG_B(256)
  }
#undef TTAGG_B
  return fail(TTAGG_ERR_UNSUPPORTED, "unsupported N2");
}

// ---- pass C
template <int N1>
int launchC(const PassCArgs& a, int N2, cudaStream_t st) {
  constexpr int T = fft_t(N1);
  const int G = std::min(256 / T, N2);
  const size_t smem = (size_t)G * fft_smem_elems(N1) * sizeof(double2);
  TRY(set_smem(passC_kernel<N1>, smem));
  passC_kernel<N1><<<N2 / G, T * G, smem, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  return TTAGG_OK;
}

int dispatchC(int N1, const PassCArgs& a, int N2, cudaStream_t st) {
  switch (N1) {
    case 4: return launchC<4>(a, N2, st);
    case 8: return launchC<8>(a, N2, st);
    case 16: return launchC<16>(a, N2, st);
    case 32: return launchC<32>(a, N2, st);
    case 64: return launchC<64>(a, N2, st);
    case 128: return launchC<128>(a, N2, st);
    case 256: return launchC<256>(a, N2, st);
    case 512: return launchC<512>(a, N2, st);
    case 1024: return launchC<1024>(a, N2, st);
    case 2048: return launchC<2048>(a, N2, st);
    case 4096: return launchC<4096>(a, N2, st);
  }
  return fail(TTAGG_ERR_UNSUPPORTED, "unsupported N1");
}

// profiling helpers
cudaEvent_t prof_event(ttagg_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  ttagg_ctx* ctx;
  int cls, d;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(ttagg_ctx* c, int k, cudaStream_t s, int order = 0) : ctx(c), cls(k), d(order), st(s) {
    if (ctx->prof) {
      a = prof_event(ctx);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (ctx->prof) {
      cudaEvent_t b = prof_event(ctx);
      cudaEventRecord(b, st);
      ctx->recs.push_back({cls, d, a, b});
    }
  }
};

// Raw exchange: pass A stores the column outputs without the four-step twiddle
// and pass B applies it from per-thread constants (tensor memory).  Only the
// kernels that implement it: the TMA-fed pass A (block transforms) feeding a
// TMA-fed pass B (N2 = 256; CP pipeline kernel, CP/TT passB_kernel).
// TTAGG_RAWX=0 restores the twiddle in pass A.
bool raw_exchange(const ttagg_kernel* k) {
  static const int on = [] {
    const char* e = getenv("TTAGG_RAWX");
    return e ? atoi(e) : 1;
  }();
  const Geom& g = k->g;
  return on && k->kind != TTAGG_KIND_DENSE && g.N2 == 256 && g.N1 >= 1024 && passA_mode() == 1 && passB_tma();
}

// Pass A (column transforms + loss column sums) and qcoef of one order.
int run_passA(ttagg_ctx* ctx, const ttagg_kernel* k, const double* nv, const double* kv, double alpha, bool wantP,
              bool wantQ, ttagg_ctx::Work& w, cudaStream_t st) {
  const OrderPlan* P = k->plan;
  const Geom& g = k->g;
  const int npairs = k->xpairs;
  if (npairs > 65535) return fail(TTAGG_ERR_UNSUPPORTED, "too many columns for one kernel");
  if (wantP) {
    const size_t need = (size_t)std::max(1, 2 * npairs) * P->K_rows * g.N2 * sizeof(double2);
    TRY(ensure((void**)&w.T, &w.T_bytes, need, true));
    TRY(ensure((void**)&w.U, &w.U_bytes, (size_t)P->K_rows * g.N2 * sizeof(double2)));
    if (ctx->poison) {
      CUDA_TRY(cudaMemsetAsync(w.T, 0xFF, w.T_bytes, st));
      CUDA_TRY(cudaMemsetAsync(w.U, 0xFF, w.U_bytes, st));
    }
  }
  if (ctx->poison) {
    CUDA_TRY(cudaMemsetAsync(k->dots, 0xFF, (size_t)std::max(2, k->C_pad) * k->nblk * sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(k->coef, 0xFF, (size_t)std::max(1, k->ntail) * sizeof(double), st));
  }
  PassAArgs a{};
  a.X = k->X;
  a.nv = nv;
  a.kv = kv;
  a.alpha = alpha;
  a.T = w.T;
  a.dots = k->dots;
  a.tw = ctx->tw4096;
  a.tabK = P->tabK;
  a.tabLlo = P->tabLlo;
  a.tabLhi = P->tabLhi;
  a.d = k->d;
  a.N2 = g.N2;
  a.K_rows = P->K_rows;
  a.nblk = k->nblk;
  a.want_T = wantP ? 1 : 0;
  a.pair0 = 0;
  a.raw = raw_exchange(k) ? 1 : 0;
  for (int j = 0; j < MAXRES; ++j) {
    a.res_base[j] = P->res_base[j];
    a.res_cnt[j] = P->res_cnt[j];
  }
  {
    ProfScope ps(ctx, 0, st, k->d);
    TRY(dispatchA(g.N1, a, g.N2, npairs, st));
    ++ctx->launches;
  }
  if (wantQ) {
    QArgs q{};
    q.dots = k->dots;
    q.coef = k->coef;
    q.nblk = k->nblk;
    q.C = k->C;
    q.kind = k->kind;
    q.d = k->d;
    q.R = k->R;
    for (int i = 0; i <= MAXD; ++i) {
      q.ranks[i] = k->ranks[i];
      q.core_off[i] = k->core_off[i];
    }
    q.cidx = k->cidx;
    q.dslot = k->dslot;
    ProfScope ps(ctx, 3, st, k->d);
    const size_t qsm = std::max(1, k->C_pad) * sizeof(double);
    TRY(set_smem(qcoef_kernel, qsm));
    qcoef_kernel<<<1, 1024, qsm, st>>>(q);
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  return TTAGG_OK;
}

// Pass B (row transforms, spectral product/chain) and pass C of one order.
int run_passBC(ttagg_ctx* ctx, const ttagg_kernel* k, double* p_out, ttagg_ctx::Work& w, cudaStream_t st) {
  const OrderPlan* P = k->plan;
  const Geom& g = k->g;
  PassBArgs b{};
  b.T = w.T;
  b.U = w.U;
  b.tw = ctx->tw4096;
  b.tabLlo = P->tabLlo;
  b.tabLhi = P->tabLhi;
  b.rowkappa = P->rowkappa;
  b.L = P->L;
  b.d = k->d;
  b.K = P->K;
  b.K_rows = P->K_rows;
  b.C = k->C;
  b.kind = k->kind;
  b.Rmax = k->Rmax;
  for (int i = 0; i <= MAXD; ++i) b.ranks[i] = k->ranks[i];
  b.fdesc = k->fdesc;
  b.pmap = k->pmap;
  b.raw = raw_exchange(k) ? 1 : 0;
  const int rows = rowsB(g.N2);
  b.nrb = (P->K_rows + rows - 1) / rows;
  b.p0 = 0;
  b.p1 = k->C_pad / 2;
  int gridB = b.nrb;
  if (k->kind == TTAGG_KIND_TT) {
    // The chain state (2 Rmax spectra per frequency) lives in a per-CTA global
    // scratch.  TTAGG_TT_CTAS_PER_SM caps the resident CTAs (persistent
    // row-block loop) so that all scratch fits L2; measured slower at C4 shape
    // (occupancy matters more), so uncapped by default.
    static int per_sm = -1;
    if (per_sm < 0) {
      const char* e = getenv("TTAGG_TT_CTAS_PER_SM");
      per_sm = e ? atoi(e) : 0;
    }
    if (per_sm > 0 && ctx->num_sms > 0) gridB = std::min(gridB, per_sm * ctx->num_sms);
    const size_t need = (size_t)gridB * 2 * k->Rmax * fft_e(g.N2) * 128 * sizeof(double2);
    TRY(ensure((void**)&w.scratch, &w.scratch_bytes, need));
    if (ctx->poison) CUDA_TRY(cudaMemsetAsync(w.scratch, 0xFF, w.scratch_bytes, st));
    b.scratch = w.scratch;
  }
  CUtensorMap tm;
  const bool use_tma = g.N2 == 256 && passB_tma();
  if (use_tma) TRY(exchange_tensor_map(&tm, w.T, P->K_rows, g.N2, std::max(1, k->xpairs)));
  {
    ProfScope ps(ctx, 1, st, k->d);
    TRY(dispatchB(g.N2, k->kind == TTAGG_KIND_TT, b, use_tma ? &tm : nullptr, gridB, st));
    ++ctx->launches;
  }
  PassCArgs c{};
  c.U = w.U;
  c.p = p_out;
  c.tw = ctx->tw4096;
  c.tabK = P->tabK;
  c.N = g.N;
  c.invL = std::ldexp(1.0 / (double)P->L, -k->d);  // 1/L and pass B's 2^-d
  double f = 1.0;
  for (int i = 2; i <= k->d; ++i) f *= i;
  c.fact = f;
  c.d = k->d;
  c.N2 = g.N2;
  c.K_rows = P->K_rows;
  c.nres = P->nres;
  for (int j = 0; j < MAXRES; ++j) {
    c.res_base[j] = P->res_base[j];
    c.res_cnt[j] = P->res_cnt[j];
  }
  ProfScope ps(ctx, 2, st, k->d);
  TRY(dispatchC(g.N1, c, g.N2, st));
  ++ctx->launches;
  return TTAGG_OK;
}

int check_set(const ttagg_kernel* const* ks, int nk, Geom* g) {
  if (nk <= 0 || !ks) return fail(TTAGG_ERR_EMPTY, "no collision orders configured");
  if (nk > MAXORD) return fail(TTAGG_ERR_UNSUPPORTED, "too many orders");
  for (int i = 0; i < nk; ++i) {
    if (!ks[i]) return fail(TTAGG_ERR_ARG, "null kernel");
    if (ks[i]->N != ks[0]->N) return fail(TTAGG_ERR_SIZE, "all kernels in a set must share the same N");
  }
  *g = ks[0]->g;
  return TTAGG_OK;
}

// Relative device cost of one order's gain (column count x transform length).
double order_cost(const ttagg_kernel* k) {
  if (k->kind == TTAGG_KIND_DENSE) return 0.0;
  return (double)std::max(k->C_pad, 1) * k->plan->K_rows;
}

// Dense order (rhs_dense_P / rhs_dense_Q): gain into p_perm, loss contraction
// into the kernel's Xt (its single "tail" column, coefficient 1).
int run_dense(ttagg_ctx* ctx, const ttagg_kernel* k, const double* nv, const double* kv, double alpha, double* p_perm,
              bool wantQ, cudaStream_t st) {
  const Geom& g = k->g;
  const int N = (int)k->N;
  dense_state_kernel<<<(N + 255) / 256, 256, 0, st>>>(nv, kv, alpha, k->nat, N, g.N1, g.N2);
  CUDA_TRY(cudaGetLastError());
  DenseArgs a{};
  a.V = k->V;
  a.nat = k->nat;
  a.p_perm = p_perm;
  a.part = k->part;
  a.w_perm = k->Xt;
  a.N = N;
  a.d = k->d;
  a.N1 = g.N1;
  a.N2 = g.N2;
  a.chunks = k->chunks;
  long long head = 1;
  for (int j = 0; j < k->d - 1; ++j) head *= N;
  a.head = head;
  double f = 1.0;
  for (int i = 2; i <= k->d; ++i) f *= i;
  a.fact = f;
  ctx->launches += 1;
  if (p_perm) {
    ProfScope ps(ctx, 0, st, k->d);
    dense_gain_kernel<<<N, 256, 0, st>>>(a);
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  if (wantQ) {
    ProfScope ps(ctx, 3, st, k->d);
    dense_loss_part_kernel<<<dim3((N + 127) / 128, k->chunks), 128, 0, st>>>(a);
    CUDA_TRY(cudaGetLastError());
    dense_loss_finish_kernel<<<(N + 255) / 256, 256, 0, st>>>(a);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 2;
  }
  return TTAGG_OK;
}

int make_streams(ttagg_ctx* ctx) {
  if (ctx->s_main) return TTAGG_OK;
  int lo = 0, hi = 0;
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CUDA_TRY(cudaStreamCreateWithPriority(&ctx->s_main, cudaStreamNonBlocking, (lo + hi) / 2));
  for (int i = 0; i < ttagg_ctx::NFILL; ++i) {
    CUDA_TRY(cudaStreamCreateWithPriority(&ctx->s_fill[i], cudaStreamNonBlocking, lo));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_fill[i], cudaEventDisableTiming));
  }
  for (cudaEvent_t* e : {&ctx->ev_fork, &ctx->ev_a}) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return TTAGG_OK;
}

// host memory the driver can DMA directly (cudaHostAlloc / cudaHostRegister)
bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// memcpy split over a few host threads for large vectors (pageable <-> pinned)
void par_copy(void* dst, const void* src, size_t bytes) {
  const size_t min_part = size_t(1) << 21;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int parts = (int)std::min<size_t>(std::min<unsigned>(8u, hw), std::max<size_t>(1, bytes / min_part));
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t chunk = (bytes / parts + 63) & ~size_t(63);
  std::vector<std::thread> th;
  for (int i = 1; i < parts; ++i) {
    const size_t off = std::min(bytes, chunk * i), end = std::min(bytes, off + chunk);
    if (end > off) th.emplace_back([=] { std::memcpy((char*)dst + off, (const char*)src + off, end - off); });
  }
  std::memcpy(dst, src, std::min(bytes, chunk));
  for (auto& t : th) t.join();
}

int ensure_pinned(ttagg_ctx* ctx, size_t need) {
  if (ctx->pin_bytes >= need) return TTAGG_OK;
  if (ctx->pin) cudaFreeHost(ctx->pin);
  ctx->pin = nullptr;
  ctx->pin_bytes = 0;
  CUDA_TRY(cudaHostAlloc((void**)&ctx->pin, need, cudaHostAllocDefault));
  ctx->pin_bytes = need;
  return TTAGG_OK;
}

// Calls on a context share its workspaces (exchange, vectors, diagnostics):
// a call's stream first waits for the previous call's last operation when
// that call used another stream, and records its own end.  Skipped under
// stream capture (a captured graph is ordered by the stream it is launched on).
struct StreamUse {
  ttagg_ctx* ctx;
  cudaStream_t st;
  bool active = false;
  int enter(ttagg_ctx* c, cudaStream_t s) {
    ctx = c;
    st = s;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return TTAGG_OK;
    if (!ctx->ev_last) CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_last, cudaEventDisableTiming));
    if (ctx->last_valid && ctx->last_stream != s) CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev_last, 0));
    active = true;
    return TTAGG_OK;
  }
  ~StreamUse() {
    if (active && cudaEventRecord(ctx->ev_last, st) == cudaSuccess) {
      ctx->last_stream = st;
      ctx->last_valid = true;
    }
  }
};

// Run all orders: gains into pbuf, loss coefficients; fill the combine descriptor.
// Several orders: the main stream runs the pass A of every cheaper order, then
// pass A and pass B/C of the costliest order; the cheaper orders' pass B/C run
// on a least-priority stream once the costliest pass A is done, so their
// blocks fill the SMs that the costliest order's pass B leaves idle (its last
// wave above all).  Both streams fork from and join back into `st` (also under capture).
int run_orders(ttagg_ctx* ctx, const ttagg_kernel* const* ks, int nk, const double* nv, const double* kv,
               double alpha, bool wantP, bool wantQ, CombineArgs* A, cudaStream_t st) {
  const Geom& g = ks[0]->g;
  if (wantP) TRY(ensure((void**)&ctx->pbuf, &ctx->pbuf_bytes, (size_t)nk * g.Np * sizeof(double)));
  if (wantP && ctx->poison) CUDA_TRY(cudaMemsetAsync(ctx->pbuf, 0xFF, ctx->pbuf_bytes, st));
  auto pslot = [&](int i) { return wantP ? ctx->pbuf + (size_t)i * g.Np : nullptr; };
  std::vector<int> order;  // FFT-route orders (CP / TT), costliest first
  for (int i = 0; i < nk; ++i) {
    if (ks[i]->kind == TTAGG_KIND_DENSE)
      TRY(run_dense(ctx, ks[i], nv, kv, alpha, pslot(i), wantQ, st));
    else
      order.push_back(i);
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return order_cost(ks[x]) > order_cost(ks[y]); });
  const int nf = (int)order.size();
  static int serial = -1;  // TTAGG_SERIAL=1: one stream (diagnostics)
  if (serial < 0) {
    const char* e = getenv("TTAGG_SERIAL");
    serial = e ? atoi(e) : 0;
  }
  const bool conc = wantP && nf > 1 && !serial;
  if (!conc) {
    for (int i : order) {
      TRY(run_passA(ctx, ks[i], nv, kv, alpha, wantP, wantQ, ctx->work[i], st));
      if (wantP) TRY(run_passBC(ctx, ks[i], pslot(i), ctx->work[i], st));
    }
  } else {
    TRY(make_streams(ctx));
    const int big = order[0];
    CUDA_TRY(cudaEventRecord(ctx->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(ctx->s_main, ctx->ev_fork, 0));
    // the cheaper orders are independent: each gets its own fill stream (up to
    // NFILL; TTAGG_FILL_STREAMS=1 serialises them), so all of them can take
    // the SMs the costliest order's last pass-B wave leaves idle
    static int nfill_env = -1;
    if (nfill_env < 0) {
      const char* e = getenv("TTAGG_FILL_STREAMS");
      nfill_env = std::max(1, std::min(ttagg_ctx::NFILL, e ? atoi(e) : ttagg_ctx::NFILL));
    }
    const int nfs = std::min(nf - 1, nfill_env);
    for (int i = 0; i < nfs; ++i) CUDA_TRY(cudaStreamWaitEvent(ctx->s_fill[i], ctx->ev_fork, 0));
    for (int n = nf - 1; n >= 1; --n)  // cheapest first: their pass B/C can start early
      TRY(run_passA(ctx, ks[order[n]], nv, kv, alpha, true, wantQ, ctx->work[order[n]], ctx->s_main));
    // The cheaper orders' pass B/C wait for the costliest order's pass A
    // (TTAGG_FILL_AFTER=0: only for their own pass A): started earlier they
    // take SMs inside the persistent pass A and slow it by more than they
    // save (C5: pass A d=5 10.25 vs 10.7 ms, same total within noise).
    static int fill_after = -1;
    if (fill_after < 0) {
      const char* e = getenv("TTAGG_FILL_AFTER");
      fill_after = e ? atoi(e) : 1;
    }
    if (!fill_after) CUDA_TRY(cudaEventRecord(ctx->ev_a, ctx->s_main));
    TRY(run_passA(ctx, ks[big], nv, kv, alpha, true, wantQ, ctx->work[big], ctx->s_main));
    if (fill_after) CUDA_TRY(cudaEventRecord(ctx->ev_a, ctx->s_main));
    TRY(run_passBC(ctx, ks[big], pslot(big), ctx->work[big], ctx->s_main));
    for (int i = 0; i < nfs; ++i) CUDA_TRY(cudaStreamWaitEvent(ctx->s_fill[i], ctx->ev_a, 0));
    for (int n = 1; n < nf; ++n)
      TRY(run_passBC(ctx, ks[order[n]], pslot(order[n]), ctx->work[order[n]], ctx->s_fill[(n - 1) % nfs]));
    CUDA_TRY(cudaEventRecord(ctx->ev_a, ctx->s_main));
    CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_a, 0));
    for (int i = 0; i < nfs; ++i) {
      CUDA_TRY(cudaEventRecord(ctx->ev_fill[i], ctx->s_fill[i]));
      CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_fill[i], 0));
    }
  }
  for (int i = 0; i < nk; ++i) {
    const ttagg_kernel* k = ks[i];
    CombineOrder& o = A->o[i];
    o.p = pslot(i);
    o.X = k->Xt;
    o.tail = k->tail_cols;
    o.coef = wantQ ? k->coef : nullptr;
    o.ntail = k->ntail;
    double f = 1.0;
    for (int j = 2; j <= k->d - 1; ++j) f *= j;
    o.qdiv = f;
  }
  A->nord = nk;
  A->nv = nv;
  A->kv = kv;
  A->alpha = alpha;
  A->N = g.N;
  A->N1 = g.N1;
  A->N2 = g.N2;
  return TTAGG_OK;
}

int launch_permute(const double* in, double* out, const Geom& g, int dir, cudaStream_t st, int* nonfinite = nullptr) {
  const int TN1 = std::min(32, g.N1), TN2 = std::min(32, g.N2);
  dim3 grid(g.N2 / TN2, g.N1 / TN1);
  permute_kernel<<<grid, 256, 0, st>>>(in, out, g.N, g.N1, g.N2, dir, nonfinite);
  CUDA_TRY(cudaGetLastError());
  return TTAGG_OK;
}

int launch_combine_perm(CombineArgs& A, const Geom& g, cudaStream_t st) {
  const int nb = (int)((g.Np + 255) / 256);
  combine_perm_kernel<<<nb, 256, 0, st>>>(A);
  CUDA_TRY(cudaGetLastError());
  return TTAGG_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int ttagg_version(void) { return 10000 * 0 + 100 * 1 + 0; }

const char* ttagg_last_error(void) { return g_err.c_str(); }

int ttagg_geometry(int64_t n_classes, int64_t* out3) {
  Geom g;
  TRY(make_geom(n_classes, &g));
  out3[0] = g.Np;
  out3[1] = g.N1;
  out3[2] = g.N2;
  return TTAGG_OK;
}

int ttagg_ctx_create(int device, ttagg_ctx** out) {
  if (!out) return fail(TTAGG_ERR_ARG, "null out");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(TTAGG_ERR_ARG, "bad device index");
  CUDA_TRY(cudaSetDevice(device));
  ttagg_ctx* ctx = new ttagg_ctx();
  ctx->device = device;
  CUDA_TRY(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  std::vector<double2> tw;
  host_twiddles(tw, TW_BASE, TW_BASE, 1);
  CUDA_TRY(cudaMalloc(&ctx->tw4096, TW_BASE * sizeof(double2)));
  CUDA_TRY(cudaMemcpy(ctx->tw4096, tw.data(), TW_BASE * sizeof(double2), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&ctx->diag, 4 * DIAGW * sizeof(double)));
  CUDA_TRY(cudaMalloc(&ctx->book, 8 * sizeof(int64_t)));
  *out = ctx;
  return TTAGG_OK;
}

int ttagg_ctx_destroy(ttagg_ctx* ctx) {
  if (!ctx) return TTAGG_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& kv : ctx->plans) {
    OrderPlan* P = kv.second;
    cudaFree(P->tabK);
    cudaFree(P->tabLlo);
    cudaFree(P->tabLhi);
    cudaFree(P->rowkappa);
    delete P;
  }
  cudaFree(ctx->tw4096);
  for (auto& w : ctx->work) {
    cudaFree(w.T);
    cudaFree(w.U);
    cudaFree(w.scratch);
  }
  if (ctx->s_main) cudaStreamDestroy(ctx->s_main);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  for (int i = 0; i < ttagg_ctx::NFILL; ++i) {
    if (ctx->s_fill[i]) cudaStreamDestroy(ctx->s_fill[i]);
    if (ctx->ev_fill[i]) cudaEventDestroy(ctx->ev_fill[i]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_last) cudaEventDestroy(ctx->ev_last);
  cudaFree(ctx->pbuf);
  if (ctx->pin) cudaFreeHost(ctx->pin);
  cudaFree(ctx->vec);
  cudaFree(ctx->diagp);
  cudaFree(ctx->diag);
  cudaFree(ctx->book);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& r : ctx->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  delete ctx;
  return TTAGG_OK;
}

// upload scratch, freed on every return path
struct Scratch {
  double* src = nullptr;
  int* sel = nullptr;
  int* map = nullptr;
  ~Scratch() {
    cudaFree(src);
    cudaFree(sel);
    cudaFree(map);
  }
};

// Frees a kernel's device buffers (cudaFree(nullptr) is a no-op) and the
// handle; upload failures release a partially built kernel through
// KernelGuard, so no error path leaks device memory.
static void release_kernel(ttagg_kernel* k) {
  if (!k) return;
  cudaSetDevice(k->ctx->device);
  cudaDeviceSynchronize();
  for (void* p : {(void*)k->X, (void*)k->Xt, (void*)k->tail_cols, (void*)k->dots, (void*)k->coef, (void*)k->fdesc,
                  (void*)k->cidx, (void*)k->V, (void*)k->nat, (void*)k->part, (void*)k->pmap, (void*)k->dslot})
    cudaFree(p);
  delete k;
}

struct KernelGuard {
  ttagg_kernel* k;
  ~KernelGuard() { release_kernel(k); }
  ttagg_kernel* release() {
    ttagg_kernel* r = k;
    k = nullptr;
    return r;
  }
};

static int finish_upload(ttagg_ctx* ctx, ttagg_kernel* k, const std::vector<int>& tails) {
  if (!k->pmap) k->xpairs = k->C_pad / 2;
  k->ntail = (int)tails.size();
  CUDA_TRY(cudaMalloc(&k->tail_cols, std::max<size_t>(1, tails.size()) * sizeof(int)));
  if (!tails.empty())
    CUDA_TRY(cudaMemcpy(k->tail_cols, tails.data(), tails.size() * sizeof(int), cudaMemcpyHostToDevice));
  k->nblk = nblk_for(k->g.N1, k->g.N2);
  CUDA_TRY(cudaMalloc(&k->dots, (size_t)std::max(2, k->C_pad) * k->nblk * sizeof(double)));
  CUDA_TRY(cudaMalloc(&k->coef, std::max<size_t>(1, tails.size()) * sizeof(double)));
  TRY(get_plan(ctx, k->d, k->g, &k->plan));
  return TTAGG_OK;
}

static int cp_upload_dedup(ttagg_ctx* ctx, ttagg_kernel* k, const double* const* factors, int64_t rank,
                           const std::vector<int>& sel, std::vector<int>& tails);

static int cp_upload(ttagg_ctx* ctx, int d, int64_t n_classes, int64_t rank, const double* const* factors,
                     const int64_t* rank_subset, int64_t n_subset, bool dedup, ttagg_kernel** out) {
  if (!ctx || !out || !factors) return fail(TTAGG_ERR_ARG, "null argument");
  if (d < 2) return fail(TTAGG_ERR_ARG, "a CP kernel needs at least two factors");
  if (d > MAXD) return fail(TTAGG_ERR_UNSUPPORTED, "collision order above 8");
  if (rank < 1) return fail(TTAGG_ERR_ARG, "CP factors must be N x R matrices with R >= 1");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(make_geom(n_classes, &g));
  std::vector<int> sel;
  if (rank_subset) {
    for (int64_t i = 0; i < n_subset; ++i) {
      if (rank_subset[i] < 0 || rank_subset[i] >= rank) return fail(TTAGG_ERR_ARG, "rank index out of range");
      sel.push_back((int)rank_subset[i]);
    }
  } else {
    for (int64_t r = 0; r < rank; ++r) sel.push_back((int)r);
  }
  ttagg_kernel* k = new ttagg_kernel();
  KernelGuard guard{k};
  k->ctx = ctx;
  k->kind = TTAGG_KIND_CP;
  k->d = d;
  k->N = n_classes;
  k->g = g;
  k->R = (int)sel.size();
  k->C = d * k->R;
  k->C_pad = (k->C + 1) & ~1;
  k->Rmax = 1;
  const size_t colbytes = (size_t)g.Np * sizeof(double);
  if (dedup) {
    for (int m = 0; m < d; ++m)
      if (!factors[m]) return fail(TTAGG_ERR_ARG, "null factor");
    std::vector<int> tails;
    TRY(cp_upload_dedup(ctx, k, factors, rank, sel, tails));
    TRY(finish_upload(ctx, k, tails));
    *out = guard.release();
    return TTAGG_OK;
  }
  {
    cudaError_t e = cudaMalloc(&k->X, std::max<size_t>(2, k->C_pad) * colbytes);
    if (e != cudaSuccess) {
      return fail(TTAGG_ERR_NOMEM, "factor upload allocation failed");
    }
  }
  CUDA_TRY(cudaMemset(k->X, 0, std::max<size_t>(2, k->C_pad) * colbytes));
  CUDA_TRY(cudaMalloc(&k->Xt, std::max<size_t>(1, k->R) * colbytes));
  std::vector<int> tails;
  if (k->R > 0) {
    Scratch sc;
    CUDA_TRY(cudaMalloc(&sc.src, (size_t)n_classes * rank * sizeof(double)));
    CUDA_TRY(cudaMalloc(&sc.sel, sel.size() * sizeof(int)));
    CUDA_TRY(cudaMalloc(&sc.map, sel.size() * sizeof(int)));
    double* dsrc = sc.src;
    int *dsel = sc.sel, *dmap = sc.map;
    CUDA_TRY(cudaMemcpy(dsel, sel.data(), sel.size() * sizeof(int), cudaMemcpyHostToDevice));
    for (int m = 0; m < d; ++m) {
      if (!factors[m]) return fail(TTAGG_ERR_ARG, "null factor");
      CUDA_TRY(cudaMemcpy(dsrc, factors[m], (size_t)n_classes * rank * sizeof(double), cudaMemcpyHostToDevice));
      std::vector<int> map(sel.size());
      for (size_t j = 0; j < sel.size(); ++j) map[j] = (int)j * d + m;  // rank-major column order
      CUDA_TRY(cudaMemcpy(dmap, map.data(), map.size() * sizeof(int), cudaMemcpyHostToDevice));
      dim3 grid((unsigned)std::min<int64_t>(1024, (g.Np + 255) / 256), (unsigned)sel.size());
      scatter_columns_kernel<<<grid, 256>>>(dsrc, n_classes, (int)rank, (int)sel.size(), dsel, dmap, k->X, g.N1, g.N2, 1);
      CUDA_TRY(cudaGetLastError());
      if (m == d - 1) {  // the loss's tail factor, one column per rank term
        for (size_t j = 0; j < sel.size(); ++j) map[j] = (int)j;
        CUDA_TRY(cudaMemcpy(dmap, map.data(), map.size() * sizeof(int), cudaMemcpyHostToDevice));
        scatter_columns_kernel<<<grid, 256>>>(dsrc, n_classes, (int)rank, (int)sel.size(), dsel, dmap, k->Xt, g.N1,
                                              g.N2, 0);
        CUDA_TRY(cudaGetLastError());
      }
    }
    CUDA_TRY(cudaDeviceSynchronize());
    for (int j = 0; j < k->R; ++j) tails.push_back(j);  // rows of Xt
  }
  TRY(finish_upload(ctx, k, tails));
  *out = guard.release();
  return TTAGG_OK;
}

int ttagg_cp_upload(ttagg_ctx* ctx, int d, int64_t n_classes, int64_t rank, const double* const* factors,
                    const int64_t* rank_subset, int64_t n_subset, ttagg_kernel** out) {
  return cp_upload(ctx, d, n_classes, rank, factors, rank_subset, n_subset, false, out);
}

int ttagg_cp_upload_dedup(ttagg_ctx* ctx, int d, int64_t n_classes, int64_t rank, const double* const* factors,
                          const int64_t* rank_subset, int64_t n_subset, ttagg_kernel** out) {
  return cp_upload(ctx, d, n_classes, rank, factors, rank_subset, n_subset, true, out);
}

// Deduplicated CP upload: identical factor columns (bitwise) are found on the
// host (FNV-1a hash per column, then a full comparison with the group's
// representative).  Column c = j d + m of the rank-major order keeps its
// place in the rank/mode structure pass B walks; only the storage changes:
// every distinct ordered pair (column 2p, column 2p+1) is stored and
// transformed once (pmap), the column sums are read from the stored pair's
// slots (dslot), and identical tail columns share one row of Xt.
static int cp_upload_dedup(ttagg_ctx* ctx, ttagg_kernel* k, const double* const* factors, int64_t rank,
                           const std::vector<int>& sel, std::vector<int>& tails) {
  const int d = k->d;
  const int64_t N = k->N;
  const int R = (int)sel.size();
  const Geom& g = k->g;
  // ---- column identities
  std::vector<uint64_t> h((size_t)d * R, 1469598103934665603ull);
  for (int m = 0; m < d; ++m)
    for (int64_t i = 0; i < N; ++i) {
      const double* row = factors[m] + i * rank;
      for (int j = 0; j < R; ++j) {
        uint64_t bits;
        std::memcpy(&bits, row + sel[j], 8);
        uint64_t& x = h[(size_t)m * R + j];
        x = (x ^ bits) * 1099511628211ull;
      }
    }
  auto same = [&](int m1, int j1, int m2, int j2) {
    const double* a = factors[m1] + sel[j1];
    const double* b = factors[m2] + sel[j2];
    for (int64_t i = 0; i < N; ++i)
      if (std::memcmp(a + i * rank, b + i * rank, 8) != 0) return false;
    return true;
  };
  std::vector<int> col_id((size_t)k->C), rep_m, rep_j;
  std::map<uint64_t, std::vector<int>> by_hash;  // hash -> distinct ids
  for (int j = 0; j < R; ++j)
    for (int m = 0; m < d; ++m) {
      const uint64_t hv = h[(size_t)m * R + j];
      int id = -1;
      for (int cand : by_hash[hv])
        if (same(rep_m[cand], rep_j[cand], m, j)) {
          id = cand;
          break;
        }
      if (id < 0) {
        id = (int)rep_m.size();
        rep_m.push_back(m);
        rep_j.push_back(j);
        by_hash[hv].push_back(id);
      }
      col_id[(size_t)j * d + m] = id;
    }
  // ---- distinct ordered pairs
  std::map<std::pair<int, int>, int> pair_id;
  std::vector<std::pair<int, int>> pairs;
  std::vector<int> pmap(k->C_pad / 2), dslot(k->C);
  for (int p = 0; p < k->C_pad / 2; ++p) {
    const std::pair<int, int> key(col_id[2 * p], 2 * p + 1 < k->C ? col_id[2 * p + 1] : -1);
    auto it = pair_id.find(key);
    if (it == pair_id.end()) {
      it = pair_id.emplace(key, (int)pairs.size()).first;
      pairs.push_back(key);
    }
    pmap[p] = it->second;
  }
  for (int cc = 0; cc < k->C; ++cc) dslot[cc] = 2 * pmap[cc / 2] + (cc & 1);
  k->xpairs = (int)pairs.size();
  // ---- distinct tails (mode d-1 of every rank term)
  std::map<int, int> tail_row;
  std::vector<int> tail_rep;  // rank index j of each distinct tail
  for (int j = 0; j < R; ++j) {
    const int id = col_id[(size_t)j * d + d - 1];
    auto it = tail_row.find(id);
    if (it == tail_row.end()) {
      it = tail_row.emplace(id, (int)tail_rep.size()).first;
      tail_rep.push_back(j);
    }
    tails.push_back(it->second);
  }
  // ---- uploads
  const size_t colbytes = (size_t)g.Np * sizeof(double);
  CUDA_TRY(cudaMalloc(&k->X, (size_t)std::max(1, k->xpairs) * 2 * colbytes));
  CUDA_TRY(cudaMemset(k->X, 0, (size_t)std::max(1, k->xpairs) * 2 * colbytes));
  CUDA_TRY(cudaMalloc(&k->Xt, std::max<size_t>(1, tail_rep.size()) * colbytes));
  CUDA_TRY(cudaMalloc(&k->pmap, pmap.size() * sizeof(int)));
  CUDA_TRY(cudaMemcpy(k->pmap, pmap.data(), pmap.size() * sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&k->dslot, dslot.size() * sizeof(int)));
  CUDA_TRY(cudaMemcpy(k->dslot, dslot.data(), dslot.size() * sizeof(int), cudaMemcpyHostToDevice));
  Scratch sc;
  CUDA_TRY(cudaMalloc(&sc.src, (size_t)N * rank * sizeof(double)));
  const size_t nmax = (size_t)2 * pairs.size() + tail_rep.size() + 1;
  CUDA_TRY(cudaMalloc(&sc.sel, nmax * sizeof(int)));
  CUDA_TRY(cudaMalloc(&sc.map, nmax * sizeof(int)));
  for (int m = 0; m < d; ++m) {
    std::vector<int> s, mp;  // source ranks, destination columns
    for (size_t q = 0; q < pairs.size(); ++q)
      for (int half = 0; half < 2; ++half) {
        const int id = half ? pairs[q].second : pairs[q].first;
        if (id >= 0 && rep_m[id] == m) {
          s.push_back(sel[rep_j[id]]);
          mp.push_back((int)(2 * q + half));
        }
      }
    if (!s.empty()) {
      CUDA_TRY(cudaMemcpy(sc.src, factors[m], (size_t)N * rank * sizeof(double), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sc.sel, s.data(), s.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sc.map, mp.data(), mp.size() * sizeof(int), cudaMemcpyHostToDevice));
      dim3 grid((unsigned)std::min<int64_t>(1024, (g.Np + 255) / 256), (unsigned)s.size());
      scatter_columns_kernel<<<grid, 256>>>(sc.src, N, (int)rank, (int)s.size(), sc.sel, sc.map, k->X, g.N1, g.N2, 1);
      CUDA_TRY(cudaGetLastError());
    }
    if (m == d - 1) {  // tails: the last factor's columns
      std::vector<int> ts, tm;
      for (size_t q = 0; q < tail_rep.size(); ++q) {
        ts.push_back(sel[tail_rep[q]]);
        tm.push_back((int)q);
      }
      if (s.empty()) CUDA_TRY(cudaMemcpy(sc.src, factors[m], (size_t)N * rank * sizeof(double), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sc.sel, ts.data(), ts.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sc.map, tm.data(), tm.size() * sizeof(int), cudaMemcpyHostToDevice));
      dim3 grid((unsigned)std::min<int64_t>(1024, (g.Np + 255) / 256), (unsigned)ts.size());
      scatter_columns_kernel<<<grid, 256>>>(sc.src, N, (int)rank, (int)ts.size(), sc.sel, sc.map, k->Xt, g.N1, g.N2,
                                            0);
      CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaDeviceSynchronize());  // sc.src is reused by the next factor
  }
  return TTAGG_OK;
}

int ttagg_tt_upload(ttagg_ctx* ctx, int d, int64_t n_classes, const int64_t* ranks, const double* const* cores,
                    ttagg_kernel** out) {
  if (!ctx || !out || !cores || !ranks) return fail(TTAGG_ERR_ARG, "null argument");
  if (d < 2) return fail(TTAGG_ERR_ARG, "a TT kernel needs at least two cores");
  if (d > MAXD) return fail(TTAGG_ERR_UNSUPPORTED, "collision order above 8");
  if (ranks[0] != 1 || ranks[d] != 1) return fail(TTAGG_ERR_ARG, "boundary TT ranks must equal 1");
  for (int l = 0; l <= d; ++l)
    if (ranks[l] < 1) return fail(TTAGG_ERR_ARG, "TT ranks must be >= 1");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(make_geom(n_classes, &g));
  ttagg_kernel* k = new ttagg_kernel();
  KernelGuard guard{k};
  k->ctx = ctx;
  k->kind = TTAGG_KIND_TT;
  k->d = d;
  k->N = n_classes;
  k->g = g;
  int C = 0, Rmax = 1;
  for (int l = 0; l <= d; ++l) {
    k->ranks[l] = (int)ranks[l];
    Rmax = std::max(Rmax, (int)ranks[l]);
  }
  if (Rmax > 64) {
    return fail(TTAGG_ERR_UNSUPPORTED, "TT ranks above 64");
  }
  for (int l = 0; l < d; ++l) {
    k->core_off[l] = C;
    C += k->ranks[l] * k->ranks[l + 1];
  }
  k->core_off[d] = C;
  k->C_full = C;
  for (int l = 0; l < d; ++l)
    if (!cores[l]) {
      return fail(TTAGG_ERR_ARG, "null core");
    }
  // Live fibers.  A fiber H_l[rp, :, rn] that is identically zero adds nothing
  // to the chain (rhs.py:277-290) nor to the loss contraction (rhs.py:305-338);
  // neither does a fiber whose input state (l, rp) is fed only by dropped
  // fibers, nor one whose output state (l+1, rn) feeds no live fiber.  The
  // exactly-structured kernels of the reference (build_brownian_tt,
  // kernels.py:332-363) are mostly such zeros.
  auto fidx = [&](int l, int rp, int rn) { return k->core_off[l] + rn * k->ranks[l] + rp; };
  std::vector<char> live(C, 0);
  {
    std::vector<std::vector<char>> fwd(d + 1), used(d + 1);
    for (int l = 0; l <= d; ++l) {
      fwd[l].assign(k->ranks[l], 0);
      used[l].assign(k->ranks[l], 0);
    }
    fwd[0][0] = 1;
    used[d][0] = 1;
    std::vector<char> nz(C, 0);
    for (int l = 0; l < d; ++l) {
      const int rp_n = k->ranks[l], rn_n = k->ranks[l + 1];
      const double* H = cores[l];
      for (int rp = 0; rp < rp_n; ++rp)
        for (int64_t o = 0; o < n_classes; ++o) {
          const double* row = H + ((size_t)rp * n_classes + o) * rn_n;
          for (int rn = 0; rn < rn_n; ++rn)
            if (row[rn] != 0.0 || row[rn] != row[rn]) nz[fidx(l, rp, rn)] = 1;  // nonzero or NaN
        }
      for (int rn = 0; rn < rn_n; ++rn)
        for (int rp = 0; rp < rp_n; ++rp)
          if (nz[fidx(l, rp, rn)] && fwd[l][rp]) {
            live[fidx(l, rp, rn)] = 1;
            fwd[l + 1][rn] = 1;
          }
    }
    for (int l = d - 1; l >= 0; --l)
      for (int rn = 0; rn < k->ranks[l + 1]; ++rn)
        for (int rp = 0; rp < k->ranks[l]; ++rp) {
          char& f = live[fidx(l, rp, rn)];
          f = f && used[l + 1][rn];
          if (f) used[l][rp] = 1;
        }
  }
  // Column order: core-major.  The first core and the last one (a single
  // input or output state) list their live fibers rn-major, rp-inner.  Every
  // other core pairs its output states (rn, rn+1): for each rp the two fibers
  // (rp, rn) and (rp, rn+1) share one exchange pair and one read of the chain
  // state rp — half the state traffic of rp-inner pairs — the second one
  // accumulating in the pass-B CTA's tensor memory (FD_ACC1); a dropped fiber
  // keeps its slot as a no-op, and an odd last output state falls back to
  // rp-inner pairs.
  std::vector<int> cidx(C, -1), desc;
  auto group_ends = [&](int l, int rn, int& first, int& last) {
    first = last = -1;
    for (int rp = 0; rp < k->ranks[l]; ++rp)
      if (live[fidx(l, rp, rn)]) {
        if (first < 0) first = rp;
        last = rp;
      }
  };
  auto push = [&](int l, int rp, int rn, int extra) {
    int first, last;
    group_ends(l, rn, first, last);
    cidx[fidx(l, rp, rn)] = (int)desc.size();
    desc.push_back(fd_pack(l, rn, rp, rp == first, rp == last) | extra);
  };
  for (int l = 0; l < d; ++l) {
    const int rp_n = k->ranks[l], rn_n = k->ranks[l + 1];
    bool paired = l > 0 && l < d - 1 && rn_n >= 2 && rp_n >= 2;
    if (paired) {  // only where the no-op slots stay rare (dense cores): they cost column transforms
      int live_n = 0, slots = 0;
      for (int rn = 0; rn < rn_n; ++rn)
        for (int rp = 0; rp < rp_n; ++rp) live_n += live[fidx(l, rp, rn)];
      for (int rn = 0; rn + 1 < rn_n; rn += 2)
        for (int rp = 0; rp < rp_n; ++rp) slots += 2 * (live[fidx(l, rp, rn)] || live[fidx(l, rp, rn + 1)]);
      for (int rp = 0; rp < rp_n && (rn_n & 1); ++rp) slots += live[fidx(l, rp, rn_n - 1)];
      paired = slots * 20 <= live_n * 21;  // <= 5% no-ops
    }
    int rn = 0;
    if (paired) {
      for (; rn + 1 < rn_n; rn += 2) {
        bool any = false;
        for (int rp = 0; rp < rp_n && !any; ++rp) any = live[fidx(l, rp, rn)] || live[fidx(l, rp, rn + 1)];
        if (!any) continue;
        if (desc.size() & 1) desc.push_back(FD_NOOP);  // pairs start on an even column
        for (int rp = 0; rp < rp_n; ++rp) {
          const bool a0 = live[fidx(l, rp, rn)], a1 = live[fidx(l, rp, rn + 1)];
          if (!a0 && !a1) continue;
          if (a0) push(l, rp, rn, 0); else desc.push_back(FD_NOOP);
          if (a1) push(l, rp, rn + 1, FD_ACC1); else desc.push_back(FD_NOOP);
        }
      }
    }
    for (; rn < rn_n; ++rn)
      for (int rp = 0; rp < rp_n; ++rp)
        if (live[fidx(l, rp, rn)]) push(l, rp, rn, 0);
  }
  for (int f : desc) k->live_cols += !(f & FD_NOOP);
  if (desc.empty()) desc.push_back(FD_NOOP);  // an all-zero kernel: one zero column
  k->C = (int)desc.size();
  k->C_pad = (k->C + 1) & ~1;
  k->Rmax = Rmax;
  k->R = k->ranks[d - 1];
  CUDA_TRY(cudaMalloc(&k->fdesc, desc.size() * sizeof(int)));
  CUDA_TRY(cudaMemcpy(k->fdesc, desc.data(), desc.size() * sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&k->cidx, (size_t)C * sizeof(int)));
  CUDA_TRY(cudaMemcpy(k->cidx, cidx.data(), (size_t)C * sizeof(int), cudaMemcpyHostToDevice));
  const size_t colbytes = (size_t)g.Np * sizeof(double);
  CUDA_TRY(cudaMalloc(&k->X, std::max<size_t>(2, k->C_pad) * colbytes));
  CUDA_TRY(cudaMemset(k->X, 0, std::max<size_t>(2, k->C_pad) * colbytes));
  CUDA_TRY(cudaMalloc(&k->Xt, std::max<size_t>(1, k->ranks[d - 1]) * colbytes));
  Scratch sc;
  size_t maxcore = 0;
  for (int l = 0; l < d; ++l) maxcore = std::max(maxcore, (size_t)k->ranks[l] * n_classes * k->ranks[l + 1]);
  CUDA_TRY(cudaMalloc(&sc.src, maxcore * sizeof(double)));
  CUDA_TRY(cudaMalloc(&sc.sel, 64 * 64 * sizeof(int)));
  CUDA_TRY(cudaMalloc(&sc.map, 64 * 64 * sizeof(int)));
  double* dsrc = sc.src;
  int *dsel = sc.sel, *dmap = sc.map;
  for (int l = 0; l < d; ++l) {
    const int rp_n = k->ranks[l], rn_n = k->ranks[l + 1];
    CUDA_TRY(cudaMemcpy(dsrc, cores[l], (size_t)rp_n * n_classes * rn_n * sizeof(double), cudaMemcpyHostToDevice));
    // element H[rp, o, rn] at rp*N*rn_n + o*rn_n + rn.  Handle one rp slab at a time:
    for (int rp = 0; rp < rp_n; ++rp) {
      std::vector<int> sidx, map;
      for (int rn = 0; rn < rn_n; ++rn)
        if (cidx[fidx(l, rp, rn)] >= 0) {
          sidx.push_back(rn);
          map.push_back(cidx[fidx(l, rp, rn)]);  // uploaded column of this live fiber
        }
      const int nsel = (int)sidx.size();
      if (nsel > 0) {
        CUDA_TRY(cudaMemcpy(dsel, sidx.data(), nsel * sizeof(int), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dmap, map.data(), nsel * sizeof(int), cudaMemcpyHostToDevice));
        dim3 grid((unsigned)std::min<int64_t>(1024, (g.Np + 255) / 256), (unsigned)nsel);
        scatter_columns_kernel<<<grid, 256>>>(dsrc + (size_t)rp * n_classes * rn_n, n_classes, rn_n, nsel, dsel,
                                              dmap, k->X, g.N1, g.N2, 1);
        CUDA_TRY(cudaGetLastError());
      }
      if (l == d - 1) {  // last core (rn_n = 1): the loss's tail fibers, one row of Xt per rp
        const int zero = 0, row = rp;
        CUDA_TRY(cudaMemcpy(dsel, &zero, sizeof(int), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dmap, &row, sizeof(int), cudaMemcpyHostToDevice));
        dim3 grid((unsigned)std::min<int64_t>(1024, (g.Np + 255) / 256), 1u);
        scatter_columns_kernel<<<grid, 256>>>(dsrc + (size_t)rp * n_classes * rn_n, n_classes, rn_n, 1, dsel, dmap,
                                              k->Xt, g.N1, g.N2, 0);
        CUDA_TRY(cudaGetLastError());
      }
      CUDA_TRY(cudaDeviceSynchronize());
    }
  }
  std::vector<int> tails;
  for (int rp = 0; rp < k->ranks[d - 1]; ++rp) tails.push_back(rp);  // rows of Xt
  TRY(finish_upload(ctx, k, tails));
  *out = guard.release();
  return TTAGG_OK;
}

int ttagg_dense_upload(ttagg_ctx* ctx, int d, int64_t n_classes, const double* values, ttagg_kernel** out) {
  if (!ctx || !out || !values) return fail(TTAGG_ERR_ARG, "null argument");
  if (d < 2) return fail(TTAGG_ERR_ARG, "dense kernels must have dimension >= 2");
  if (d > MAXD) return fail(TTAGG_ERR_UNSUPPORTED, "collision order above 8");
  int64_t total = 1;
  for (int j = 0; j < d; ++j) {
    total *= n_classes;
    if (total > (int64_t(1) << 26))
      return fail(TTAGG_ERR_UNSUPPORTED, "dense evaluation over the budget of 2^26 elements (rhs.py:47, 188-199)");
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(make_geom(n_classes, &g));
  ttagg_kernel* k = new ttagg_kernel();
  KernelGuard guard{k};
  k->ctx = ctx;
  k->kind = TTAGG_KIND_DENSE;
  k->d = d;
  k->N = n_classes;
  k->g = g;
  k->C = 0;
  k->C_pad = 0;
  k->R = 1;
  const int64_t head = total / n_classes;
  k->chunks = (int)std::max<int64_t>(1, std::min<int64_t>(head, 2048 / std::max<int64_t>(1, (n_classes + 127) / 128)));
  CUDA_TRY(cudaMalloc(&k->V, (size_t)total * sizeof(double)));
  CUDA_TRY(cudaMemcpy(k->V, values, (size_t)total * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&k->nat, (size_t)n_classes * sizeof(double)));
  CUDA_TRY(cudaMalloc(&k->part, (size_t)k->chunks * n_classes * sizeof(double)));
  // the loss contraction is the order's single tail column (coefficient 1):
  // the combine forms -(n w)/(d-1)! exactly as rhs.py:227
  CUDA_TRY(cudaMalloc(&k->Xt, (size_t)g.Np * sizeof(double)));
  CUDA_TRY(cudaMemset(k->Xt, 0, (size_t)g.Np * sizeof(double)));
  const int zero = 0;
  const double one = 1.0;
  k->ntail = 1;
  CUDA_TRY(cudaMalloc(&k->tail_cols, sizeof(int)));
  CUDA_TRY(cudaMemcpy(k->tail_cols, &zero, sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&k->coef, sizeof(double)));
  CUDA_TRY(cudaMemcpy(k->coef, &one, sizeof(double), cudaMemcpyHostToDevice));
  *out = guard.release();
  return TTAGG_OK;
}

int ttagg_kernel_free(ttagg_kernel* k) {
  release_kernel(k);
  return TTAGG_OK;
}

int ttagg_kernel_info(const ttagg_kernel* k, int64_t* info) {
  if (!k || !info) return fail(TTAGG_ERR_ARG, "null argument");
  info[0] = k->kind;
  info[1] = k->d;
  info[2] = k->N;
  info[3] = k->kind == TTAGG_KIND_TT ? k->live_cols : k->C;
  info[4] = k->g.Np;
  info[5] = k->g.N1;
  info[6] = k->g.N2;
  info[7] = k->plan ? k->plan->K_rows : 0;
  return TTAGG_OK;
}

int ttagg_rhs(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels, const double* n, double* p,
              double* q, double* s, int flags, void* stream) {
  if (!ctx || !n) return fail(TTAGG_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(check_set(kernels, n_kernels, &g));
  cudaStream_t st = (cudaStream_t)stream;
  StreamUse use;
  TRY(use.enter(ctx, st));
  bool wantP = flags & TTAGG_WANT_P, wantQ = flags & TTAGG_WANT_Q;
  if (!wantP && !wantQ) wantP = wantQ = true;
  const bool host = flags & TTAGG_HOST_PTRS;
  // vec layout: [n natural N][n perm Np][p N][q N][s N]
  const size_t nb = (size_t)g.N * sizeof(double);
  const int64_t Na = (g.N + 31) & ~(int64_t)31;  // 256-byte aligned sub-buffers
  TRY(ensure((void**)&ctx->vec, &ctx->vec_bytes, (4 * Na + g.Np) * sizeof(double) + 1024));
  double* v_nat = ctx->vec;
  double* v_perm = v_nat + Na;
  double* v_p = v_perm + g.Np;
  double* v_q = v_p + Na;
  double* v_s = v_q + Na;
  const double* nsrc = n;
  int* dflag = reinterpret_cast<int*>(ctx->book + 6);
  // host-pointer path: pageable buffers go through the context's page-locked
  // staging area ([n][p][q][s], copied by a few host threads); pinned ones
  // are transferred directly
  double* out_host[3] = {p, q, s};
  double* out_stage[3] = {nullptr, nullptr, nullptr};
  if (host) {
    const bool in_pinned = is_pinned(n);
    bool need_stage = !in_pinned;
    for (double* o : out_host) need_stage |= (o && !is_pinned(o));
    if (need_stage) TRY(ensure_pinned(ctx, 4 * Na * sizeof(double)));
    CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    const double* src = n;
    if (!in_pinned) {
      CUDA_TRY(cudaStreamSynchronize(st));  // the staging area may still feed an earlier copy
      par_copy(ctx->pin, n, nb);
      src = ctx->pin;
    }
    for (int i = 0; i < 3; ++i)
      if (out_host[i] && !is_pinned(out_host[i])) out_stage[i] = ctx->pin + (size_t)(i + 1) * Na;
    CUDA_TRY(cudaMemcpyAsync(v_nat, src, nb, cudaMemcpyHostToDevice, st));
    nsrc = v_nat;
  }
  TRY(launch_permute(nsrc, v_perm, g, 0, st, host ? dflag : nullptr));
  ++ctx->launches;
  CombineArgs A{};
  TRY(run_orders(ctx, kernels, n_kernels, v_perm, nullptr, 0.0, wantP, wantQ, &A, st));
  A.p = p ? (host ? v_p : p) : nullptr;
  A.q = q ? (host ? v_q : q) : nullptr;
  A.s = s ? (host ? v_s : s) : nullptr;
  {
    ProfScope ps(ctx, 3, st);
    const int TN1 = std::min(32, g.N1), TN2 = std::min(32, g.N2);
    dim3 grid(g.N2 / TN2, g.N1 / TN1);
    combine_natural_kernel<<<grid, 1024, 0, st>>>(A);
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  if (host) {
    int hflag = 0;
    CUDA_TRY(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    const double* dev_out[3] = {v_p, v_q, v_s};
    for (int i = 0; i < 3; ++i)
      if (out_host[i])
        CUDA_TRY(cudaMemcpyAsync(out_stage[i] ? out_stage[i] : out_host[i], dev_out[i], nb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (hflag) return fail(TTAGG_ERR_NONFINITE, "concentration state contains non-finite entries");
    for (int i = 0; i < 3; ++i)
      if (out_stage[i]) par_copy(out_host[i], out_stage[i], nb);
  }
  return TTAGG_OK;
}

int ttagg_rhs_perm(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels, const double* n_perm,
                   const double* k_perm, double alpha, double* s_perm, void* stream) {
  if (!ctx || !n_perm || !s_perm) return fail(TTAGG_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(check_set(kernels, n_kernels, &g));
  cudaStream_t st = (cudaStream_t)stream;
  StreamUse use;
  TRY(use.enter(ctx, st));
  CombineArgs A{};
  TRY(run_orders(ctx, kernels, n_kernels, n_perm, k_perm, alpha, true, true, &A, st));
  A.out_perm = s_perm;
  A.base = nullptr;
  A.diagp = nullptr;
  ProfScope ps(ctx, 3, st);
  TRY(launch_combine_perm(A, g, st));
  ++ctx->launches;
  return TTAGG_OK;
}

int ttagg_permute(ttagg_ctx* ctx, int64_t n_classes, const double* in, double* out, int dir, void* stream) {
  if (!ctx || !in || !out) return fail(TTAGG_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(make_geom(n_classes, &g));
  return launch_permute(in, out, g, dir ? 1 : 0, (cudaStream_t)stream);
}

int ttagg_stage(ttagg_ctx* ctx, int64_t n_classes, const double* base, const double* s, double a, double* out,
                double* diag, void* stream) {
  if (!ctx || !s) return fail(TTAGG_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(make_geom(n_classes, &g));
  cudaStream_t st = (cudaStream_t)stream;
  StreamUse use;
  TRY(use.enter(ctx, st));
  const int nb = (int)((g.Np + 255) / 256);
  double* dp = nullptr;
  if (diag) {
    TRY(ensure((void**)&ctx->diagp, &ctx->diagp_bytes, (size_t)nb * DIAGW * sizeof(double)));
    dp = ctx->diagp;
  }
  stage_kernel<<<nb, 256, 0, st>>>(base, s, a, out, g.N, g.N1, g.N2, dp);
  CUDA_TRY(cudaGetLastError());
  if (diag) {
    diag_finalize_kernel<<<1, 256, 0, st>>>(dp, nb, diag);
    CUDA_TRY(cudaGetLastError());
  }
  return TTAGG_OK;
}

int ttagg_rk2(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels, double* n_inout, double t0,
              double dt, int64_t steps, int64_t record_every, double* records, int64_t* fail_step,
              int64_t* neg_step, int flags, void* stream) {
  if (!ctx || !n_inout || !records || !fail_step || !neg_step) return fail(TTAGG_ERR_ARG, "null argument");
  if (!(dt > 0)) return fail(TTAGG_ERR_ARG, "dt must be positive");
  if (steps < 1 || record_every < 1) return fail(TTAGG_ERR_ARG, "steps and record_every must be >= 1");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CUDA_TRY(cudaSetDevice(ctx->device));
  Geom g;
  TRY(check_set(kernels, n_kernels, &g));
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & TTAGG_HOST_PTRS;
  const int64_t nrows = steps / record_every + 1;
  // graphs and the stream this call may create are released on every path
  struct Owned {
    cudaGraphExec_t ge[2] = {nullptr, nullptr};
    cudaStream_t own = nullptr;
    ~Owned() {
      for (auto& e : ge)
        if (e) cudaGraphExecDestroy(e);
      if (own) {
        cudaStreamSynchronize(own);
        cudaStreamDestroy(own);
      }
    }
  } owned;
  const bool use_graph = !ctx->prof;
  cudaStream_t cap = st;
  if (use_graph && st == nullptr) {
    // the legacy stream cannot be captured: run on a stream of our own, after
    // everything already queued on the device
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaStreamCreateWithFlags(&owned.own, cudaStreamNonBlocking));
    cap = owned.own;
  }
  st = cap;
  StreamUse use;
  TRY(use.enter(ctx, st));
  // vec layout: [nat N][A Np][B Np][C Np][rec nrows*4]
  const size_t nb = (size_t)g.N * sizeof(double);
  const int64_t Na = (g.N + 31) & ~(int64_t)31;  // 256-byte aligned sub-buffers
  TRY(ensure((void**)&ctx->vec, &ctx->vec_bytes, (Na + 3 * g.Np + nrows * 4) * sizeof(double) + 1024));
  double* v_nat = ctx->vec;
  double* vA = v_nat + Na;
  double* vB = vA + g.Np;
  double* vC = vB + g.Np;
  double* rec = vC + g.Np;
  const int nblk = (int)((g.Np + 255) / 256);
  TRY(ensure((void**)&ctx->diagp, &ctx->diagp_bytes, (size_t)2 * nblk * DIAGW * sizeof(double)));
  double* dpm = ctx->diagp;
  double* dpn = ctx->diagp + (size_t)nblk * DIAGW;
  double* dmid = ctx->diag;
  double* dnew = ctx->diag + DIAGW;
  double* d0 = ctx->diag + 2 * DIAGW;
  // the initial state's finiteness (ConcentrationState, rhs.py:71-72) is
  // checked on the device while it is permuted
  int* dflag = reinterpret_cast<int*>(ctx->book + 6);
  CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int), st));
  CUDA_TRY(cudaMemcpyAsync(v_nat, n_inout, nb, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  TRY(launch_permute(v_nat, vA, g, 0, st, dflag));
  {
    int hflag = 0;
    CUDA_TRY(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (hflag) return fail(TTAGG_ERR_NONFINITE, "concentration state contains non-finite entries");
  }
  // initial record
  stage_kernel<<<nblk, 256, 0, st>>>(vA, vA, 0.0, nullptr, g.N, g.N1, g.N2, dpn);
  diag_finalize_kernel<<<1, 256, 0, st>>>(dpn, nblk, d0);
  rk2_book_init_kernel<<<1, 32, 0, st>>>(d0, ctx->book, rec);
  CUDA_TRY(cudaGetLastError());

  double* cur = vA;
  double* mid = vB;
  double* nxt = vC;
  // one step: k1 -> mid = n + dt/2 k1 ; k2 at mid -> nxt = n + dt k2
  auto step_once = [&](double* n_cur, double* n_mid, double* n_nxt) -> int {
    CombineArgs A{};
    TRY(run_orders(ctx, kernels, n_kernels, n_cur, nullptr, 0.0, true, true, &A, st));
    A.out_perm = n_mid;
    A.base = n_cur;
    A.a = 0.5 * dt;
    A.diagp = dpm;
    TRY(launch_combine_perm(A, g, st));
    diag_finalize_kernel<<<1, 256, 0, st>>>(dpm, nblk, dmid);
    CombineArgs B{};
    TRY(run_orders(ctx, kernels, n_kernels, n_mid, nullptr, 0.0, true, true, &B, st));
    B.out_perm = n_nxt;
    B.base = n_cur;
    B.a = dt;
    B.diagp = dpn;
    TRY(launch_combine_perm(B, g, st));
    diag_finalize_kernel<<<1, 256, 0, st>>>(dpn, nblk, dnew);
    rk2_book_kernel<<<1, 32, 0, st>>>(dmid, dnew, ctx->book, record_every, rec);
    CUDA_TRY(cudaGetLastError());
    return TTAGG_OK;
  };
  int64_t host_book[4] = {0, 0, 0, 0};
  if (use_graph) {
    // capture one step for each buffer parity into CUDA graphs; step 1 runs
    // eagerly (workspaces are allocated before capture, which cannot allocate)
    TRY(step_once(cur, mid, nxt));
    std::swap(cur, nxt);
    for (int par = 0; par < 2 && steps > 1; ++par) {
      double* c0 = par == 0 ? cur : nxt;
      double* c1 = par == 0 ? nxt : cur;
      cudaGraph_t gr = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      const int rc = step_once(c0, mid, c1);
      const cudaError_t ec = cudaStreamEndCapture(cap, &gr);
      if (rc) {
        if (gr) cudaGraphDestroy(gr);
        return rc;
      }
      if (ec != cudaSuccess) return fail(TTAGG_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
      const cudaError_t ei = cudaGraphInstantiate(&owned.ge[par], gr, 0);
      cudaGraphDestroy(gr);
      if (ei != cudaSuccess) return fail(TTAGG_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    }
    int64_t done = 1;
    int par = 0;
    while (done < steps) {
      const int64_t chunk = std::min<int64_t>(steps - done, 64);
      for (int64_t i = 0; i < chunk; ++i) {
        CUDA_TRY(cudaGraphLaunch(owned.ge[par], cap));
        par ^= 1;
      }
      done += chunk;
      CUDA_TRY(cudaMemcpyAsync(host_book, ctx->book, sizeof(host_book), cudaMemcpyDeviceToHost, cap));
      CUDA_TRY(cudaStreamSynchronize(cap));
      if (host_book[1] != 0) break;
    }
    if (par == 1) std::swap(cur, nxt);  // final state location
  } else {
    for (int64_t s = 1; s <= steps; ++s) {
      TRY(step_once(cur, mid, nxt));
      std::swap(cur, nxt);
      if (s % 64 == 0 || s == steps) {
        CUDA_TRY(cudaMemcpyAsync(host_book, ctx->book, sizeof(host_book), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (host_book[1] != 0) break;
      }
    }
  }
  CUDA_TRY(cudaMemcpyAsync(host_book, ctx->book, sizeof(host_book), cudaMemcpyDeviceToHost, cap));
  TRY(launch_permute(cur, v_nat, g, 1, cap));
  // records: device rows (M0, M1, M2, min) -> (t, M0, M1, M2, min)
  std::vector<double> hrec((size_t)nrows * 4);
  CUDA_TRY(cudaMemcpyAsync(hrec.data(), rec, hrec.size() * sizeof(double), cudaMemcpyDeviceToHost, cap));
  CUDA_TRY(cudaMemcpyAsync(n_inout, v_nat, nb, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, cap));
  CUDA_TRY(cudaStreamSynchronize(cap));
  const int64_t rows = std::min<int64_t>(host_book[3], nrows);
  std::vector<double> out((size_t)nrows * 5, 0.0);
  // times as the reference accumulates them (state.t + dt per step,
  // integrator.py:179, 207): row r holds step r * record_every
  double t = t0;
  int64_t row = 0;
  for (int64_t step = 0; row < rows; ++step) {
    if (step > 0) t = t + dt;
    if (step % record_every == 0) {
      out[row * 5] = t;
      for (int c = 0; c < 4; ++c) out[row * 5 + 1 + c] = hrec[row * 4 + c];
      ++row;
    }
  }
  if (host) {
    std::memcpy(records, out.data(), out.size() * sizeof(double));
  } else {
    CUDA_TRY(cudaMemcpy(records, out.data(), out.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  *fail_step = host_book[1];
  *neg_step = host_book[2];
  return TTAGG_OK;
}

int ttagg_profile_enable(ttagg_ctx* ctx, int on) {
  if (!ctx) return fail(TTAGG_ERR_ARG, "null ctx");
  ctx->prof = on != 0;
  return TTAGG_OK;
}

int ttagg_debug_poison(ttagg_ctx* ctx, int on) {
  if (!ctx) return fail(TTAGG_ERR_ARG, "null argument");
  ctx->poison = on != 0;
  return TTAGG_OK;
}

int ttagg_launch_count(ttagg_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return fail(TTAGG_ERR_ARG, "null argument");
  *out = ctx->launches;
  return TTAGG_OK;
}

int ttagg_profile_read(ttagg_ctx* ctx, double* out72) {
  if (!ctx || !out72) return fail(TTAGG_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  for (int i = 0; i < 72; ++i) out72[i] = 0.0;
  for (auto& r : ctx->recs) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    const int slot = (r.cls * 9 + std::min(std::max(r.d, 0), 8)) * 2;
    out72[slot] += ms;
    out72[slot + 1] += 1.0;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->recs.clear();
  return TTAGG_OK;
}


// ---------------------------------------------------------------------------
// Device group: rank-sharded RHS / RK2 over several GPUs of one process
// (the single-process counterpart of dist.py's torchrun
// path).  Every device holds its own context and the kernel shards the caller
// uploaded there; one NCCL all-reduce (sum) per RHS completes dn/dt on every
// device, which then applies the identical stage update to its replica of n.
// NCCL is loaded at run time (dlopen, the process's libnccl.so.2 — torch's
// copy when torch is loaded), so the library has no link-time NCCL
// dependency and single-device use needs none.
// ---------------------------------------------------------------------------
}  // extern "C"

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.commInitAll = (decltype(api.commInitAll))dlsym(h, "ncclCommInitAll");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
    api.ok = api.commInitAll && api.commDestroy && api.allReduce && api.groupStart && api.groupEnd && api.errStr;
  });
  return api;
}

#define NCCL_TRY(x)                                                                                 \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess) return fail(TTAGG_ERR_NCCL, std::string(#x) + ": " + nccl().errStr(r_)); \
  } while (0)

}  // namespace

struct ttagg_group {
  int n = 0;
  std::vector<ttagg_ctx*> ctx;
  std::vector<cudaStream_t> st;
  std::vector<ncclComm_t> comm;
  std::vector<double*> buf;  // per device: natural n, 3 perm states, perm s, 3N natural partials
  std::vector<size_t> buf_bytes;
  double* pin = nullptr;  // page-locked staging on device 0's side
  size_t pin_bytes = 0;
  std::mutex mu;
};

namespace {

// all-reduce (sum) of `count` doubles at ptr[i] on every device of the group
int group_allreduce(ttagg_group* G, const std::vector<double*>& ptr, size_t count) {
  if (G->n == 1 && G->comm.empty()) return TTAGG_OK;
  NCCL_TRY(nccl().groupStart());
  for (int i = 0; i < G->n; ++i) {
    CUDA_TRY(cudaSetDevice(G->ctx[i]->device));
    const ncclResult_t r = nccl().allReduce(ptr[i], ptr[i], count, ncclFloat64, ncclSum, G->comm[i], G->st[i]);
    if (r != ncclSuccess) {
      nccl().groupEnd();
      return fail(TTAGG_ERR_NCCL, std::string("ncclAllReduce: ") + nccl().errStr(r));
    }
  }
  NCCL_TRY(nccl().groupEnd());
  return TTAGG_OK;
}

int group_kernels(ttagg_group* G, const ttagg_kernel* const* kernels, int nk, int i, std::vector<const ttagg_kernel*>& out,
                  Geom* g) {
  out.clear();
  for (int j = 0; j < nk; ++j) {
    const ttagg_kernel* k = kernels[(size_t)i * nk + j];
    if (!k) continue;
    if (k->ctx != G->ctx[i]) return fail(TTAGG_ERR_ARG, "kernel shard uploaded to another device's context");
    out.push_back(k);
  }
  if (!out.empty()) TRY(check_set(out.data(), (int)out.size(), g));
  return TTAGG_OK;
}

}  // namespace

extern "C" {

int ttagg_group_create(const int* devices, int n_dev, ttagg_group** out) {
  if (!devices || !out || n_dev < 1) return fail(TTAGG_ERR_ARG, "a device group needs at least one device");
  auto* G = new ttagg_group();
  struct Guard {
    ttagg_group* g;
    ~Guard() {
      if (g) ttagg_group_destroy(g);
    }
  } guard{G};
  G->n = n_dev;
  for (int i = 0; i < n_dev; ++i) {
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) return fail(TTAGG_ERR_ARG, "a device appears twice in the group");
    ttagg_ctx* c = nullptr;
    TRY(ttagg_ctx_create(devices[i], &c));
    G->ctx.push_back(c);
    cudaStream_t s = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    G->st.push_back(s);
    G->buf.push_back(nullptr);
    G->buf_bytes.push_back(0);
  }
  if (n_dev > 1 || getenv("TTAGG_GROUP_NCCL")) {  // one device: no collective needed (forced on for tests)
    if (!nccl().ok) return fail(TTAGG_ERR_NCCL, "libnccl.so.2 could not be loaded");
    G->comm.resize(n_dev);
    NCCL_TRY(nccl().commInitAll(G->comm.data(), n_dev, devices));
  }
  *out = G;
  guard.g = nullptr;
  return TTAGG_OK;
}

int ttagg_group_destroy(ttagg_group* G) {
  if (!G) return TTAGG_OK;
  for (int i = 0; i < (int)G->ctx.size(); ++i) {
    cudaSetDevice(G->ctx[i]->device);
    if (i < (int)G->st.size() && G->st[i]) {
      cudaStreamSynchronize(G->st[i]);
      cudaStreamDestroy(G->st[i]);
    }
    if (i < (int)G->buf.size()) cudaFree(G->buf[i]);
  }
  for (ncclComm_t c : G->comm)
    if (c) nccl().commDestroy(c);
  for (ttagg_ctx* c : G->ctx) ttagg_ctx_destroy(c);
  if (G->pin) cudaFreeHost(G->pin);
  delete G;
  return TTAGG_OK;
}

int ttagg_group_size(const ttagg_group* G, int* n) {
  if (!G || !n) return fail(TTAGG_ERR_ARG, "null argument");
  *n = G->n;
  return TTAGG_OK;
}

int ttagg_group_ctx(ttagg_group* G, int i, ttagg_ctx** out) {
  if (!G || !out) return fail(TTAGG_ERR_ARG, "null argument");
  if (i < 0 || i >= G->n) return fail(TTAGG_ERR_ARG, "device index outside the group");
  *out = G->ctx[i];
  return TTAGG_OK;
}

int ttagg_group_rhs(ttagg_group* G, const ttagg_kernel* const* kernels, int n_kernels, const double* n, double* p,
                    double* q, double* s) {
  if (!G || !kernels || !n) return fail(TTAGG_ERR_ARG, "null argument");
  if (n_kernels < 1) return fail(TTAGG_ERR_EMPTY, "no collision orders configured");
  std::lock_guard<std::mutex> lock(G->mu);
  Geom g;
  bool any = false;
  std::vector<std::vector<const ttagg_kernel*>> ks(G->n);
  for (int i = 0; i < G->n; ++i) {
    Geom gi;
    TRY(group_kernels(G, kernels, n_kernels, i, ks[i], &gi));
    if (ks[i].empty()) continue;
    if (any && gi.N != g.N) return fail(TTAGG_ERR_SIZE, "kernel shards disagree on N");
    g = gi;
    any = true;
  }
  if (!any) return fail(TTAGG_ERR_EMPTY, "no collision orders configured");
  for (int64_t j = 0; j < g.N; ++j)  // ConcentrationState's check (rhs.py:71-72)
    if (!std::isfinite(n[j])) return fail(TTAGG_ERR_NONFINITE, "concentration state contains non-finite entries");
  const int64_t Na = (g.N + 31) & ~(int64_t)31;
  const size_t nb = (size_t)g.N * sizeof(double);
  // page-locked buffers are transferred directly; pageable ones through the
  // group's staging area [n][p][q][s]
  double* outs[3] = {p, q, s};
  bool stage = !is_pinned(n);
  for (double* o : outs) stage |= (o && !is_pinned(o));
  if (stage && G->pin_bytes < 4 * Na * sizeof(double)) {
    if (G->pin) cudaFreeHost(G->pin);
    G->pin = nullptr;
    G->pin_bytes = 0;
    CUDA_TRY(cudaHostAlloc((void**)&G->pin, 4 * Na * sizeof(double), cudaHostAllocDefault));
    G->pin_bytes = 4 * Na * sizeof(double);
  }
  const double* nsrc = n;
  if (!is_pinned(n)) {
    par_copy(G->pin, n, nb);
    nsrc = G->pin;
  }
  std::vector<double*> part(G->n);
  for (int i = 0; i < G->n; ++i) {
    ttagg_ctx* c = G->ctx[i];
    CUDA_TRY(cudaSetDevice(c->device));
    const size_t need = (size_t)4 * Na * sizeof(double);
    if (G->buf_bytes[i] < need) {
      cudaFree(G->buf[i]);
      G->buf[i] = nullptr;
      G->buf_bytes[i] = 0;
      CUDA_TRY(cudaMalloc(&G->buf[i], need));
      G->buf_bytes[i] = need;
    }
    double* nd = G->buf[i];
    part[i] = nd + Na;  // [p][q][s], contiguous: one all-reduce
    if (ks[i].empty()) {
      CUDA_TRY(cudaMemsetAsync(part[i], 0, 3 * Na * sizeof(double), G->st[i]));
      continue;
    }
    CUDA_TRY(cudaMemcpyAsync(nd, nsrc, nb, cudaMemcpyHostToDevice, G->st[i]));
    TRY(ttagg_rhs(c, ks[i].data(), (int)ks[i].size(), nd, part[i], part[i] + Na, part[i] + 2 * Na,
                  TTAGG_WANT_P | TTAGG_WANT_Q, G->st[i]));
  }
  TRY(group_allreduce(G, part, 3 * (size_t)Na));
  CUDA_TRY(cudaSetDevice(G->ctx[0]->device));
  for (int j = 0; j < 3; ++j)
    if (outs[j])
      CUDA_TRY(cudaMemcpyAsync(is_pinned(outs[j]) ? outs[j] : G->pin + (size_t)(j + 1) * Na, part[0] + (size_t)j * Na,
                               nb, cudaMemcpyDeviceToHost, G->st[0]));
  for (int i = 0; i < G->n; ++i) {
    CUDA_TRY(cudaSetDevice(G->ctx[i]->device));
    CUDA_TRY(cudaStreamSynchronize(G->st[i]));
  }
  for (int j = 0; j < 3; ++j)
    if (outs[j] && !is_pinned(outs[j])) par_copy(outs[j], G->pin + (size_t)(j + 1) * Na, nb);
  return TTAGG_OK;
}

int ttagg_group_rk2(ttagg_group* G, const ttagg_kernel* const* kernels, int n_kernels, double* n_inout, double t0,
                    double dt, int64_t steps, int64_t record_every, double* records, int64_t* fail_step,
                    int64_t* neg_step) {
  if (!G || !kernels || !n_inout || !records || !fail_step || !neg_step) return fail(TTAGG_ERR_ARG, "null argument");
  if (!(dt > 0)) return fail(TTAGG_ERR_ARG, "dt must be positive");
  if (steps < 1 || record_every < 1) return fail(TTAGG_ERR_ARG, "steps and record_every must be >= 1");
  if (n_kernels < 1) return fail(TTAGG_ERR_EMPTY, "no collision orders configured");
  std::lock_guard<std::mutex> lock(G->mu);
  Geom g;
  bool any = false;
  std::vector<std::vector<const ttagg_kernel*>> ks(G->n);
  for (int i = 0; i < G->n; ++i) {
    Geom gi;
    TRY(group_kernels(G, kernels, n_kernels, i, ks[i], &gi));
    if (ks[i].empty()) continue;
    if (any && gi.N != g.N) return fail(TTAGG_ERR_SIZE, "kernel shards disagree on N");
    g = gi;
    any = true;
  }
  if (!any) return fail(TTAGG_ERR_EMPTY, "no collision orders configured");
  for (int64_t j = 0; j < g.N; ++j)
    if (!std::isfinite(n_inout[j])) return fail(TTAGG_ERR_NONFINITE, "concentration state contains non-finite entries");
  const int64_t nrows = steps / record_every + 1;
  const int64_t Na = (g.N + 31) & ~(int64_t)31;
  const size_t nb = (size_t)g.N * sizeof(double);
  const int nblk = (int)((g.Np + 255) / 256);
  // per device: [nat Na][A Np][B Np][C Np][s Np]; device 0 also [rec nrows*4]
  std::vector<double*> vA(G->n), vB(G->n), vC(G->n), vS(G->n);
  for (int i = 0; i < G->n; ++i) {
    ttagg_ctx* c = G->ctx[i];
    CUDA_TRY(cudaSetDevice(c->device));
    const size_t need = (size_t)(Na + 4 * g.Np + (i == 0 ? nrows * 4 : 0)) * sizeof(double) + 1024;
    if (G->buf_bytes[i] < need) {
      cudaFree(G->buf[i]);
      G->buf[i] = nullptr;
      G->buf_bytes[i] = 0;
      CUDA_TRY(cudaMalloc(&G->buf[i], need));
      G->buf_bytes[i] = need;
    }
    double* nat = G->buf[i];
    vA[i] = nat + Na;
    vB[i] = vA[i] + g.Np;
    vC[i] = vB[i] + g.Np;
    vS[i] = vC[i] + g.Np;
    CUDA_TRY(cudaMemcpyAsync(nat, n_inout, nb, cudaMemcpyHostToDevice, G->st[i]));
    TRY(launch_permute(nat, vA[i], g, 0, G->st[i]));
  }
  ttagg_ctx* c0 = G->ctx[0];
  cudaStream_t s0 = G->st[0];
  double* rec = vS[0] + g.Np;
  CUDA_TRY(cudaSetDevice(c0->device));
  TRY(ensure((void**)&c0->diagp, &c0->diagp_bytes, (size_t)2 * nblk * DIAGW * sizeof(double)));
  double* dpm = c0->diagp;
  double* dpn = c0->diagp + (size_t)nblk * DIAGW;
  double* dmid = c0->diag;
  double* dnew = c0->diag + DIAGW;
  double* d0 = c0->diag + 2 * DIAGW;
  stage_kernel<<<nblk, 256, 0, s0>>>(vA[0], vA[0], 0.0, nullptr, g.N, g.N1, g.N2, dpn);
  diag_finalize_kernel<<<1, 256, 0, s0>>>(dpn, nblk, d0);
  rk2_book_init_kernel<<<1, 32, 0, s0>>>(d0, c0->book, rec);
  CUDA_TRY(cudaGetLastError());
  // partial RHS at x (perm) into vS on every device, then the all-reduce
  auto rhs = [&](const std::vector<double*>& x) -> int {
    for (int i = 0; i < G->n; ++i) {
      ttagg_ctx* c = G->ctx[i];
      CUDA_TRY(cudaSetDevice(c->device));
      if (ks[i].empty()) {
        CUDA_TRY(cudaMemsetAsync(vS[i], 0, g.Np * sizeof(double), G->st[i]));
        continue;
      }
      TRY(ttagg_rhs_perm(c, ks[i].data(), (int)ks[i].size(), x[i], nullptr, 0.0, vS[i], G->st[i]));
    }
    return group_allreduce(G, vS, (size_t)g.Np);
  };
  // out = base + a s on every device; diagnostics on device 0
  auto stage = [&](const std::vector<double*>& base, double a, const std::vector<double*>& out, double* dp,
                   double* dg) -> int {
    for (int i = 0; i < G->n; ++i) {
      CUDA_TRY(cudaSetDevice(G->ctx[i]->device));
      stage_kernel<<<nblk, 256, 0, G->st[i]>>>(base[i], vS[i], a, out[i], g.N, g.N1, g.N2, i == 0 ? dp : nullptr);
      if (i == 0) diag_finalize_kernel<<<1, 256, 0, G->st[i]>>>(dp, nblk, dg);
      CUDA_TRY(cudaGetLastError());
    }
    return TTAGG_OK;
  };
  std::vector<double*> cur = vA, mid = vB, nxt = vC;
  int64_t host_book[4] = {0, 0, 0, 0};
  for (int64_t step = 1; step <= steps; ++step) {
    TRY(rhs(cur));
    TRY(stage(cur, 0.5 * dt, mid, dpm, dmid));
    TRY(rhs(mid));
    TRY(stage(cur, dt, nxt, dpn, dnew));
    CUDA_TRY(cudaSetDevice(c0->device));
    rk2_book_kernel<<<1, 32, 0, s0>>>(dmid, dnew, c0->book, record_every, rec);
    CUDA_TRY(cudaGetLastError());
    std::swap(cur, nxt);
    if (step % 64 == 0 || step == steps) {
      CUDA_TRY(cudaMemcpyAsync(host_book, c0->book, sizeof(host_book), cudaMemcpyDeviceToHost, s0));
      CUDA_TRY(cudaStreamSynchronize(s0));
      if (host_book[1] != 0) break;
    }
  }
  CUDA_TRY(cudaSetDevice(c0->device));
  CUDA_TRY(cudaMemcpyAsync(host_book, c0->book, sizeof(host_book), cudaMemcpyDeviceToHost, s0));
  TRY(launch_permute(cur[0], G->buf[0], g, 1, s0));
  std::vector<double> hrec((size_t)nrows * 4);
  CUDA_TRY(cudaMemcpyAsync(hrec.data(), rec, hrec.size() * sizeof(double), cudaMemcpyDeviceToHost, s0));
  CUDA_TRY(cudaMemcpyAsync(n_inout, G->buf[0], nb, cudaMemcpyDeviceToHost, s0));
  for (int i = 0; i < G->n; ++i) {
    CUDA_TRY(cudaSetDevice(G->ctx[i]->device));
    CUDA_TRY(cudaStreamSynchronize(G->st[i]));
  }
  const int64_t rows = std::min<int64_t>(host_book[3], nrows);
  std::vector<double> outr((size_t)nrows * 5, 0.0);
  double t = t0;
  int64_t row = 0;
  for (int64_t stp = 0; row < rows; ++stp) {
    if (stp > 0) t = t + dt;
    if (stp % record_every == 0) {
      outr[row * 5] = t;
      for (int cc = 0; cc < 4; ++cc) outr[row * 5 + 1 + cc] = hrec[row * 4 + cc];
      ++row;
    }
  }
  std::memcpy(records, outr.data(), outr.size() * sizeof(double));
  *fail_step = host_book[1];
  *neg_step = host_book[2];
  return TTAGG_OK;
}

}  // extern "C"
