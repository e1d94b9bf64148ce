/*
 * ttagg_b200 — C-ABI of the B200-native right-hand-side evaluator for the
 * multi-particle Smoluchowski equations (arXiv 1905.09071, reference package
 * `ttagg` v0.1.0).
 *
 * The reference has no FFI: its boundary is the Python operator API
 * (pkg/src/ttagg/rhs.py, integrator.py).  Every entry point below replaces
 * one piece of that API; the citation next to each names the reference
 * function it stands in for.  All arithmetic is IEEE fp64.  No C++ types,
 * no torch types: plain pointers, sizes and a CUDA stream passed as void*.
 *
 * Conventions
 *   - Every call returns int status (TTAGG_OK == 0).  On failure
 *     ttagg_last_error() (thread-local) holds a message.  No exceptions
 *     cross the ABI.
 *   - "device" pointers are CUDA device pointers on the context's device;
 *     "host" pointers are ordinary host memory.  Which one a call takes is
 *     stated per call (flag TTAGG_HOST_PTRS switches ttagg_rhs / ttagg_rk2).
 *   - The "perm" layout of a length-N vector is the transposed view used by
 *     the kernels: element o = n1*N2 + n2 (size o+1) is stored at
 *     n2*N1 + n1 of a buffer of length Np (zero padded).  ttagg_geometry()
 *     reports Np, N1, N2 for a given N.
 */
#ifndef TTAGG_B200_H
#define TTAGG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTAGG_OK 0
#define TTAGG_ERR_ARG 1         /* bad argument or shape   (kernels.py:147-164, 193-203) */
#define TTAGG_ERR_SIZE 2        /* N mismatch              (rhs.py:178-183, 436-439)    */
#define TTAGG_ERR_EMPTY 3       /* no collision orders     (rhs.py:434-435)             */
#define TTAGG_ERR_NONFINITE 4   /* non-finite state        (rhs.py:71-72)               */
#define TTAGG_ERR_CUDA 5        /* CUDA runtime failure                                  */
#define TTAGG_ERR_UNSUPPORTED 6 /* size or rank outside what this build handles          */
#define TTAGG_ERR_NOMEM 7       /* device allocation failed                              */
#define TTAGG_ERR_NCCL 8        /* NCCL failure (device groups)                          */

/* flags */
#define TTAGG_HOST_PTRS 1 /* n/p/q/s (rhs) or n/records (rk2) are host pointers      */
#define TTAGG_WANT_P 2    /* compute the gain P                                       */
#define TTAGG_WANT_Q 4    /* compute the loss Q                                       */

#define TTAGG_KIND_CP 1
#define TTAGG_KIND_TT 2
#define TTAGG_KIND_DENSE 3

typedef struct ttagg_ctx ttagg_ctx;       /* one per CUDA device (workspaces, tables) */
typedef struct ttagg_kernel ttagg_kernel; /* one uploaded collision kernel of order d */

/* version as 10000*major + 100*minor + patch */
int ttagg_version(void);
const char* ttagg_last_error(void);

/* Size-class geometry for N: writes {Np, N1, N2}.  Np = padded length. */
int ttagg_geometry(int64_t n_classes, int64_t* out3);

int ttagg_ctx_create(int device, ttagg_ctx** out);
int ttagg_ctx_destroy(ttagg_ctx* ctx);

/* Upload a CP kernel (replaces CPKernel, kernels.py:183-215, plus the
 * weighting layout of rhs_cp_P, rhs.py:361-369).  factors: d host pointers,
 * each an N x R row-major fp64 matrix (the reference's factor layout).
 * rank_subset (nullable): the rank indices this context owns, for rank
 * sharding across GPUs; n_subset entries. */
int ttagg_cp_upload(ttagg_ctx* ctx, int d, int64_t n_classes, int64_t rank,
                    const double* const* factors, const int64_t* rank_subset,
                    int64_t n_subset, ttagg_kernel** out);

/* Opt-in variant (no reference counterpart): identical
 * factor columns (bitwise) are stored and transformed once — every distinct
 * ordered pair of columns gets one exchange slot that pass B reads for each
 * pair mapping to it, identical tail columns share one row.  Same results
 * as ttagg_cp_upload (the rank/mode structure is unchanged); for kernels
 * built from few distinct vectors (the permutation-power and Brownian
 * families) the column transforms shrink accordingly. */
int ttagg_cp_upload_dedup(ttagg_ctx* ctx, int d, int64_t n_classes, int64_t rank,
                          const double* const* factors, const int64_t* rank_subset,
                          int64_t n_subset, ttagg_kernel** out);

/* Upload a TT kernel (replaces TTKernel, kernels.py:137-180, plus the fiber
 * layout of rhs_tt_P, rhs.py:256-269).  ranks: d+1 entries with
 * ranks[0] == ranks[d] == 1; cores: d host pointers, core l of shape
 * (ranks[l], N, ranks[l+1]) row-major.  Only live fibers are uploaded:
 * identically zero fibers and fibers on chain paths that are zero add
 * nothing to the gain or the loss and are dropped. */
int ttagg_tt_upload(ttagg_ctx* ctx, int d, int64_t n_classes, const int64_t* ranks,
                    const double* const* cores, ttagg_kernel** out);

/* Upload a dense kernel (replaces DenseKernel, kernels.py:218-238, for the
 * direct-summation operators rhs_dense_P / rhs_dense_Q, rhs.py:202-227).
 * values: host pointer to N^d fp64 coefficients in row-major index order;
 * N^d must not exceed 2^26 (DENSE_RHS_BUDGET, rhs.py:47).  Dense orders take
 * part in ttagg_rhs / ttagg_rk2 like CP and TT orders (single GPU). */
int ttagg_dense_upload(ttagg_ctx* ctx, int d, int64_t n_classes, const double* values,
                       ttagg_kernel** out);

int ttagg_kernel_free(ttagg_kernel* k);

/* info[0]=kind, [1]=d, [2]=N, [3]=columns (CP d*R_local / TT live fibers / dense 0),
 * [4]=Np, [5]=N1, [6]=N2, [7]=rows per column in the exchange */
int ttagg_kernel_info(const ttagg_kernel* k, int64_t* info8);

/* dn/dt over a set of orders — replaces rhs_total (rhs.py:421-459); with a
 * single kernel and flags WANT_P or WANT_Q it replaces rhs_cp_P / rhs_cp_Q /
 * rhs_tt_P / rhs_tt_Q (rhs.py:234-414).  n: length-N state.  p, q, s:
 * length-N outputs, each nullable (p = sum of gains, q = sum of losses,
 * s = p + q).  flags: TTAGG_HOST_PTRS | TTAGG_WANT_P | TTAGG_WANT_Q (neither
 * WANT bit means both).  stream: cudaStream_t or NULL. */
int ttagg_rhs(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels,
              const double* n, double* p, double* q, double* s, int flags, void* stream);

/* Engine-level pieces for the multi-GPU (rank-sharded) path, device
 * pointers in the perm layout.  s_perm = partial RHS at state
 * n_perm + alpha * k_perm (k_perm nullable), over this context's rank
 * shard; all-reduce across GPUs is the caller's (NCCL via torch.distributed). */
int ttagg_rhs_perm(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels,
                   const double* n_perm, const double* k_perm, double alpha,
                   double* s_perm, void* stream);

/* natural <-> perm layout (dir 0: natural -> perm, 1: perm -> natural) */
int ttagg_permute(ttagg_ctx* ctx, int64_t n_classes, const double* in, double* out, int dir,
                  void* stream);

/* RK2 stage update in perm layout — the state updates of midpoint_step
 * (integrator.py:153-157) with the checks of rk2_step / integrate
 * (integrator.py:177-178, 216-223):  out = base + a * s.
 * diag (device, nullable, 8 doubles): [0] nonfinite flag (0/1),
 * [1] min(out), [2] max|out|, [3] M0, [4] M1, [5] M2 (moments of out, sizes
 * k = 1..N; integrator.py:141-150). */
int ttagg_stage(ttagg_ctx* ctx, int64_t n_classes, const double* base, const double* s,
                double a, double* out, double* diag, void* stream);

/* Whole explicit-midpoint trajectory on one GPU with the state resident in
 * HBM — replaces integrate / rk2_step (integrator.py:160-228).
 * n_inout: initial state in, final state out (length N).  records:
 * (steps / record_every + 1) x 5 rows of (t, M0, M1, M2, min_n), the first
 * row being the initial state.  fail_step: 0, or the first step whose
 * midpoint or final state was non-finite (integrator.py:207-215); rows after
 * the failure are not written.  neg_step: 0, or the first step with
 * min(n) < -1e-9 max|n| (integrator.py:216-223).  flags: TTAGG_HOST_PTRS
 * applies to n_inout and records. */
int ttagg_rk2(ttagg_ctx* ctx, const ttagg_kernel* const* kernels, int n_kernels,
              double* n_inout, double t0, double dt, int64_t steps, int64_t record_every,
              double* records, int64_t* fail_step, int64_t* neg_step, int flags,
              void* stream);

/* Per-launch timing for the roofline report: after
 * ttagg_profile_enable(ctx, 1) every launch issued by ttagg_rhs / ttagg_rhs_perm
 * is bracketed by CUDA events on its stream.  ttagg_profile_read fills
 * out72[(cls*9 + d)*2 + {0: milliseconds, 1: launches}] accumulated since
 * the last read; cls 0 = pass A (column FFTs), 1 = pass B (row FFTs +
 * spectral product), 2 = pass C (inverse column FFTs), 3 = other (loss
 * coefficients, combine); d = collision order (0 for order-free launches). */
int ttagg_profile_enable(ttagg_ctx* ctx, int on);
int ttagg_profile_read(ttagg_ctx* ctx, double* out72);

/* Number of kernel launches this context has issued from ttagg_rhs /
 * ttagg_rhs_perm (monotone counter; the bench reports the difference). */
int ttagg_launch_count(ttagg_ctx* ctx, int64_t* out);

/* Debug (no reference counterpart): with on = 1 every scratch buffer the
 * context uses (exchange, inverse rows, TT chain state, per-order gains,
 * column sums, loss coefficients) is filled with NaN bytes on the call's
 * stream before use, so any read of a value the call did not write first
 * shows up as a non-finite result.  The bounds/initialisation check that
 * stands in for compute-sanitizer initcheck (tests/test_gpu_guard.py). */
int ttagg_debug_poison(ttagg_ctx* ctx, int on);

/* Device group (single process, several GPUs; SURVEY.md §8(e), §8(b)'s
 * ttagg_ctx_create(devices, n)): one context per device plus an NCCL
 * communicator (ncclCommInitAll; libnccl.so.2 is loaded at run time, and a
 * one-device group needs none).  The caller uploads each device's kernel
 * shard (CP rank subsets, TT slices of the first internal rank; a dense
 * order on one device only) to ttagg_group_ctx(g, i) and passes them as an
 * n_dev x n_kernels row-major table (null: that device holds no share of the
 * order).  ttagg_group_rhs: host n in, host p/q/s out (each nullable), one
 * all-reduce of the partial [p q s] per call.  ttagg_group_rk2: same
 * contract as ttagg_rk2 with host pointers; per RHS one all-reduce of the
 * partial dn/dt, then every device applies the identical stage update to
 * its replica (integrator.py:153-228). */
typedef struct ttagg_group ttagg_group;
int ttagg_group_create(const int* devices, int n_dev, ttagg_group** out);
int ttagg_group_destroy(ttagg_group* g);
int ttagg_group_size(const ttagg_group* g, int* n_dev);
int ttagg_group_ctx(ttagg_group* g, int i, ttagg_ctx** out);
int ttagg_group_rhs(ttagg_group* g, const ttagg_kernel* const* kernels, int n_kernels,
                    const double* n, double* p, double* q, double* s);
int ttagg_group_rk2(ttagg_group* g, const ttagg_kernel* const* kernels, int n_kernels,
                    double* n_inout, double t0, double dt, int64_t steps, int64_t record_every,
                    double* records, int64_t* fail_step, int64_t* neg_step);

#ifdef __cplusplus
}
#endif

#endif /* TTAGG_B200_H */
