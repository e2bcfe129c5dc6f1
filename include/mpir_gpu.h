/*
 * mpir_gpu.h -- C-ABI of the B200 mixed-precision iterative-refinement (IR)
 * hot path: interprecision copy, low-precision LU with partial pivoting,
 * triangular solves, and the TR-precision residual.
 *
 * The reference (proj/ in arxiv/paper_2311_14616, "mpir") has no FFI layer of
 * its own: its boundary is the header-only C++ API
 *   MPFactorization<TW,TF,TR>   proj/include/mpir/mp_structures.hpp:97-213
 *   mp_lu / mp_refactor         proj/include/mpir/mp_structures.hpp:215-237
 *   ir_solve_report / ir_solve  proj/include/mpir/ir_engine.hpp:291-304
 *   residual_tr                 proj/include/mpir/ir_engine.hpp:277-287
 * plus the kernels it is built from (dense_lu.hpp, matrix.hpp). Every entry
 * point below names the reference function it replaces. The C++ twin of the
 * reference API (mpir_gpu.hpp) and the Python mirror of the reference module
 * (paper_2311_14616_b200/mpir.py) are thin layers over these symbols.
 *
 * Conventions
 *  - Matrices are n x n, column-major, leading dimension n (matrix.hpp:17-61).
 *  - Precision codes follow mpir::Precision (precision.hpp:20-25).
 *    B16 data is IEEE binary16 stored as uint16_t bits (half.hpp:25-192).
 *  - Every call returns an int status (MPIRG_OK or an MPIRG_ERR_* code that
 *    names the reference exception type, errors.hpp:14-94) and, when err is
 *    non-NULL, fills err with the exception payload.
 *  - Calls are synchronous, like the reference API. Kernel-level entry points
 *    take device pointers and a cudaStream_t passed as void* (NULL = the
 *    legacy default stream); they synchronise that stream before returning.
 *  - No torch types cross this boundary; there is no CPU fallback. A missing
 *    or unusable GPU yields MPIRG_ERR_CUDA.
 */
#ifndef MPIR_GPU_H
#define MPIR_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPIRG_ABI_VERSION 1

/* mpir::Precision, precision.hpp:20-25 */
enum mpirg_precision { MPIRG_B64 = 0, MPIRG_B32 = 1, MPIRG_B16 = 2 };

/* Status codes; one per reference exception type (errors.hpp:14-94). */
enum mpirg_status {
  MPIRG_OK = 0,
  MPIRG_ERR_OVERFLOW = 1,       /* OverflowDetected   (precision.hpp:177-180) */
  MPIRG_ERR_SINGULAR = 2,       /* SingularPivot{column} (dense_lu.hpp:76-77) */
  MPIRG_ERR_NONFINITE = 3,      /* NonFiniteResult{rhist,dhist} (ir_engine.hpp:217-231) */
  MPIRG_ERR_DIMENSION = 4,      /* DimensionMismatch */
  MPIRG_ERR_INVALID_CONFIG = 5, /* InvalidConfig      (precision.hpp:222-230) */
  MPIRG_ERR_INVALID_PARAM = 6,  /* InvalidParameter   (ir_engine.hpp:29-47) */
  MPIRG_ERR_INVALID_SIZE = 7,   /* InvalidSize        (matrix.hpp:24-28) */
  MPIRG_ERR_CUDA = 8,           /* CUDA runtime failure (no reference analogue) */
  MPIRG_ERR_NCCL = 9            /* NCCL failure (no reference analogue) */
};

/* mpir::StopReason, ir_engine.hpp:66-90 */
enum mpirg_stop_reason {
  MPIRG_SMALL_RESIDUAL = 0,
  MPIRG_SMALL_BACKWARD_ERROR = 1,
  MPIRG_RESIDUAL_STAGNATION = 2,
  MPIRG_CORRECTION_STAGNATION = 3,
  MPIRG_ITERATION_LIMIT = 4
};

/* LU arithmetic mode. EXACT reproduces lu_inplace (dense_lu.hpp:50-109)
 * bit for bit for every factor precision. TC is the fp16 tensor-core
 * trailing update (tcgen05, fp32 accumulation in TMEM, one rounding to fp16
 * per panel block); it is only valid for TF = B16 and is tolerance-checked,
 * not bitwise. */
enum mpirg_lu_mode { MPIRG_LU_EXACT = 0, MPIRG_LU_TC = 1 };

/* Exception payload. */
typedef struct mpirg_error {
  int status;        /* same as the return value */
  int column;        /* SingularPivot::column; -1 otherwise */
  double value;      /* OverflowDetected: the first offending value */
  char message[256]; /* the reference's what() text where it has one */
} mpirg_error;

/* PrecisionConfig (precision.hpp:210-231) + FactorOptions
 * (mp_structures.hpp:82-90) + device/tuning knobs. */
typedef struct mpirg_config {
  int tw;         /* working precision (B64 or B32) */
  int tf;         /* factorization precision */
  int tr;         /* residual precision */
  int on_the_fly; /* -1: resolve like mp_structures.hpp:118-121; 0/1 explicit */
  int resid_term; /* FactorOptions::resid_term (default 1) */
  int lu_mode;    /* enum mpirg_lu_mode (default EXACT) */
  int nb;         /* LU panel width; 0 = automatic */
  int device;     /* CUDA device ordinal; -1 = current device */
} mpirg_config;

/* TermParams, ir_engine.hpp:29-47 (defaults cr=1, ce=1, rmax=0.5, litmax=10). */
typedef struct mpirg_term_params {
  double cr;
  double ce;
  double rmax;
  int litmax;
} mpirg_term_params;

/* SolveReport<TW>, ir_engine.hpp:96-105. The caller owns every buffer:
 * sol holds n values of TW (host or device memory per sol_on_device);
 * rhist/dhist hold hist_capacity doubles (capacity >= litmax suffices).
 * On MPIRG_ERR_NONFINITE the partial histories are written, like the
 * NonFiniteResult payload. */
typedef struct mpirg_report {
  void *sol;
  int sol_on_device;
  double *rhist;
  double *dhist;
  int hist_capacity;
  int rhist_len;
  int dhist_len;
  int reason;          /* enum mpirg_stop_reason */
  double solve_ms;     /* device time of the IR loop (CUDA events) */
} mpirg_report;

typedef struct mpirg_factorization mpirg_factorization;

/* ---------------------------------------------------------------------------
 * Library / config
 * ------------------------------------------------------------------------- */
int mpirg_abi_version(void);
/* Number of CUDA devices visible; 0 when no GPU (then every GPU call fails). */
int mpirg_device_count(void);
/* resolve_config (mp_structures.hpp:44-59): fills TF/TR/on_the_fly defaults.
 * Pass tf/tr/on_the_fly = -1 for "not given". */
int mpirg_resolve_config(int tw, int tf, int tr, int on_the_fly, mpirg_config *out,
                         mpirg_error *err);
/* update_parms (ir_engine.hpp:49-64). NaN in a field = "not given"; litmax<=0 not given. */
int mpirg_update_parms(double cr, double ce, double rmax, int litmax,
                       mpirg_term_params *out, mpirg_error *err);
double mpirg_machine_eps(int precision);   /* precision.hpp:43-54 */
double mpirg_unit_roundoff(int precision); /* precision.hpp:28-39 */

/* ---------------------------------------------------------------------------
 * MPFactorization<TW,TF,TR> (mp_structures.hpp:97-213)
 * ------------------------------------------------------------------------- */
/* Constructor: takes a copy of the TW matrix a (host or device memory), then
 * refactor(): one-norm of a_high in TW, demotion into the factor storage with
 * overflow/underflow checks, LU in place. a == NULL allocates only (no
 * factorization yet: call refactor or cast + set_factored before solving). */
int mpirg_factorization_create(mpirg_factorization **out, int n, const mpirg_config *cfg,
                               const void *a, int a_on_device, mpirg_error *err);
/* refactor(const Matrix<TW>&) (mp_structures.hpp:155-169). a == NULL
 * refactors the resident a_high (the reference's self-refactor, no copy).
 * Every device buffer is reused; pointers stay stable. */
int mpirg_factorization_refactor(mpirg_factorization *f, const void *a, int a_on_device,
                                 mpirg_error *err);
void mpirg_factorization_destroy(mpirg_factorization *f);

int mpirg_factorization_n(const mpirg_factorization *f);
int mpirg_factorization_config(const mpirg_factorization *f, mpirg_config *out);
double mpirg_factorization_a_norm1(const mpirg_factorization *f);
int mpirg_factorization_demotion_underflowed(const mpirg_factorization *f);
size_t mpirg_factorization_matrix_bytes(const mpirg_factorization *f);
/* Device time (ms) of the last refactor: one-norm + demotion + LU. */
double mpirg_factorization_last_factor_ms(const mpirg_factorization *f);
/* Host copies of the factor state (lazy device->host mirrors). */
int mpirg_factorization_get_ipiv(const mpirg_factorization *f, int *ipiv);
int mpirg_factorization_get_pivots(const mpirg_factorization *f, int *perm);
int mpirg_factorization_get_packed_lu(const mpirg_factorization *f, void *out_tf);
int mpirg_factorization_get_a_high(const mpirg_factorization *f, void *out_tw);
/* Stable device pointers (column-major n x n). */
const void *mpirg_factorization_a_high_device(const mpirg_factorization *f);
const void *mpirg_factorization_packed_lu_device(const mpirg_factorization *f);
const int *mpirg_factorization_ipiv_device(const mpirg_factorization *f);
/* Preallocated solver state (mp_structures.hpp:186-192: residual_buf, sol_buf,
 * comp_buf, low_buf, work_buf) as stable device pointers, n values each of
 * TR / TR / TR / TF / TW. The refinement loop owns them during a solve.
 * comp_buf is scratch only (the device residual keeps its compensation in
 * registers); low_buf and work_buf alias the one substitution scratch. */
void *mpirg_factorization_residual_buf_device(mpirg_factorization *f);
void *mpirg_factorization_sol_buf_device(mpirg_factorization *f);
void *mpirg_factorization_comp_buf_device(mpirg_factorization *f);
void *mpirg_factorization_low_buf_device(mpirg_factorization *f);
void *mpirg_factorization_work_buf_device(mpirg_factorization *f);
/* The CUDA stream every call on this handle runs on (cudaStream_t). */
void *mpirg_factorization_stream(const mpirg_factorization *f);

/* ir_solve_report(f, b, tp) (ir_engine.hpp:291-297, loop 186-271). b holds n
 * values of TW. tp == NULL uses the defaults. */
int mpirg_ir_solve(mpirg_factorization *f, const void *b, int b_on_device,
                   const mpirg_term_params *tp, mpirg_report *rep, mpirg_error *err);
/* Krylov corrections (krylov_ir.hpp:62-171, 297-318): MPFactorization's
 * KrylovKind / basissize constructor arguments (mp_structures.hpp:108-151) as a
 * call on an existing handle. With GMRES enabled, mpirg_ir_solve is
 * krylov_ir_solve_report: each correction is one left-preconditioned GMRES
 * solve (modified Gram-Schmidt, Givens rotations, at most `basissize` basis
 * vectors, relative tolerance 1e-2) with the low-precision factors as the
 * preconditioner; with BiCGSTAB one left-preconditioned bi-conjugate gradient
 * stabilised solve (bicgstab_correction_into, 173-254: at most `basissize`
 * iterations, relative tolerance 0.1). Both bitwise equal to the reference's.
 * khist (inner iteration counts, one per correction) and the breakdown flag of
 * the last solve: _last_khist. */
enum mpirg_krylov_kind { MPIRG_KRYLOV_NONE = 0, MPIRG_KRYLOV_GMRES = 1, MPIRG_KRYLOV_BICGSTAB = 2 };
int mpirg_factorization_enable_krylov(mpirg_factorization *f, int kind, int basissize,
                                      mpirg_error *err);
int mpirg_factorization_last_khist(const mpirg_factorization *f, int *khist, int capacity,
                                   int *len, int *breakdown);
/* residual_tr(f, x, b) (ir_engine.hpp:277-287): r (n values of TR) = b - A x,
 * x and b in TW. Host or device buffers per on_device. */
int mpirg_residual_tr(mpirg_factorization *f, const void *x, const void *b, void *r,
                      int on_device, mpirg_error *err);

/* ---------------------------------------------------------------------------
 * Kernel-level entry points (device pointers, explicit stream)
 * ------------------------------------------------------------------------- */
/* demote_matrix_into<To,From> (matrix.hpp:74-85) with demote_checked
 * (precision.hpp:172-185). Overflow is reported for the first offending
 * element in storage order; *underflow (optional) receives the sticky flag. */
int mpirg_demote(int from, int to, size_t count, const void *src, void *dst, int *underflow,
                 void *stream, mpirg_error *err);
/* matrix_one_norm<T> (mp_structures.hpp:22-36), accumulated in T. */
int mpirg_one_norm(int prec, int rows, int cols, const void *a, double *out, void *stream,
                   mpirg_error *err);
/* lu_factor / lu_factor_half (dense_lu.hpp:151-171): in-place LU of the
 * n x n matrix a (precision prec), ipiv[n] (device) receives the swap rows. */
int mpirg_lu_factor(int prec, int n, void *a, int *ipiv, int lu_mode, int nb, void *stream,
                    mpirg_error *err);
/* solve_mps_into<TS,TF> (dense_lu.hpp:175-182): in place on x (TS). */
int mpirg_solve_mps(int ts, int tf, int n, const void *packed, const int *ipiv, void *x,
                    void *stream, mpirg_error *err);
/* solve_lps_into<TW,TF> (dense_lu.hpp:204-232): in place on r_to_d (TW),
 * scratch holds n values of TF. */
int mpirg_solve_lps(int tw, int tf, int n, const void *packed, const int *ipiv, void *r_to_d,
                    void *scratch, int *underflow, void *stream, mpirg_error *err);
/* detail::residual_into<TW,TR> (ir_engine.hpp:115-139): r = b - A x in TR,
 * compensated; a, b in TW; x, r in TR. */
int mpirg_residual(int tw, int tr, int n, const void *a, const void *x, const void *b,
                   void *r, void *stream, mpirg_error *err);

/* One K5b tensor-core trailing update (lu_mode TC, binary16, nb = 64): for
 * the panel at column k0, A22[rows k0+64..n) x [cb, ce) = fp16(fp32(A22) -
 * L21 U12) with the 64-term product accumulated in fp32 on tcgen05.
 * a: n x n binary16 bits, column-major, n % 8 == 0. Exposed for testing. */
int mpirg_tc_update(int n, void *a, int k0, int cb, int ce, void *stream, mpirg_error *err);
/* The general K5b update the recursive tensor-core LU is built from:
 * A[r0:r1, cb:ce] = fp16(fp32(A[r0:r1, cb:ce]) - A[r0:r1, k0:k0+K] A[k0:k0+K, cb:ce]),
 * K a multiple of 64, ranges disjoint as in a right-looking LU
 * (k0 + K <= r0, k0 + K <= cb). Exposed for testing. */
int mpirg_tc_gemm(int n, void *a, int r0, int r1, int cb, int ce, int k0, int K, void *stream,
                  mpirg_error *err);

/* ---------------------------------------------------------------------------
 * Batched independent systems (BASELINE config 5b): count systems of size n,
 * each a separate MPFactorization<TW,TF,TR> + ir_solve_report with the same
 * termination parameters. a: count*n*n TW (system s at offset s*n*n);
 * b, sol: count*n TW. rhist/dhist: count*hist_capacity; lens/reasons: count.
 * Per-system errors are reported in status[count] (0 = ok) and the call
 * returns the first non-OK status.
 * ------------------------------------------------------------------------- */
int mpirg_batch_ir_solve(int count, int n, const mpirg_config *cfg, const void *a,
                         const void *b, int on_device, const mpirg_term_params *tp,
                         void *sol, double *rhist, double *dhist, int hist_capacity,
                         int *rhist_len, int *reason, int *status, double *device_ms,
                         mpirg_error *err);

/* ---------------------------------------------------------------------------
 * Config 5a: the 1-D block-cyclic LU across ranks.
 * One handle per rank (one process per GPU). Column block b (block_cols
 * columns, a power of two and a multiple of nb; <= 0 picks 512) lives on
 * rank b mod nranks. Each rank holds an n x n factor buffer `a` (TF,
 * column-major, ld n; B200's 180 GB holds the full fp32 matrix of N=65536
 * per GPU) of which it owns its column blocks. Per panel p:
 *   owner:   mpirg_dlu_panel -> mpirg_dlu_pack(msg)
 *   all:     broadcast msg (mpirg_dlu_msg_bytes(p) bytes) from the owner
 *   others:  mpirg_dlu_unpack(msg)
 *   all:     mpirg_dlu_update(part 1 = next panel's columns if owned, then
 *            part 2 = the rest on the handle's side stream; or part 0 = all)
 * The factors, pivots and moves are bit-identical to the single-GPU LU
 * (detail::lu_inplace, dense_lu.hpp:63-107) for every nranks. Reference: no
 * counterpart (the reference is single-process); the per-element order is
 * the blocked equivalence of SURVEY.md 8(c).
 * ------------------------------------------------------------------------- */
typedef struct mpirg_dlu mpirg_dlu;
int mpirg_dlu_create(mpirg_dlu **out, int prec, int n, int nb, int nranks, int rank,
                     int block_cols, int device, mpirg_error *err);
void mpirg_dlu_destroy(mpirg_dlu *h);
int mpirg_dlu_nb(const mpirg_dlu *h);
int mpirg_dlu_npanels(const mpirg_dlu *h);
int mpirg_dlu_block_cols(const mpirg_dlu *h);
int mpirg_dlu_owner(const mpirg_dlu *h, int p);
size_t mpirg_dlu_msg_bytes(const mpirg_dlu *h, int p);
/* perm (optional, device int[n]) receives the row permutation (rank 0). */
int mpirg_dlu_begin(mpirg_dlu *h, int *perm, void *stream, mpirg_error *err);
int mpirg_dlu_panel(mpirg_dlu *h, void *a, int p, int *ipiv, void *stream, mpirg_error *err);
int mpirg_dlu_pack(mpirg_dlu *h, const void *a, int p, const int *ipiv, void *msg,
                   void *stream, mpirg_error *err);
int mpirg_dlu_unpack(mpirg_dlu *h, void *a, int p, int *ipiv, const void *msg, void *stream,
                     mpirg_error *err);
int mpirg_dlu_update(mpirg_dlu *h, void *a, int p, int part, int *perm, void *stream,
                     mpirg_error *err);
/* Joins the side stream into `stream`, synchronises, and returns the first
 * exactly-zero pivot column seen by this rank (-1 = none). */
int mpirg_dlu_end(mpirg_dlu *h, void *stream, int *singular_col, mpirg_error *err);

/* The whole LU of this rank in one call, driven from C++ (no host round trip
 * between a panel and its broadcast). `bcast` broadcasts `bytes` bytes of
 * device memory at buf from rank `root`, ordered on `stream` (cudaStream_t);
 * it is called once per panel, in panel order, on every rank, and returns 0
 * on success. mpirg_comm_bcast (NCCL) is the product hook; tests pass a
 * host-staged gloo broadcast. binary32 factors at nb = 64 use the single-GPU
 * LU's TMA-fed paired-step update on the rank's columns. nranks == 1 may
 * pass bcast = NULL. Results are bit-identical to mpirg_lu_factor. */
typedef int (*mpirg_bcast_fn)(void *ctx, void *buf, size_t bytes, int root, void *stream);
int mpirg_dlu_factor(mpirg_dlu *h, void *a, int *ipiv, int *perm, mpirg_bcast_fn bcast,
                     void *ctx, void *stream, int *singular_col, mpirg_error *err);

/* NCCL communicator for the hook above: one per rank, made from a 128-byte
 * unique id created on one rank (mpirg_comm_unique_id) and handed to the
 * others by the host side. NCCL is bound at run time (libnccl.so.2). */
typedef struct mpirg_comm mpirg_comm;
int mpirg_comm_unique_id(void *id128, mpirg_error *err);
int mpirg_comm_create(mpirg_comm **out, int nranks, int rank, const void *id128, int device,
                      mpirg_error *err);
void mpirg_comm_destroy(mpirg_comm *c);
int mpirg_comm_nranks(const mpirg_comm *c);
int mpirg_comm_rank(const mpirg_comm *c);
int mpirg_comm_version(void); /* NCCL version code, 0 when NCCL is not loadable */
int mpirg_comm_bcast(void *comm, void *buf, size_t bytes, int root, void *stream);
int mpirg_comm_send(mpirg_comm *c, const void *buf, size_t bytes, int peer, void *stream);
int mpirg_comm_recv(mpirg_comm *c, void *buf, size_t bytes, int peer, void *stream);

/* A handle whose LU is computed elsewhere (the distributed LU on rank 0):
 * _cast runs MPFactorization::refactor up to and including the demotion
 * (A_F in the handle's factor buffer, ||A||_1, overflow/underflow checks);
 * _buffers exposes the device factor buffer, ipiv, perm and stream;
 * _set_factored validates the external factorization (SingularPivot). */
int mpirg_factorization_cast(mpirg_factorization *f, const void *a, int a_on_device,
                             mpirg_error *err);
int mpirg_factorization_buffers(mpirg_factorization *f, void **a_low, int **ipiv, int **perm,
                                void **stream);
int mpirg_factorization_set_factored(mpirg_factorization *f, int singular_col,
                                     mpirg_error *err);

/* ---------------------------------------------------------------------------
 * Measurement hooks (bench.py): per-kernel-class CUDA-event timing and an
 * FP32 FFMA peak microbenchmark (the roofline denominator of the fp32 LU
 * trailing update, which may not use tensor cores).
 * ------------------------------------------------------------------------- */
enum mpirg_kernel_class {
  MPIRG_K_CAST = 0,       /* K1 cast + one-norm */
  MPIRG_K_PANEL = 1,      /* K2 panel factorization (cluster) */
  MPIRG_K_MOVES = 2,      /* K3 row moves (laswp gather) */
  MPIRG_K_TRSM = 3,       /* K4 U12 = L11^-1 A12 */
  MPIRG_K_GEMM = 4,       /* K5 trailing update */
  MPIRG_K_TRSV_LOWER = 5, /* K6 forward substitution (+LPS/MPS prologue) */
  MPIRG_K_TRSV_UPPER = 6, /* K6 back substitution (+IR epilogue) */
  MPIRG_K_RESIDUAL = 7,   /* K7 compensated residual */
  MPIRG_K_VECTOR = 8,     /* K8 small vector kernels */
  MPIRG_K_COUNT = 9
};
void mpirg_profile_enable(int on);
int mpirg_profile_collect(double *ms, int *count, int nclass);
/* Runs a pure-FFMA kernel on the current device; *tflops = achieved fp32 FMA
 * rate (2 flops per FFMA), *ms = its duration. */
int mpirg_ffma_peak(double *tflops, double *ms);
/* The same for binary64 DFMA (the roofline denominator of the fp64 chains:
 * residual and one-norm at small n, where rows/columns < lanes x SMSPs). */
int mpirg_dfma_peak(double *tflops, double *ms);
/* Dependent-chain latency of one FMA in cycles (MPIRG_B64 / MPIRG_B32): the
 * per-column floor of the residual's and the substitutions' row chains. */
int mpirg_fma_latency(int prec, double *cycles);
/* Diagnostics: the binary32 trailing update (lu_f32.cuh gemm_tma_kernel) of
 * rows/columns [K, n) by K <= 128 steps on a zeroed n x n matrix, tile edge
 * `tile` (128, 64, or 0 = the LU's own choice), averaged over `reps` launches;
 * *tflops counts 2 (n-K)^2 K flops per launch. */
int mpirg_ubench_gemm_f32(int n, int K, int tile, int reps, double *tflops, double *ms);
/* Diagnostics: compares the reciprocal-based division used on the back
 * substitution's critical path (common.cuh div_rcp) with IEEE div.rn on
 * `count` seeded operand pairs of precision `prec` (MPIRG_B64 / MPIRG_B32);
 * *mismatches = differing results, example[0..1] = one offending (a, b). */
int mpirg_check_fast_div(int prec, unsigned long long seed, long long count,
                         long long *mismatches, double *example);

/* ---------------------------------------------------------------------------
 * Seeded input generators (host; not on the timed path). See problems.cpp.
 * ------------------------------------------------------------------------- */
void mpirg_gen_uniform_matrix(int rows, int cols, uint64_t seed, double lo, double hi,
                              double *out);
void mpirg_gen_normal_matrix(int rows, int cols, uint64_t seed, double *out);
void mpirg_gen_diag_dominant(int n, uint64_t seed, double shift, double *out);
void mpirg_gen_greens_operator(int n, double alpha, double *out);
void mpirg_gen_integral_rhs(int n, double alpha, double *out);
/* The same operator generated on the device (greens.cpp:11-59, bitwise):
 * columns [col0, col0 + ncols) of I - alpha G into out (device memory,
 * column-major, leading dimension ld >= n). Lets config 5a's 34 GB matrix --
 * or one rank's column blocks of it -- be built in HBM directly. */
int mpirg_gen_greens_operator_device(int n, double alpha, int col0, int ncols, double *out,
                                     size_t ld, void *stream);
void mpirg_gen_matvec_compensated_f64(int n, const double *a, const double *x, double *y);

#ifdef __cplusplus
}
#endif

#endif /* MPIR_GPU_H */
