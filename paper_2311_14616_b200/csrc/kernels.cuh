// Launcher declarations for the IR hot-path kernels (host side).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace mpirg
{

struct CudaError : std::runtime_error
{
  cudaError_t code;
  CudaError(cudaError_t c, const char *expr, const char *file, int line)
    : std::runtime_error(std::string(cudaGetErrorString(c)) + " in " + expr + " at " + file +
                         ":" + std::to_string(line)),
      code(c)
  {
  }
};

// One-time setup per CUDA device (cudaFuncSetAttribute is per device/context;
// mpirg_config.device and mpirg_dlu_create(device) let one process use
// several). Redoing the setup from two threads at once is harmless.
struct DeviceOnce
{
  std::atomic<unsigned long long> mask{0};
  static unsigned long long bit()
  {
    int d = 0;
    cudaGetDevice(&d);
    return 1ull << (d & 63);
  }
  bool needed() const { return (mask.load(std::memory_order_acquire) & bit()) == 0; }
  void done() { mask.fetch_or(bit(), std::memory_order_release); }
};

// True when a CUDA profiler/injection tool is attached to this process
// (ncu, nsys, compute-sanitizer set CUDA_INJECTION64_PATH or
// NV_COMPUTE_PROFILER_* / NV_SANITIZER_*): the LU then runs on plain streams
// with no green contexts and no CUDA graphs, so every kernel of the schedule
// is visible to the tool (prof.cu).
bool tool_attached();

// ---- profiling hooks (prof.cu) --------------------------------------------
enum KClass
{
  KC_CAST = 0,
  KC_PANEL,
  KC_MOVES,
  KC_TRSM,
  KC_GEMM,
  KC_TRSV_L,
  KC_TRSV_U,
  KC_RESID,
  KC_VEC
};
bool prof_on();
void prof_begin(int kind, cudaStream_t s);
void prof_end(int kind, cudaStream_t s);
struct ProfScope
{
  int k;
  cudaStream_t s;
  ProfScope(int k_, cudaStream_t s_) : k(k_), s(s_) { prof_begin(k, s); }
  ~ProfScope() { prof_end(k, s); }
};

// ---- K1: interprecision copy --------------------------------------------
// Elementwise demotion (matrix.hpp:74-85 + precision.hpp:172-185), any length.
void launch_demote(int from, int to, const void *src, void *dst, size_t count, DevInfo *info,
                   cudaStream_t s);
// Fused refactor prologue (mp_structures.hpp:161-163): one read of the TW
// matrix produces the TF copy, the column-sum one-norm in TW (bits of the
// double max in *norm_bits, which must be zeroed) and the demotion flags.
// cols columns starting at col_off of the rows x * column-major src (rows is
// also the leading dimension); storage-order indices stay global.
void launch_cast_norm(int from, int to, int rows, int cols, const void *src, void *dst,
                      unsigned long long *norm_bits, DevInfo *info, cudaStream_t s,
                      int col_off = 0, int ns = 1);
// ns > 1 (config 5b): ns systems stored back to back (rows*cols elements
// each), norm slot norm_bits[z] and error record info[z] per system.
void launch_one_norm(int prec, int rows, int cols, const void *src,
                     unsigned long long *norm_bits, cudaStream_t s);

// ---- K2-K5: blocked right-looking LU with partial pivoting --------------
struct LuWorkspace
{
  int n = 0;
  int nb = 0;
  int npanels = 0;
  int2 *moves = nullptr;  // [npanels][2*nb] (dst,src) row moves of each panel
  int *nmoves = nullptr;  // [npanels]
  void *side = nullptr;   // cudaStream_t: look-ahead side stream
  void *crit = nullptr;   // cudaStream_t of the critical-chain SM group (MPIRG_LU_GREEN) or null
  void *events = nullptr; // cudaEvent_t[3*npanels]
  int *pp = nullptr;      // [n] composed row map of a tall panel
  int2 *smv = nullptr;    // [2*nb] row moves of the tall panel's 8-column leaves
  int *snm = nullptr;     // [nb/8]
  int *zero = nullptr;    // one int, always 0 ("no row moves" for solve-only U12 launches)
  void *ut = nullptr;     // float[2*nb][n]: transposed U12 of two steps (binary32)
  // late columns (launch_lu_late): panel snapshots, per-chunk U12 copies,
  // per-chunk streams and events; sized for late_n
  void *lsnap = nullptr, *utl = nullptr, *lstreams = nullptr, *levents = nullptr;
  int late_n = 0, late_np = 0;
};
// Chooses the panel width for n and the factor precision (0 = auto).
int lu_choose_nb(int prec, int n, int requested);
void lu_workspace_alloc(LuWorkspace &ws, int prec, int n, int nb);
void lu_partition_allowed(bool on);  // thread-local: next workspaces use the SM partition
void lu_workspace_free(LuWorkspace &ws);
// In-place LU of the n x n column-major matrix a (precision prec). ipiv[k]
// receives the pivot row of step k (dense_lu.hpp:79); perm (optional) the
// accumulated permutation (row i of PA is row perm[i] of A). The first
// exactly-zero pivot column is recorded in info->singular_col.
// Columns that arrive while the LU runs (refactor from host memory): chunk c
// holds columns [lo[c], hi[c]) and is present (copied and cast) once event
// ready[c] has completed. It is brought up to date by the panel steps before
// join[c] on its own stream -- from snapshots of those panels, so the later
// row moves of the regular schedule cannot race with it -- and joins the
// regular schedule at step join[c] (even, <= its first panel - 2). Chunk 0
// must be present when the LU starts (join 0).
struct LuLate
{
  static constexpr int MAXCH = 24;
  int nch = 0;
  int lo[MAXCH], hi[MAXCH], join[MAXCH];
  void *ready[MAXCH];  // cudaEvent_t
};
// A low-priority stream on the SMs of the LU's bulk update (the whole device
// when the SMs are not partitioned): side work that must not take the SMs of
// the LU's critical chain.
cudaStream_t lu_bulk_stream_create();
// True when launch_lu_late can take (prec, lu_mode, n) (binary32 exact LU).
bool lu_late_supported(int prec, int lu_mode, int n);
void launch_lu_late(void *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                    cudaStream_t s, const LuLate &late);
void launch_lu(int prec, int lu_mode, void *a, int n, int *ipiv, int *perm, LuWorkspace &ws,
               DevInfo *info, cudaStream_t s);
// Config 5b: the binary32 LU of ns independent n x n systems stored back to
// back (a + z n^2, ipiv/perm + z n, moves + z np 128, nmoves + z np, info + z),
// one launch per step for the whole group (lu.cu).
bool lu_batched_supported(int prec, int n);
// ut: optional scratch of 64 x (n ns) floats (the transposed U12 of the
// current step) enabling the TMA-fed trailing update.
void launch_lu_batched_f32(float *a, int n, int ns, int *ipiv, int *perm, int2 *moves,
                           int *nmoves, DevInfo *info, cudaStream_t s, float *ut = nullptr);
// perm from ipiv for callers that only hold ipiv (standalone solves).
void launch_perm_from_ipiv(const int *ipiv, int n, int *perm, cudaStream_t s);

// K5b: tensor-core trailing update for binary16 factors (lu_tc.cu).
struct TcPlan
{
  alignas(64) unsigned char mapA[128];  // CUtensorMap: L21 boxes (64 rows x 64 k)
  alignas(64) unsigned char mapB[128];  // CUtensorMap: U12 boxes (64 k x 256 cols)
  alignas(64) unsigned char mapB128[128];  // 64 k x 128 cols
  alignas(64) unsigned char mapB64[128];   // 64 k x 64 cols
  void *a = nullptr;
  int n = 0;
};
bool tc_update_supported(int n, int nb);
void tc_plan_make(TcPlan &p, void *a, int n);
// rows [r0, r1) x columns [cb, ce) -= L[:, k0..k0+K) U[k0..k0+K, :) on tcgen05
// (fp32 accumulation, one rounding to binary16); K a multiple of 64.
void tc_gemm(const TcPlan &p, int r0, int r1, int cb, int ce, int k0, int K, cudaStream_t s,
             int kclass = 4 /* KC_GEMM */);
void launch_gemm_tc(const TcPlan &p, int k0, int cb, int ce, cudaStream_t s);

// One rank of the 1-D block-cyclic LU (config 5a). a is the
// rank's n x n factor buffer (ld n) of which it owns the column blocks
// b with b mod G == r (block_cols columns each, a power-of-two multiple of
// nb); the broadcast of each panel between ranks is the caller's.
struct DluPlan
{
  int prec = 0, n = 0, G = 1, r = 0, sh = 30;
  LuWorkspace ws;
  // binary32 paired schedule (dlu_f32_*): tensor maps + pairing state, the
  // communication stream and its events ([0..1] message slot free, [2] join)
  void *f32 = nullptr;
  void *comm = nullptr;     // cudaStream_t
  void *cevents = nullptr;  // cudaEvent_t[3]
};
void dlu_alloc(DluPlan &d, int prec, int n, int nb, int G, int r, int block_cols);
void dlu_free(DluPlan &d);
void dlu_begin(DluPlan &d, int *perm, cudaStream_t s);
void dlu_panel(DluPlan &d, void *a, int p, int *ipiv, DevInfo *info, cudaStream_t s);
// part 0: whole step on s; 1: the next panel's columns (if owned) on s;
// 2: the remaining owned columns + left-column moves on the side stream.
void dlu_update(DluPlan &d, void *a, int p, int part, int *perm, cudaStream_t s);
void dlu_end(DluPlan &d, cudaStream_t s);
// The binary32 schedule of the single-GPU LU (TMA-fed update, paired K = 2nb
// steps, SM partition) restricted to this rank's columns. True when
// (prec, nb, n, a) qualify; otherwise the caller uses dlu_panel/dlu_update.
//   begin:  streams + tensor maps; `caller` is joined at dlu_f32_end
//   crit(): the stream the owner's panel (dlu_panel) and pack must run on
//   panel_ready(p, s): records "panel p is in this rank's buffer" on s
//   step(p): this rank's share of step p (next panel's columns on the
//            critical stream, the rest on the side stream)
bool dlu_f32_supported(const DluPlan &d, const void *a);
void dlu_f32_begin(DluPlan &d, void *a, int *perm, cudaStream_t caller);
cudaStream_t dlu_f32_crit(DluPlan &d);
cudaStream_t dlu_f32_comm(DluPlan &d);
void dlu_f32_panel_ready(DluPlan &d, int p, cudaStream_t s);
void dlu_f32_step(DluPlan &d, int p, int *perm, bool own_panel);
void dlu_f32_end(DluPlan &d, cudaStream_t caller);
void dlu_merge_singular(int *dst, const int *src, cudaStream_t s);

// ---- K6: triangular solves ------------------------------------------------
struct TrsvWorkspace
{
  int n = 0;
  int nblk = 0;
  int *tickets = nullptr;  // [2] block tickets
  unsigned long long *xw = nullptr;  // [2][2 cap_n] tagged hand-off words (lower, upper; two per binary64 x)
  int cap_n = 0;                     // allocated capacity
  void *map_cache = nullptr;         // host: the TMA map of the factor matrix last solved with (trsv.cu)
  int epoch = 0;
};
void trsv_workspace_alloc(TrsvWorkspace &ws, int n);
void trsv_workspace_free(TrsvWorkspace &ws);

// Substitution request. The solve runs in TS with TF factors.
//  prologue: y_i = LPS ? TS( rin[perm[i]] / rho ) : TS( rin[perm[i]] )  (rin in TIN)
//  epilogue (IR): d_i = LPS ? TR(y_i) * rho : TR(y_i); x_i += d_i; norms
//  epilogue (standalone): out_i = LPS ? TIN(y_i) * rho : y_i
struct TrsvArgs
{
  int ts, tf, tin;     // precisions
  int lps;             // scaled (solve_lps_into) vs promoting (solve_mps_into)
  int ir;              // fused refinement epilogue
  int n;
  const void *lu;      // packed factors (TF)
  const int *perm;     // accumulated permutation
  const void *rin;     // right-hand side / residual (TIN)
  const unsigned long long *rho_bits;  // LPS scale (bits of a non-negative double), or null
  void *y;             // scratch, n values of TS
  void *out;           // standalone: result (TIN for LPS, TS for MPS); IR: x accumulator (TIN=TR)
  unsigned long long *dnorm_bits;  // IR: ||d||_inf
  unsigned long long *xnorm_bits;  // IR: ||x||_inf after the update
  DevInfo *info;
};
void launch_trsv(const TrsvArgs &a, TrsvWorkspace &ws, cudaStream_t s);

// ---- K7: compensated residual r = b - A x in TR -------------------------
struct ResidualPlan
{
  void *tmap = nullptr;  // host copy of the CUtensorMap (128 B), owned
  int n = 0, tw = 0;
  const void *a = nullptr;
};
void residual_plan_make(ResidualPlan &p, int tw, int n, const void *a);
void residual_plan_free(ResidualPlan &p);
void launch_residual(const ResidualPlan &p, int tr, const void *x, const void *b, void *r,
                     unsigned long long *rnorm_bits, cudaStream_t s);

// ---- GMRES-IR corrections (krylov.cu; krylov_ir.hpp:62-171, 297-318) ---------
struct GmresCtx
{
  int n = 0, tw = 0, tf = 0, bs = 0;
  double rtol = 1e-2;       // gmres_correction_into's default
  const void *a_high = nullptr;
  const void *a_low = nullptr;
  const int *perm = nullptr;
  void *basis = nullptr;    // max(bs + 1, 7) x n values of TW
  void *tmp = nullptr;      // n values of TW
  void *dots = nullptr;     // bs + 2 device scalars of TW
  void *h_dots = nullptr;   // pinned mirror
  void *y = nullptr;        // substitution scratch
  DevInfo *info = nullptr, *h_info = nullptr;
  TrsvWorkspace *tws = nullptr;
  cudaStream_t s = nullptr;
  bool nonfinite = false;   // a preconditioner solve produced Inf/NaN
};
// w (n values of TW on the device): the residual on entry, the correction on
// exit (d may alias r, krylov_ir.hpp:57). Synchronises the stream.
void gmres_correction(GmresCtx &c, void *w, int *iters, bool *breakdown);
// bicgstab_correction_into (krylov_ir.hpp:173-254): same context (bs = the
// iteration budget, rtol = 0.1, seven work vectors at the start of basis).
void bicgstab_correction(GmresCtx &c, void *w, int *iters, bool *breakdown);
void launch_demote_vec(int tw, int tr, int n, const void *r, void *w, cudaStream_t s);
void launch_ir_update(int tw, int tr, int n, const void *w, void *x, unsigned long long *dnorm,
                      unsigned long long *xnorm, cudaStream_t s);

// ---- small vector kernels -------------------------------------------------
// r = TR(b); x = 0; *bnorm_bits = ||r||_inf (refine_loop start, ir_engine.hpp:190-205)
void launch_ir_init(int tw, int tr, int n, const void *b, void *r, void *x,
                    unsigned long long *bnorm_bits, cudaStream_t s);
// sol = TW(x) (ir_engine.hpp:267-269)
void launch_ir_finish(int tw, int tr, int n, const void *x, void *sol, cudaStream_t s);

}  // namespace mpirg
