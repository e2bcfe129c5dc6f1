// Host side of the B200 IR hot path: the MPFactorization handle, the
// refinement loop, and the C-ABI declared in include/mpir_gpu.h.
//
// Mirrors, line for line where it matters:
//   resolve_config / PrecisionConfig::validate  mp_structures.hpp:44-59, precision.hpp:222-230
//   MPFactorization ctor + refactor             mp_structures.hpp:108-169
//   TermParams / update_parms                   ir_engine.hpp:29-64
//   detail::plain_correction                    ir_engine.hpp:144-181
//   detail::refine_loop (termination ledger)    ir_engine.hpp:186-271
//   residual_tr                                 ir_engine.hpp:277-287
// The loop runs on the host exactly as in the reference; each pass launches
// the fused substitution pair and the residual kernel and reads back three
// doubles (||d||, ||x||, ||r||) plus the non-finite flag.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpir_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace mpirg;

namespace
{

struct ApiError
{
  int status;
  std::string msg;
  int column = -1;
  double value = 0.0;
};

const char *prec_name(int p) { return p == B64 ? "b64" : (p == B32 ? "b32" : "b16"); }
bool at_least_as_wide(int p, int q) { return p <= q; }  // codes: 0 widest
double machine_eps_of(int p) { return p == B64 ? 0x1p-52 : (p == B32 ? 0x1p-23 : 0x1p-10); }
double max_finite_of(int p) { return p == B64 ? DBL_MAX : (p == B32 ? (double)FLT_MAX : 65504.0); }

void validate_config(const mpirg_config &c)
{
  if (c.tw < 0 || c.tw > 2 || c.tf < 0 || c.tf > 2 || c.tr < 0 || c.tr > 2)
    throw ApiError{MPIRG_ERR_INVALID_CONFIG, "unknown precision"};
  if (c.tw == B16)
    throw ApiError{MPIRG_ERR_INVALID_CONFIG, "working precision must be b64 or b32"};
  if (!at_least_as_wide(c.tw, c.tf))
    throw ApiError{MPIRG_ERR_INVALID_CONFIG,
                   "factorization precision must not exceed the working precision"};
  if (!at_least_as_wide(c.tr, c.tw))
    throw ApiError{MPIRG_ERR_INVALID_CONFIG,
                   "residual precision must be at least the working precision"};
  if (c.tr == B16)
    throw ApiError{MPIRG_ERR_INVALID_CONFIG, "residual precision must be b64 or b32"};
  if (c.tf == c.tw && !c.on_the_fly)
    throw ApiError{MPIRG_ERR_INVALID_CONFIG, "equal-precision factors require on-the-fly solves"};
  if (c.lu_mode == MPIRG_LU_TC && c.tf != B16)
    throw ApiError{MPIRG_ERR_INVALID_CONFIG, "tensor-core LU needs binary16 factors"};
}

void validate_term(const mpirg_term_params &t)
{
  if (!(t.cr > 0.0) || !std::isfinite(t.cr))
    throw ApiError{MPIRG_ERR_INVALID_PARAM, "cr must be positive and finite"};
  if (!(t.ce > 0.0) || !std::isfinite(t.ce))
    throw ApiError{MPIRG_ERR_INVALID_PARAM, "ce must be positive and finite"};
  if (!(t.rmax > 0.0) || !(t.rmax <= 1.0))
    throw ApiError{MPIRG_ERR_INVALID_PARAM, "rmax must lie in (0, 1]"};
  if (t.litmax < 1)
    throw ApiError{MPIRG_ERR_INVALID_PARAM, "litmax must be at least 1"};
}

double bits_to_d(unsigned long long b)
{
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

void fill_err(mpirg_error *err, int status, const std::string &msg, int column = -1,
              double value = 0.0)
{
  if (!err)
    return;
  err->status = status;
  err->column = column;
  err->value = value;
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

template <typename F>
int guarded(mpirg_error *err, F &&fn)
{
  try
  {
    fn();
    fill_err(err, MPIRG_OK, "");
    return MPIRG_OK;
  }
  catch (const ApiError &e)
  {
    fill_err(err, e.status, e.msg, e.column, e.value);
    return e.status;
  }
  catch (const CudaError &e)
  {
    fill_err(err, MPIRG_ERR_CUDA, e.what());
    return MPIRG_ERR_CUDA;
  }
  catch (const std::invalid_argument &e)
  {
    fill_err(err, MPIRG_ERR_INVALID_CONFIG, e.what());
    return MPIRG_ERR_INVALID_CONFIG;
  }
  catch (const std::exception &e)
  {
    fill_err(err, MPIRG_ERR_CUDA, e.what());
    return MPIRG_ERR_CUDA;
  }
}

void require_gpu()
{
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw ApiError{MPIRG_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)"};
}

template <typename T>
T *dalloc(size_t count)
{
  void *p = nullptr;
  MPIRG_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T *>(p);
}
void *dalloc_bytes(size_t bytes)
{
  void *p = nullptr;
  MPIRG_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  return p;
}

void reset_info(DevInfo *info, cudaStream_t s)
{
  DevInfo h;
  h.overflow_index = ~0ull;
  h.underflow = 0;
  h.singular_col = INT_MAX;
  h.nonfinite = 0;
  h.pad = 0;
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(info, &h, sizeof(h), cudaMemcpyHostToDevice, s));
}

}  // namespace

// ---------------------------------------------------------------------------
// The handle
// ---------------------------------------------------------------------------
struct mpirg_factorization
{
  int n = 0;
  mpirg_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  void *a_high = nullptr;  // TW
  void *a_low = nullptr;   // TF: packed LU
  int *ipiv = nullptr;
  int *perm = nullptr;
  void *b = nullptr;       // TW
  void *r = nullptr;       // TR
  void *x = nullptr;       // TR
  void *y = nullptr;       // substitution scratch (max(TW, TF) bytes)
  void *sol = nullptr;     // TW
  void *comp = nullptr;    // TR: comp_buf of the reference's storage ledger (scratch)
  unsigned long long *scal = nullptr;  // [0] ||A||_1, [1] ||b||, [2+3i..] per pass
  int scal_cap = 0;
  DevInfo *info = nullptr;
  DevInfo *h_info = nullptr;               // pinned
  unsigned long long *h_scal = nullptr;    // pinned
  LuWorkspace luws;
  TrsvWorkspace tws;
  ResidualPlan rplan;
  double anorm1 = 0.0;
  int underflow = 0;
  float factor_ms = 0.0f;
  cudaEvent_t ev[4] = {};
  // refactor from host memory (refactor_streamed): copy stream + chunk events
  cudaStream_t cstream = nullptr;
  cudaEvent_t cev[LuLate::MAXCH + 1] = {};
  // the streamed refactor's launches as one CUDA graph, per pinned host pointer
  const void *sg_host = nullptr;
  int sg_seen = 0;
  cudaGraphExec_t sg_exec = nullptr;

  // GMRES-IR (krylov_ir.hpp): workspace carried by the factorization
  // (mp_structures.hpp:134-151), enabled by mpirg_factorization_enable_krylov
  int kry_kind = 0, kry_bs = 0;
  void *kry_basis = nullptr, *kry_tmp = nullptr, *kry_w = nullptr, *kry_dots = nullptr;
  void *kry_hdots = nullptr;  // pinned
  std::vector<int> khist;
  bool kry_breakdown = false;
  void enable_krylov(int kind, int basissize)
  {
    free_krylov();
    kry_kind = kind;
    kry_bs = basissize;
    // GMRES: basissize + 1 basis vectors; BiCGSTAB: its seven work vectors
    kry_basis = dalloc_bytes((size_t)std::max(basissize + 1, 7) * n * tw_bytes());
    kry_tmp = dalloc_bytes((size_t)n * tw_bytes());
    kry_w = dalloc_bytes((size_t)n * tw_bytes());
    kry_dots = dalloc_bytes((size_t)(basissize + 2) * 8);
    MPIRG_CUDA_CHECK(cudaMallocHost(&kry_hdots, (size_t)(basissize + 2) * 8));
  }
  void free_krylov()
  {
    for (void *p : {kry_basis, kry_tmp, kry_w, kry_dots})
      if (p)
        cudaFree(p);
    if (kry_hdots)
      cudaFreeHost(kry_hdots);
    kry_basis = kry_tmp = kry_w = kry_dots = kry_hdots = nullptr;
    kry_kind = kry_bs = 0;
  }

  // External storage (config 5b's batched LU factors many systems in shared
  // group buffers; a worker handle then runs the refinement on one system's
  // views of them). The handle's own matrices are kept and restored.
  bool ext_bound = false;
  void *own_a_high = nullptr, *own_a_low = nullptr;
  int *own_ipiv = nullptr, *own_perm = nullptr;
  void bind_external(const void *ah, void *al, int *ip, int *pm, double an1, int uf)
  {
    if (!ext_bound)
    {
      own_a_high = a_high;
      own_a_low = a_low;
      own_ipiv = ipiv;
      own_perm = perm;
      ext_bound = true;
    }
    a_high = const_cast<void *>(ah);
    a_low = al;
    ipiv = ip;
    perm = pm;
    anorm1 = an1;
    underflow = uf;
    residual_plan_make(rplan, cfg.tw, n, a_high);
  }
  void unbind()
  {
    if (!ext_bound)
      return;
    a_high = own_a_high;
    a_low = own_a_low;
    ipiv = own_ipiv;
    perm = own_perm;
    ext_bound = false;
    residual_plan_make(rplan, cfg.tw, n, a_high);
  }

  size_t tw_bytes() const { return elem_size(cfg.tw); }
  size_t tf_bytes() const { return elem_size(cfg.tf); }
  size_t tr_bytes() const { return elem_size(cfg.tr); }
  bool ext() const { return cfg.tr != cfg.tw; }

  void ensure_scal(int litmax)
  {
    const int need = 2 + 3 * (litmax + 1);
    if (need <= scal_cap)
      return;
    // the streamed-refactor graph has the old scal pointer baked into its
    // cast kernels (||A||_1 slot): drop it, the next refactor re-captures
    if (sg_exec)
      cudaGraphExecDestroy(sg_exec);
    sg_exec = nullptr;
    sg_host = nullptr;
    sg_seen = 0;
    if (scal)
      cudaFree(scal);
    if (h_scal)
      cudaFreeHost(h_scal);
    scal = dalloc<unsigned long long>(need);
    MPIRG_CUDA_CHECK(cudaMallocHost(&h_scal, sizeof(unsigned long long) * need));
    scal_cap = need;
  }

  void alloc()
  {
    const size_t nn = (size_t)n * n;
    int lo = 0, hi = 0;  // the handle's stream runs the LU's critical chain
    MPIRG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MPIRG_CUDA_CHECK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
    a_high = dalloc_bytes(nn * tw_bytes());
    a_low = dalloc_bytes(nn * tf_bytes());
    ipiv = dalloc<int>(n);
    perm = dalloc<int>(n);
    b = dalloc_bytes(n * tw_bytes());
    r = dalloc_bytes(n * tr_bytes());
    x = dalloc_bytes(n * tr_bytes());
    y = dalloc_bytes(n * 8);
    sol = dalloc_bytes(n * tw_bytes());
    comp = dalloc_bytes(n * tr_bytes());
    info = dalloc<DevInfo>(1);
    MPIRG_CUDA_CHECK(cudaMallocHost(&h_info, sizeof(DevInfo)));
    ensure_scal(16);
    lu_workspace_alloc(luws, cfg.tf, n, cfg.nb);
    trsv_workspace_alloc(tws, n);
    residual_plan_make(rplan, cfg.tw, n, a_high);
    for (auto &e : ev)
      MPIRG_CUDA_CHECK(cudaEventCreate(&e));
  }

  void release()
  {
    cudaSetDevice(device);
    unbind();
    free_krylov();
    for (void *p : {a_high, a_low, (void *)ipiv, (void *)perm, b, r, x, y, sol, comp, (void *)scal,
                    (void *)info})
      if (p)
        cudaFree(p);
    if (h_info)
      cudaFreeHost(h_info);
    if (h_scal)
      cudaFreeHost(h_scal);
    lu_workspace_free(luws);
    trsv_workspace_free(tws);
    residual_plan_free(rplan);
    for (auto &e : ev)
      if (e)
        cudaEventDestroy(e);
    for (auto &e : cev)
      if (e)
        cudaEventDestroy(e);
    if (sg_exec)
      cudaGraphExecDestroy(sg_exec);
    if (cstream)
      cudaStreamDestroy(cstream);
    if (stream)
      cudaStreamDestroy(stream);
  }

  // MPFactorization::refactor (mp_structures.hpp:155-169). do_lu = false
  // stops after the interprecision copy (the distributed LU of config 5a
  // factors a_low itself, then calls set_factored).
  void refactor(bool do_lu = true)
  {
    cudaStream_t s = stream;
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[0], s));
    reset_info(info, s);
    MPIRG_CUDA_CHECK(cudaMemsetAsync(scal, 0, sizeof(unsigned long long), s));
    launch_cast_norm(cfg.tw, cfg.tf, n, n, a_high, a_low, scal, info, s);
    if (do_lu)
      launch_lu(cfg.tf, cfg.lu_mode, a_low, n, ipiv, perm, luws, info, s);
    finish_refactor(do_lu);
  }

  // refactor from a host matrix with the host-to-device copy overlapped with
  // the factorization: the columns travel in chunks on a copy stream, each
  // chunk is cast (and its column sums folded into ||A||_1) as it lands, and
  // the LU starts as soon as the first chunk is in; later chunks catch up
  // with the panels already factored and then join the schedule
  // (launch_lu_late). Same results, bit for bit, as the copy-then-refactor
  // path: every kernel sees the same values, only earlier.
  static bool streamed_enabled()
  {
    static const bool v = [] {
      const char *e = std::getenv("MPIRG_STREAMED_H2D");
      return !(e && std::atoi(e) == 0);
    }();
    return v;
  }
  bool can_stream() const
  {
    return streamed_enabled() && lu_late_supported(cfg.tf, cfg.lu_mode, n) &&
           lu_choose_nb(cfg.tf, n, cfg.nb) == 64;
  }
  void refactor_streamed(const void *host_a)
  {
    cudaStream_t s = stream;
    if (!cstream)
    {
      cstream = lu_bulk_stream_create();
      for (auto &e : cev)
        MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // chunk plan: 256 + 256 columns, then equal chunks of >= 512 columns;
    // chunk c joins at the last even step before its first panel - 1
    LuLate L;
    std::vector<int> cuts{0, 256, 512};
    const int rest = n - 512;
    const int per = std::max(512, ((rest + (LuLate::MAXCH - 3) - 1) / (LuLate::MAXCH - 3) + 63) /
                                      64 * 64);
    for (int c = 512 + per; c < n; c += per)
      cuts.push_back(c);
    cuts.push_back(n);
    L.nch = (int)cuts.size() - 1;
    for (int c = 0; c < L.nch; ++c)
    {
      L.lo[c] = cuts[c];
      L.hi[c] = cuts[c + 1];
      L.join[c] = c == 0 ? 0 : std::max(0, ((cuts[c] / 64 - 2) / 2) * 2);
      L.ready[c] = cev[c + 1];
    }
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[0], s));
    reset_info(info, s);
    MPIRG_CUDA_CHECK(cudaMemsetAsync(scal, 0, sizeof(unsigned long long), s));
    // From a pinned host pointer seen before, the ~7 launches per panel step
    // on five streams replay as one graph (the first call with a pointer runs
    // directly: it also makes the lazily allocated late-chunk resources).
    const bool graph = streamed_graph_enabled() && !prof_on() && host_pinned(host_a);
    if (graph && sg_exec && sg_host == host_a)
    {
      MPIRG_CUDA_CHECK(cudaGraphLaunch(sg_exec, s));
      finish_refactor(true);
      return;
    }
    if (graph && sg_host != host_a)
    {
      if (sg_exec)
        cudaGraphExecDestroy(sg_exec);
      sg_exec = nullptr;
      sg_host = host_a;
      sg_seen = 0;
    }
    const bool capture = graph && sg_seen > 0;
    if (capture)
      MPIRG_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try
    {
      streamed_body(host_a, L);
    }
    catch (...)
    {
      if (capture)
      {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(s, &g);
        if (g)
          cudaGraphDestroy(g);
        sg_host = nullptr;
      }
      throw;
    }
    if (capture)
    {
      cudaGraph_t g = nullptr;
      MPIRG_CUDA_CHECK(cudaStreamEndCapture(s, &g));
      MPIRG_CUDA_CHECK(cudaGraphInstantiate(&sg_exec, g, 0));
      cudaGraphDestroy(g);
      MPIRG_CUDA_CHECK(cudaGraphLaunch(sg_exec, s));
    }
    else if (graph)
      ++sg_seen;
    finish_refactor(true);
  }
  static bool streamed_graph_enabled()
  {
    static const bool v = [] {
      const char *e = std::getenv("MPIRG_STREAMED_GRAPH");
      return !(e && std::atoi(e) == 0) && std::getenv("MPIRG_LU_TIMELINE") == nullptr &&
             !tool_attached();
    }();
    return v;
  }
  static bool host_pinned(const void *p)
  {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess)
    {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  }
  void streamed_body(const void *host_a, const LuLate &L)
  {
    cudaStream_t s = stream;
    MPIRG_CUDA_CHECK(cudaEventRecord(cev[0], s));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(cstream, cev[0], 0));
    const size_t colb = (size_t)n * tw_bytes();
    for (int c = 0; c < L.nch; ++c)
    {
      MPIRG_CUDA_CHECK(cudaMemcpyAsync(static_cast<char *>(a_high) + L.lo[c] * colb,
                                       static_cast<const char *>(host_a) + L.lo[c] * colb,
                                       (L.hi[c] - L.lo[c]) * colb, cudaMemcpyHostToDevice,
                                       cstream));
      launch_cast_norm(cfg.tw, cfg.tf, n, L.hi[c] - L.lo[c], a_high, a_low, scal, info, cstream,
                       L.lo[c]);
      MPIRG_CUDA_CHECK(cudaEventRecord(cev[c + 1], cstream));
    }
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, cev[1], 0));
    launch_lu_late(a_low, n, ipiv, perm, luws, info, s, L);
    for (int c = 0; c < L.nch; ++c)
      MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, cev[c + 1], 0));
  }

  void finish_refactor(bool do_lu)
  {
    cudaStream_t s = stream;
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[1], s));
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(h_info, info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(
        cudaMemcpyAsync(h_scal, scal, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    MPIRG_CUDA_CHECK(cudaEventElapsedTime(&factor_ms, ev[0], ev[1]));
    anorm1 = bits_to_d(h_scal[0]);
    underflow = h_info->underflow;
    if (h_info->overflow_index != ~0ull)
    {
      double v = 0.0;
      const size_t idx = (size_t)h_info->overflow_index;
      if (cfg.tw == B64)
        MPIRG_CUDA_CHECK(cudaMemcpy(&v, (char *)a_high + idx * 8, 8, cudaMemcpyDeviceToHost));
      else
      {
        float f;
        MPIRG_CUDA_CHECK(cudaMemcpy(&f, (char *)a_high + idx * 4, 4, cudaMemcpyDeviceToHost));
        v = f;
      }
      throw ApiError{MPIRG_ERR_OVERFLOW,
                     "value " + std::to_string(v) + " exceeds the largest finite " +
                         prec_name(cfg.tf) + " value",
                     -1, v};
    }
    if (do_lu && h_info->singular_col != INT_MAX)
      throw ApiError{MPIRG_ERR_SINGULAR, "pivot column is exactly zero", h_info->singular_col};
  }

  // detail::refine_loop + plain_correction (ir_engine.hpp:144-271).
  void solve(const mpirg_term_params &tp, mpirg_report *rep)
  {
    validate_term(tp);
    ensure_scal(tp.litmax);
    cudaStream_t s = stream;
    const int ns = 2 + 3 * (tp.litmax + 1);
    std::vector<double> rhist, dhist;
    rhist.reserve(tp.litmax + 1);
    dhist.reserve(tp.litmax + 1);
    auto emit = [&](int reason) {
      rep->rhist_len = (int)rhist.size();
      rep->dhist_len = (int)dhist.size();
      const int cap = rep->hist_capacity;
      for (int i = 0; i < (int)rhist.size() && i < cap; ++i)
        rep->rhist[i] = rhist[i];
      for (int i = 0; i < (int)dhist.size() && i < cap; ++i)
        rep->dhist[i] = dhist[i];
      rep->reason = reason;
    };

    khist.clear();
    kry_breakdown = false;
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[2], s));
    MPIRG_CUDA_CHECK(cudaMemsetAsync(scal + 1, 0, sizeof(unsigned long long) * (ns - 1), s));
    reset_info(info, s);
    launch_ir_init(cfg.tw, cfg.tr, n, b, r, x, scal + 1, s);

    const bool extended = ext();
    const double eps_w = machine_eps_of(cfg.tw);
    double bnorm = 0.0, rnorm = 0.0;
    int reason = MPIRG_ITERATION_LIMIT;
    for (int it = 0;; ++it)
    {
      unsigned long long *slot = scal + 2 + 3 * it;
      TrsvArgs a{};
      a.n = n;
      a.lu = a_low;
      a.perm = perm;
      a.rin = r;
      a.y = y;
      a.out = x;
      a.ir = 1;
      a.tin = cfg.tr;
      a.tf = cfg.tf;
      a.dnorm_bits = slot + 0;
      a.xnorm_bits = slot + 1;
      a.info = info;
      if (cfg.on_the_fly)
      {
        a.ts = cfg.tw;  // solve_mps_into<TW,TF> (on TW(r) when TR > TW)
        a.lps = 0;
      }
      else
      {
        a.ts = cfg.tf;  // solve_lps_into<TR,TF>
        a.lps = 1;
        a.rho_bits = it == 0 ? scal + 1 : scal + 2 + 3 * (it - 1) + 2;
      }
      if (kry_kind == 0)
        launch_trsv(a, tws, s);
      else
      {
        // krylov_ir_solve_report's corrector (krylov_ir.hpp:303-317): w = TW(r),
        // d = GMRES(A, M; w), x += TR(d), ||d||_inf
        launch_demote_vec(cfg.tw, cfg.tr, n, r, kry_w, s);
        GmresCtx g;
        g.n = n;
        g.tw = cfg.tw;
        g.tf = cfg.tf;
        g.bs = kry_bs;
        g.a_high = a_high;
        g.a_low = a_low;
        g.perm = perm;
        g.basis = kry_basis;
        g.tmp = kry_tmp;
        g.dots = kry_dots;
        g.h_dots = kry_hdots;
        g.y = y;
        g.info = info;
        g.h_info = h_info;
        g.tws = &tws;
        g.s = s;
        int its = 0;
        bool brk = false;
        if (kry_kind == MPIRG_KRYLOV_BICGSTAB)
        {
          g.rtol = 0.1;  // bicgstab_correction_into's default
          bicgstab_correction(g, kry_w, &its, &brk);
        }
        else
          gmres_correction(g, kry_w, &its, &brk);
        if (g.nonfinite)
        {
          if (it == 0)
          {
            MPIRG_CUDA_CHECK(cudaMemcpy(h_scal + 1, scal + 1, sizeof(unsigned long long),
                                        cudaMemcpyDeviceToHost));
            rhist.push_back(bits_to_d(h_scal[1]));
          }
          emit(MPIRG_ITERATION_LIMIT);
          throw ApiError{MPIRG_ERR_NONFINITE,
                         "promoting substitution produced a non-finite entry"};
        }
        khist.push_back(its);
        kry_breakdown = kry_breakdown || brk;
        launch_ir_update(cfg.tw, cfg.tr, n, kry_w, x, slot + 0, slot + 1, s);
      }
      launch_residual(rplan, cfg.tr, x, b, r, slot + 2, s);
      const int nread = 2 + 3 * (it + 1);
      MPIRG_CUDA_CHECK(cudaMemcpyAsync(h_scal + 1, scal + 1,
                                       sizeof(unsigned long long) * (nread - 1),
                                       cudaMemcpyDeviceToHost, s));
      MPIRG_CUDA_CHECK(
          cudaMemcpyAsync(h_info, info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
      MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));

      if (it == 0)
      {
        bnorm = bits_to_d(h_scal[1]);
        rhist.push_back(bnorm);
        if (!std::isfinite(bnorm))
        {
          emit(MPIRG_ITERATION_LIMIT);
          throw ApiError{MPIRG_ERR_NONFINITE, "right-hand side is not finite"};
        }
        rnorm = bnorm;
      }
      if (h_info->nonfinite)
      {
        emit(MPIRG_ITERATION_LIMIT);
        throw ApiError{MPIRG_ERR_NONFINITE,
                       cfg.on_the_fly ? "promoting substitution produced a non-finite entry"
                                      : "scaled substitution produced a non-finite entry"};
      }
      const unsigned long long *hs = h_scal + 2 + 3 * it;
      const double dnorm = bits_to_d(hs[0]);
      const double xnorm = bits_to_d(hs[1]);
      const double rnew = bits_to_d(hs[2]);
      dhist.push_back(dnorm);
      rhist.push_back(rnew);
      if (!std::isfinite(rnew) || !std::isfinite(dnorm))
      {
        emit(MPIRG_ITERATION_LIMIT);
        throw ApiError{MPIRG_ERR_NONFINITE, "refinement produced a non-finite iterate"};
      }
      if (!extended)
      {
        // ir_engine.hpp:234-236; the reference build contracts
        // bnorm + a_norm1 * ||x|| into one fma (GCC, -O3 -march, FMA host).
        const bool small = cfg.resid_term ? rnew <= tp.cr * eps_w * bnorm
                                          : rnew <= tp.ce * eps_w * std::fma(anorm1, xnorm, bnorm);
        if (small)
        {
          reason = cfg.resid_term ? MPIRG_SMALL_RESIDUAL : MPIRG_SMALL_BACKWARD_ERROR;
          break;
        }
        if (rnew >= tp.rmax * rnorm)
        {
          reason = MPIRG_RESIDUAL_STAGNATION;
          break;
        }
      }
      else
      {
        const size_t k = dhist.size();
        if (k >= 2 && dhist[k - 1] >= tp.rmax * dhist[k - 2])
        {
          reason = MPIRG_CORRECTION_STAGNATION;
          break;
        }
      }
      if ((int)rhist.size() >= tp.litmax)
      {
        reason = MPIRG_ITERATION_LIMIT;
        break;
      }
      rnorm = rnew;
    }
    launch_ir_finish(cfg.tw, cfg.tr, n, x, sol, s);
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[3], s));
    if (rep->sol)
      MPIRG_CUDA_CHECK(cudaMemcpyAsync(rep->sol, sol, n * tw_bytes(),
                                       rep->sol_on_device ? cudaMemcpyDeviceToDevice
                                                          : cudaMemcpyDeviceToHost,
                                       s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0.0f;
    MPIRG_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[2], ev[3]));
    rep->solve_ms = ms;
    emit(reason);
  }
};

// ---------------------------------------------------------------------------
// Shared context for the kernel-level entry points (one per device).
// ---------------------------------------------------------------------------
namespace
{

struct KernelCtx
{
  DevInfo *info = nullptr;
  DevInfo *h_info = nullptr;
  unsigned long long *bits = nullptr;
  LuWorkspace luws;
  int lu_prec = -1, lu_nb = -1;
  TrsvWorkspace tws;
  int *perm = nullptr;
  int perm_n = 0;
};

std::mutex g_mu;
KernelCtx g_ctx[64];

KernelCtx &ctx_for_current()
{
  int dev = 0;
  MPIRG_CUDA_CHECK(cudaGetDevice(&dev));
  KernelCtx &c = g_ctx[dev & 63];
  if (!c.info)
  {
    c.info = dalloc<DevInfo>(1);
    c.bits = dalloc<unsigned long long>(4);
    MPIRG_CUDA_CHECK(cudaMallocHost(&c.h_info, sizeof(DevInfo)));
  }
  return c;
}

int *ctx_perm(KernelCtx &c, int n)
{
  if (c.perm_n < n)
  {
    if (c.perm)
      cudaFree(c.perm);
    c.perm = dalloc<int>(n);
    c.perm_n = n;
  }
  return c.perm;
}

DevInfo read_info(KernelCtx &c, cudaStream_t s)
{
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(c.h_info, c.info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
  MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
  return *c.h_info;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int mpirg_abi_version(void) { return MPIRG_ABI_VERSION; }

int mpirg_device_count(void)
{
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess)
  {
    cudaGetLastError();
    return 0;
  }
  return c;
}

double mpirg_machine_eps(int p) { return machine_eps_of(p); }
double mpirg_unit_roundoff(int p) { return p == B64 ? 0x1p-53 : (p == B32 ? 0x1p-24 : 0x1p-11); }

int mpirg_resolve_config(int tw, int tf, int tr, int on_the_fly, mpirg_config *out,
                         mpirg_error *err)
{
  return guarded(err, [&] {
    if (tw == B16)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "working precision must be b64 or b32"};
    if (tw < 0 || tw > 2)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "unknown precision"};
    mpirg_config c{};
    c.tw = tw;
    c.tr = tr >= 0 ? tr : tw;
    c.tf = tf >= 0 ? tf : (tw == B32 ? B16 : B32);
    c.on_the_fly = on_the_fly >= 0 ? on_the_fly : (c.tf == B16);
    if (c.tf == c.tw)
      c.on_the_fly = 1;
    c.resid_term = 1;
    c.lu_mode = MPIRG_LU_EXACT;
    c.nb = 0;
    c.device = -1;
    validate_config(c);
    *out = c;
  });
}

int mpirg_update_parms(double cr, double ce, double rmax, int litmax, mpirg_term_params *out,
                       mpirg_error *err)
{
  return guarded(err, [&] {
    mpirg_term_params t{1.0, 1.0, 0.5, 10};
    if (!std::isnan(cr))
      t.cr = cr;
    if (!std::isnan(ce))
      t.ce = ce;
    if (!std::isnan(rmax))
      t.rmax = rmax;
    if (litmax > 0)
      t.litmax = litmax;
    validate_term(t);
    *out = t;
  });
}

int mpirg_factorization_create(mpirg_factorization **out, int n, const mpirg_config *cfg_in,
                               const void *a, int a_on_device, mpirg_error *err)
{
  *out = nullptr;
  return guarded(err, [&] {
    if (n < 0)
      throw ApiError{MPIRG_ERR_INVALID_SIZE, "matrix dimensions must be nonnegative"};
    mpirg_config c = *cfg_in;
    // mp_structures.hpp:118-122
    if (c.on_the_fly < 0)
      c.on_the_fly = (c.tf == B16 || c.tf == c.tw);
    if (c.tf == c.tw)
      c.on_the_fly = 1;
    validate_config(c);
    require_gpu();
    auto *f = new mpirg_factorization;
    f->n = n;
    f->cfg = c;
    if (c.device >= 0)
      MPIRG_CUDA_CHECK(cudaSetDevice(c.device));
    MPIRG_CUDA_CHECK(cudaGetDevice(&f->device));
    f->cfg.device = f->device;
    try
    {
      f->alloc();
      if (n > 0 && a)  // a == NULL: allocate only (refactor supplies A later)
      {
        MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->a_high, a, (size_t)n * n * f->tw_bytes(),
                                         a_on_device ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyHostToDevice,
                                         f->stream));
        f->refactor();
      }
    }
    catch (...)
    {
      f->release();
      delete f;
      throw;
    }
    *out = f;
  });
}

int mpirg_factorization_refactor(mpirg_factorization *f, const void *a, int a_on_device,
                                 mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(f->device));
    if (a && !a_on_device && f->n > 0 && f->can_stream())
    {
      f->refactor_streamed(a);
      return;
    }
    if (a)
      MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->a_high, a, (size_t)f->n * f->n * f->tw_bytes(),
                                       a_on_device ? cudaMemcpyDeviceToDevice
                                                   : cudaMemcpyHostToDevice,
                                       f->stream));
    if (f->n > 0)
      f->refactor();
  });
}

void mpirg_factorization_destroy(mpirg_factorization *f)
{
  if (!f)
    return;
  f->release();
  delete f;
}

int mpirg_factorization_n(const mpirg_factorization *f) { return f->n; }
int mpirg_factorization_config(const mpirg_factorization *f, mpirg_config *out)
{
  *out = f->cfg;
  return MPIRG_OK;
}
double mpirg_factorization_a_norm1(const mpirg_factorization *f) { return f->anorm1; }
int mpirg_factorization_demotion_underflowed(const mpirg_factorization *f) { return f->underflow; }
size_t mpirg_factorization_matrix_bytes(const mpirg_factorization *f)
{
  return (size_t)f->n * f->n * (f->tw_bytes() + f->tf_bytes());
}
double mpirg_factorization_last_factor_ms(const mpirg_factorization *f) { return f->factor_ms; }

int mpirg_factorization_get_ipiv(const mpirg_factorization *f, int *ipiv)
{
  cudaSetDevice(f->device);
  return cudaMemcpy(ipiv, f->ipiv, sizeof(int) * f->n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? MPIRG_OK
             : MPIRG_ERR_CUDA;
}
int mpirg_factorization_get_pivots(const mpirg_factorization *f, int *perm)
{
  cudaSetDevice(f->device);
  return cudaMemcpy(perm, f->perm, sizeof(int) * f->n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? MPIRG_OK
             : MPIRG_ERR_CUDA;
}
int mpirg_factorization_get_packed_lu(const mpirg_factorization *f, void *out)
{
  cudaSetDevice(f->device);
  return cudaMemcpy(out, f->a_low, (size_t)f->n * f->n * f->tf_bytes(),
                    cudaMemcpyDeviceToHost) == cudaSuccess
             ? MPIRG_OK
             : MPIRG_ERR_CUDA;
}
int mpirg_factorization_get_a_high(const mpirg_factorization *f, void *out)
{
  cudaSetDevice(f->device);
  return cudaMemcpy(out, f->a_high, (size_t)f->n * f->n * f->tw_bytes(),
                    cudaMemcpyDeviceToHost) == cudaSuccess
             ? MPIRG_OK
             : MPIRG_ERR_CUDA;
}
const void *mpirg_factorization_a_high_device(const mpirg_factorization *f) { return f->a_high; }
const void *mpirg_factorization_packed_lu_device(const mpirg_factorization *f) { return f->a_low; }
const int *mpirg_factorization_ipiv_device(const mpirg_factorization *f) { return f->ipiv; }
void *mpirg_factorization_stream(const mpirg_factorization *f) { return f->stream; }
void *mpirg_factorization_residual_buf_device(mpirg_factorization *f) { return f->r; }
void *mpirg_factorization_sol_buf_device(mpirg_factorization *f) { return f->x; }
void *mpirg_factorization_comp_buf_device(mpirg_factorization *f) { return f->comp; }
void *mpirg_factorization_low_buf_device(mpirg_factorization *f) { return f->y; }
void *mpirg_factorization_work_buf_device(mpirg_factorization *f) { return f->y; }

int mpirg_ir_solve(mpirg_factorization *f, const void *b, int b_on_device,
                   const mpirg_term_params *tp, mpirg_report *rep, mpirg_error *err)
{
  rep->rhist_len = 0;
  rep->dhist_len = 0;
  return guarded(err, [&] {
    mpirg_term_params t = tp ? *tp : mpirg_term_params{1.0, 1.0, 0.5, 10};
    MPIRG_CUDA_CHECK(cudaSetDevice(f->device));
    if (f->n == 0)
    {
      validate_term(t);
      rep->rhist_len = 0;
      rep->reason = MPIRG_ITERATION_LIMIT;
      return;
    }
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->b, b, f->n * f->tw_bytes(),
                                     b_on_device ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyHostToDevice,
                                     f->stream));
    f->solve(t, rep);
  });
}

int mpirg_residual_tr(mpirg_factorization *f, const void *x, const void *b, void *r,
                      int on_device, mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(f->device));
    const int n = f->n;
    cudaStream_t s = f->stream;
    const cudaMemcpyKind in = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // x (TW) -> sol scratch, widen into f->x (TR); b -> f->b.
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->sol, x, n * f->tw_bytes(), in, s));
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->b, b, n * f->tw_bytes(), in, s));
    MPIRG_CUDA_CHECK(cudaMemsetAsync(f->scal + 1, 0, 2 * sizeof(unsigned long long), s));
    launch_ir_init(f->cfg.tw, f->cfg.tr, n, f->sol, f->x, f->r, f->scal + 1, s);
    launch_residual(f->rplan, f->cfg.tr, f->x, f->b, f->r, f->scal + 2, s);
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(r, f->r, n * f->tr_bytes(),
                                     on_device ? cudaMemcpyDeviceToDevice
                                               : cudaMemcpyDeviceToHost,
                                     s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

// ---- kernel-level entry points ----------------------------------------------
int mpirg_demote(int from, int to, size_t count, const void *src, void *dst, int *underflow,
                 void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    reset_info(c.info, s);
    launch_demote(from, to, src, dst, count, c.info, s);
    const DevInfo h = read_info(c, s);
    if (underflow)
      *underflow = h.underflow;
    if (h.overflow_index != ~0ull)
    {
      double v = 0.0;
      const size_t idx = (size_t)h.overflow_index;
      if (from == B64)
        MPIRG_CUDA_CHECK(cudaMemcpy(&v, (const char *)src + idx * 8, 8, cudaMemcpyDeviceToHost));
      else
      {
        float fv;
        MPIRG_CUDA_CHECK(cudaMemcpy(&fv, (const char *)src + idx * 4, 4, cudaMemcpyDeviceToHost));
        v = fv;
      }
      throw ApiError{MPIRG_ERR_OVERFLOW,
                     "value " + std::to_string(v) + " exceeds the largest finite " +
                         prec_name(to) + " value",
                     -1, v};
    }
  });
}

int mpirg_one_norm(int prec, int rows, int cols, const void *a, double *out, void *stream,
                   mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    MPIRG_CUDA_CHECK(cudaMemsetAsync(c.bits, 0, sizeof(unsigned long long), s));
    launch_one_norm(prec, rows, cols, a, c.bits, s);
    unsigned long long hb = 0;
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(&hb, c.bits, 8, cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    *out = bits_to_d(hb);
  });
}

int mpirg_lu_factor(int prec, int n, void *a, int *ipiv, int lu_mode, int nb, void *stream,
                    mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    if (lu_mode == MPIRG_LU_TC && prec != B16)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "tensor-core LU needs binary16 factors"};
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    const int want_nb = lu_choose_nb(prec, n, nb);
    if (c.luws.n < n || c.lu_nb != want_nb || c.lu_prec != prec)
    {
      lu_workspace_alloc(c.luws, prec, n, nb);
      c.lu_prec = prec;
      c.lu_nb = c.luws.nb;
    }
    LuWorkspace ws = c.luws;  // sized for >= n panels
    ws.n = n;
    ws.npanels = (n + ws.nb - 1) / ws.nb;
    reset_info(c.info, s);
    launch_lu(prec, lu_mode, a, n, ipiv, nullptr, ws, c.info, s);
    const DevInfo h = read_info(c, s);
    if (h.singular_col != INT_MAX)
      throw ApiError{MPIRG_ERR_SINGULAR, "pivot column is exactly zero", h.singular_col};
  });
}

static void standalone_trsv(TrsvArgs &a, KernelCtx &c, cudaStream_t s)
{
  if (c.tws.n < a.n)
    trsv_workspace_alloc(c.tws, a.n);
  TrsvWorkspace ws = c.tws;
  ws.n = a.n;
  ws.nblk = (a.n + 31) / 32;
  launch_trsv(a, ws, s);
  c.tws.epoch = ws.epoch;
}

int mpirg_solve_mps(int ts, int tf, int n, const void *packed, const int *ipiv, void *x,
                    void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    if (!at_least_as_wide(ts, tf))
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "promotion must not lose precision"};
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    if (n == 0)
      return;
    int *perm = ctx_perm(c, n);
    launch_perm_from_ipiv(ipiv, n, perm, s);
    reset_info(c.info, s);
    // Gather into scratch y first (the epilogue writes x in place).
    void *xin = dalloc_bytes((size_t)n * elem_size(ts));
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(xin, x, (size_t)n * elem_size(ts), cudaMemcpyDeviceToDevice, s));
    void *y = dalloc_bytes((size_t)n * 8);
    TrsvArgs a{};
    a.ts = ts;
    a.tf = tf;
    a.tin = ts;
    a.lps = 0;
    a.ir = 0;
    a.n = n;
    a.lu = packed;
    a.perm = perm;
    a.rin = xin;
    a.y = y;
    a.out = x;
    a.info = c.info;
    standalone_trsv(a, c, s);
    const DevInfo h = read_info(c, s);
    cudaFree(xin);
    cudaFree(y);
    if (h.nonfinite)
      throw ApiError{MPIRG_ERR_NONFINITE, "promoting substitution produced a non-finite entry"};
  });
}

int mpirg_solve_lps(int tw, int tf, int n, const void *packed, const int *ipiv, void *r_to_d,
                    void *scratch, int *underflow, void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    if (!at_least_as_wide(tw, tf) || tw == B16)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "demotion must not gain precision"};
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    if (n == 0)
      return;
    int *perm = ctx_perm(c, n);
    launch_perm_from_ipiv(ipiv, n, perm, s);
    reset_info(c.info, s);
    // rho = max |r_i| with a > rho (NaN ignored): dense_lu.hpp:208-214.
    MPIRG_CUDA_CHECK(cudaMemsetAsync(c.bits, 0, sizeof(unsigned long long), s));
    launch_one_norm(tw, 1, n, r_to_d, c.bits, s);  // max over "columns" of |r_i|, NaN ignored
    void *rin = dalloc_bytes((size_t)n * elem_size(tw));
    MPIRG_CUDA_CHECK(
        cudaMemcpyAsync(rin, r_to_d, (size_t)n * elem_size(tw), cudaMemcpyDeviceToDevice, s));
    TrsvArgs a{};
    a.ts = tf;
    a.tf = tf;
    a.tin = tw;
    a.lps = 1;
    a.ir = 0;
    a.n = n;
    a.lu = packed;
    a.perm = perm;
    a.rin = rin;
    a.rho_bits = c.bits;
    a.y = scratch;
    a.out = r_to_d;
    a.info = c.info;
    standalone_trsv(a, c, s);
    const DevInfo h = read_info(c, s);
    cudaFree(rin);
    if (underflow)
      *underflow = h.underflow;
    if (h.nonfinite)
      throw ApiError{MPIRG_ERR_NONFINITE, "scaled substitution produced a non-finite entry"};
  });
}

int mpirg_residual(int tw, int tr, int n, const void *a, const void *x, const void *b, void *r,
                   void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    require_gpu();
    if (!at_least_as_wide(tr, tw) || tw == B16 || tr == B16)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG,
                     "residual precision must be at least the working precision"};
    std::lock_guard<std::mutex> lk(g_mu);
    auto s = static_cast<cudaStream_t>(stream);
    KernelCtx &c = ctx_for_current();
    if (n == 0)
      return;
    ResidualPlan p;
    residual_plan_make(p, tw, n, a);
    MPIRG_CUDA_CHECK(cudaMemsetAsync(c.bits, 0, sizeof(unsigned long long), s));
    launch_residual(p, tr, x, b, r, c.bits, s);
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    residual_plan_free(p);
  });
}

// Config 5b: independent systems solved concurrently. W host workers, each
// driving its own handle (own streams, workspaces and pinned mirrors), take
// systems from a shared counter; their kernels overlap on the SMs that one
// N~1024 system leaves idle. Each system is exactly one MPFactorization +
// ir_solve_report, so results equal the sequential ones bit for bit.
// Device staging of a host batch (see mpirg_batch_ir_solve). Used only when
// the host arrays are pinned (page-locked copies are truly asynchronous) and
// the batch fits in half of the free HBM; otherwise each worker copies its own
// system as before.
struct BatchStage
{
  bool ok = false;
  void *a = nullptr, *b = nullptr, *sol = nullptr;
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> ready;
  int per = 16;  // systems per copy chunk
  static bool pinned(const void *p)
  {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess)
    {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  }
  void make(int count, int n, size_t tw, const void *ha, const void *hb)
  {
    const size_t abytes = (size_t)count * n * n * tw, vbytes = (size_t)count * n * tw;
    size_t fr = 0, tot = 0;
    if (!pinned(ha) || !pinned(hb) || cudaMemGetInfo(&fr, &tot) != cudaSuccess ||
        abytes + 2 * vbytes > fr / 2)
      return;
    if (cudaMalloc(&a, abytes) != cudaSuccess || cudaMalloc(&b, vbytes) != cudaSuccess ||
        cudaMalloc(&sol, vbytes) != cudaSuccess ||
        cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
    {
      cudaGetLastError();
      release();
      return;
    }
    const int nch = (count + per - 1) / per;
    ready.assign(nch, nullptr);
    bool good = cudaMemcpyAsync(b, hb, vbytes, cudaMemcpyHostToDevice, cs) == cudaSuccess;
    for (int c = 0; c < nch && good; ++c)
    {
      const size_t lo = (size_t)c * per, hi = std::min((size_t)count, lo + per);
      const size_t sz = (size_t)n * n * tw;
      good = cudaEventCreateWithFlags(&ready[c], cudaEventDisableTiming) == cudaSuccess &&
             cudaMemcpyAsync(static_cast<char *>(a) + lo * sz,
                             static_cast<const char *>(ha) + lo * sz, (hi - lo) * sz,
                             cudaMemcpyHostToDevice, cs) == cudaSuccess &&
             cudaEventRecord(ready[c], cs) == cudaSuccess;
    }
    if (!good)
    {
      cudaGetLastError();
      cudaStreamSynchronize(cs);
      release();
      return;
    }
    ok = true;
  }
  void release()
  {
    if (cs)
      cudaStreamSynchronize(cs);
    for (auto &e : ready)
      if (e)
        cudaEventDestroy(e);
    ready.clear();
    if (a)
      cudaFree(a);
    if (b)
      cudaFree(b);
    if (sol)
      cudaFree(sol);
    if (cs)
      cudaStreamDestroy(cs);
    a = b = sol = nullptr;
    cs = nullptr;
    ok = false;
  }
};

static int batch_workers(int count, int n)
{
  int w = n <= 1024 ? 16 : (n <= 2048 ? 8 : (n <= 4096 ? 4 : 1));
  if (const char *e = std::getenv("MPIRG_BATCH_WORKERS"))
    w = std::max(1, std::atoi(e));
  return std::max(1, std::min(w, count));
}

// ---- config 5b, batched kernels ------------------------------------------------
// <f64, f32, f64> scaled-correction batches (BASELINE 5b) take this path: the
// systems are factored in groups of NS by batched launches (lu.cu
// launch_lu_batched_f32: one launch per step for the whole group instead of
// ~100 launches per system), double-buffered so that the refinement of group
// g -- W host workers, each binding a reusable handle to one system's views of
// the group buffers -- overlaps the LUs of groups g + 1 .. g + 3 on the device. Every
// kernel is the single-system one: per-system results equal the sequential
// ones bit for bit. MPIRG_BATCH_MODE=handles keeps the per-system path.
static int batch_group_size(int count, int n)
{
  int g = n <= 1024 ? 128 : (n <= 2048 ? 32 : 8);
  if (const char *e = std::getenv("MPIRG_BATCH_GROUP"))
    g = std::max(1, std::atoi(e));
  return std::max(1, std::min(g, count));
}

static bool batch_fast_ok(const mpirg_config &c, int n)
{
  if (const char *e = std::getenv("MPIRG_BATCH_MODE"))
    if (std::string(e) == "handles")
      return false;
  const int otf = c.on_the_fly < 0 ? (c.tf == B16 || c.tf == c.tw) : c.on_the_fly;
  return c.tw == B64 && c.tf == B32 && c.tr == B64 && otf == 0 && c.lu_mode == MPIRG_LU_EXACT &&
         (c.nb == 0 || c.nb == 64) && n >= 64 && lu_batched_supported(B32, n);
}

struct BatchSlot
{
  float *a_low = nullptr, *ut = nullptr;
  int *ipiv = nullptr, *perm = nullptr, *nmoves = nullptr;
  int2 *moves = nullptr;
  DevInfo *info = nullptr, *h_info = nullptr, *h_init = nullptr;
  unsigned long long *norm = nullptr, *h_norm = nullptr;
  cudaEvent_t done = nullptr;
  void alloc(int ns, int n)
  {
    const int np = (n + 63) / 64;
    a_low = dalloc<float>((size_t)ns * n * n);
    ut = dalloc<float>((size_t)64 * ns * n);
    ipiv = dalloc<int>((size_t)ns * n);
    perm = dalloc<int>((size_t)ns * n);
    nmoves = dalloc<int>((size_t)ns * np);
    moves = dalloc<int2>((size_t)ns * np * 128);
    info = dalloc<DevInfo>(ns);
    norm = dalloc<unsigned long long>(ns);
    MPIRG_CUDA_CHECK(cudaMallocHost(&h_info, sizeof(DevInfo) * ns));
    MPIRG_CUDA_CHECK(cudaMallocHost(&h_init, sizeof(DevInfo) * ns));
    MPIRG_CUDA_CHECK(cudaMallocHost(&h_norm, sizeof(unsigned long long) * ns));
    for (int i = 0; i < ns; ++i)
    {
      h_init[i].overflow_index = ~0ull;
      h_init[i].underflow = 0;
      h_init[i].singular_col = INT_MAX;
      h_init[i].nonfinite = 0;
      h_init[i].pad = 0;
    }
    MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  }
  void release()
  {
    for (void *p : {(void *)a_low, (void *)ut, (void *)ipiv, (void *)perm, (void *)nmoves,
                    (void *)moves, (void *)info, (void *)norm})
      if (p)
        cudaFree(p);
    for (void *p : {(void *)h_info, (void *)h_init, (void *)h_norm})
      if (p)
        cudaFreeHost(p);
    if (done)
      cudaEventDestroy(done);
  }
};

static int batch_ir_solve_fast(int count, int n, const mpirg_config &cfg_in, const char *a_dev,
                               const char *b_dev, char *sol_dev, const BatchStage *stage,
                               const mpirg_term_params *tp, double *rhist, double *dhist,
                               int hist_capacity, int *rhist_len, int *reason, int *status,
                               double *device_ms, mpirg_error *err, int dev)
{
  const int NS = batch_group_size(count, n), G = (count + NS - 1) / NS;
  const int W = batch_workers(count, n);
  const size_t nn = (size_t)n * n;
  // NSLOT group buffers, each with its own stream: the LUs of consecutive
  // groups overlap each other (one group's latency-bound panel launches run
  // beside another's trailing updates) and the refinement of earlier groups
  constexpr int NSLOT = 4;
  BatchSlot slot[NSLOT];
  cudaStream_t lstream[NSLOT] = {};
  cudaEvent_t start = nullptr;
  std::vector<mpirg_factorization *> handles(W, nullptr);
  std::vector<cudaEvent_t> ends(W, nullptr);
  std::mutex emu;
  int first = MPIRG_OK;
  mpirg_error first_err{};
  auto note = [&](int st, const mpirg_error &e) {
    std::lock_guard<std::mutex> lk(emu);
    if (first == MPIRG_OK && st != MPIRG_OK)
    {
      first = st;
      first_err = e;
    }
  };
  auto cleanup = [&] {
    for (auto *f : handles)
      mpirg_factorization_destroy(f);
    for (auto &e : ends)
      if (e)
        cudaEventDestroy(e);
    for (int i = 0; i < NSLOT; ++i)
    {
      slot[i].release();
      if (lstream[i])
        cudaStreamDestroy(lstream[i]);
    }
    if (start)
      cudaEventDestroy(start);
  };
  mpirg_config c = cfg_in;
  c.device = dev;
  {
    mpirg_error e{};
    const int st = guarded(&e, [&] {
      MPIRG_CUDA_CHECK(cudaEventCreate(&start));
      for (int i = 0; i < NSLOT && i < G; ++i)
      {
        MPIRG_CUDA_CHECK(cudaStreamCreateWithFlags(&lstream[i], cudaStreamNonBlocking));
        slot[i].alloc(NS, n);
      }
      struct NoPartition  // the workers' handles share the whole GPU (lu.cu)
      {
        NoPartition() { lu_partition_allowed(false); }
        ~NoPartition() { lu_partition_allowed(true); }
      } no_partition;
      for (int w = 0; w < W; ++w)
      {
        mpirg_error ce{};
        const int cs = mpirg_factorization_create(&handles[w], n, &c, nullptr, 1, &ce);
        if (cs != MPIRG_OK)
          throw ApiError{cs, ce.message};
        MPIRG_CUDA_CHECK(cudaEventCreate(&ends[w]));
      }
      MPIRG_CUDA_CHECK(cudaEventRecord(start, lstream[0]));
      for (int i = 1; i < NSLOT && i < G; ++i)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(lstream[i], start, 0));
    });
    if (st != MPIRG_OK)
    {
      cleanup();
      if (err)
        *err = e;
      for (int i = 0; i < count; ++i)
        status[i] = st;
      return st;
    }
  }
  // host-side pipeline state
  std::atomic<int> next{0}, ready_upto{0}, failed{0};
  std::vector<std::atomic<int>> finished(G);
  for (auto &f : finished)
    f.store(0);
  auto group_size = [&](int g) { return std::min(NS, count - g * NS); };

  auto enqueue = [&](int g) {
    BatchSlot &S = slot[g % NSLOT];
    cudaStream_t ls = lstream[g % NSLOT];
    const int lo = g * NS, ns = group_size(g);
    if (stage)
      for (int ch = lo / stage->per; ch <= (lo + ns - 1) / stage->per; ++ch)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(ls, stage->ready[ch], 0));
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(S.info, S.h_init, sizeof(DevInfo) * ns,
                                     cudaMemcpyHostToDevice, ls));
    MPIRG_CUDA_CHECK(cudaMemsetAsync(S.norm, 0, sizeof(unsigned long long) * ns, ls));
    if (ns > 1)
      launch_cast_norm(B64, B32, n, n, a_dev + (size_t)lo * nn * 8, S.a_low, S.norm, S.info, ls, 0,
                       ns);
    else
      launch_cast_norm(B64, B32, n, n, a_dev + (size_t)lo * nn * 8, S.a_low, S.norm, S.info, ls);
    launch_lu_batched_f32(S.a_low, n, ns, S.ipiv, S.perm, S.moves, S.nmoves, S.info, ls, S.ut);
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(S.h_info, S.info, sizeof(DevInfo) * ns,
                                     cudaMemcpyDeviceToHost, ls));
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(S.h_norm, S.norm, sizeof(unsigned long long) * ns,
                                     cudaMemcpyDeviceToHost, ls));
    MPIRG_CUDA_CHECK(cudaEventRecord(S.done, ls));
  };

  auto worker = [&](int w) {
    cudaSetDevice(dev);
    mpirg_factorization *f = handles[w];
    for (int idx; (idx = next.fetch_add(1)) < count;)
    {
      const int g = idx / NS, z = idx - g * NS;
      while (ready_upto.load(std::memory_order_acquire) <= g && !failed.load())
        std::this_thread::yield();
      if (failed.load())
      {
        finished[g].fetch_add(1);
        continue;
      }
      if (status[idx] == MPIRG_OK)
      {
        BatchSlot &S = slot[g % NSLOT];
        mpirg_error e{};
        mpirg_report rep{};
        rep.sol = sol_dev + (size_t)idx * n * 8;
        rep.sol_on_device = 1;
        rep.rhist = rhist + (size_t)idx * hist_capacity;
        rep.dhist = dhist + (size_t)idx * hist_capacity;
        rep.hist_capacity = hist_capacity;
        const int st = guarded(&e, [&] {
          f->bind_external(a_dev + (size_t)idx * nn * 8, S.a_low + (size_t)z * nn,
                           S.ipiv + (size_t)z * n, S.perm + (size_t)z * n,
                           bits_to_d(S.h_norm[z]), S.h_info[z].underflow);
          MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->b, b_dev + (size_t)idx * n * 8, (size_t)n * 8,
                                           cudaMemcpyDeviceToDevice, f->stream));
          const mpirg_term_params t = tp ? *tp : mpirg_term_params{1.0, 1.0, 0.5, 10};
          f->solve(t, &rep);
        });
        rhist_len[idx] = rep.rhist_len;
        reason[idx] = rep.reason;
        status[idx] = st;
        note(st, e);
      }
      finished[g].fetch_add(1, std::memory_order_release);
    }
    cudaEventRecord(ends[w], f->stream);
    cudaEventSynchronize(ends[w]);
  };

  for (int i = 0; i < count; ++i)
  {
    status[i] = MPIRG_OK;
    rhist_len[i] = 0;
    reason[i] = MPIRG_ITERATION_LIMIT;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < W; ++w)
    pool.emplace_back(worker, w);
  {
    mpirg_error e{};
    const int st = guarded(&e, [&] {
      int enq = 0;
      for (int g = 0; g < G; ++g)
      {
        while (enq <= std::min(g + NSLOT - 1, G - 1))
        {
          if (enq >= NSLOT)  // the slot is free once every system of its last group is refined
            while (finished[enq - NSLOT].load(std::memory_order_acquire) <
                   group_size(enq - NSLOT))
              std::this_thread::yield();
          enqueue(enq);
          ++enq;
        }
        BatchSlot &S = slot[g % NSLOT];
        MPIRG_CUDA_CHECK(cudaEventSynchronize(S.done));
        const int lo = g * NS, ns = group_size(g);
        for (int z = 0; z < ns; ++z)
        {
          const DevInfo &hi = S.h_info[z];
          mpirg_error se{};
          if (hi.overflow_index != ~0ull)
          {
            double v = 0.0;
            MPIRG_CUDA_CHECK(cudaMemcpy(&v, a_dev + ((size_t)(lo + z) * nn + hi.overflow_index) * 8,
                                        8, cudaMemcpyDeviceToHost));
            fill_err(&se, MPIRG_ERR_OVERFLOW,
                     "value " + std::to_string(v) + " exceeds the largest finite b32 value", -1,
                     v);
            status[lo + z] = MPIRG_ERR_OVERFLOW;
            note(MPIRG_ERR_OVERFLOW, se);
          }
          else if (hi.singular_col != INT_MAX)
          {
            fill_err(&se, MPIRG_ERR_SINGULAR, "pivot column is exactly zero", hi.singular_col);
            status[lo + z] = MPIRG_ERR_SINGULAR;
            note(MPIRG_ERR_SINGULAR, se);
          }
        }
        ready_upto.store(g + 1, std::memory_order_release);
      }
    });
    if (st != MPIRG_OK)
    {
      note(st, e);
      failed.store(1);
      for (int i = 0; i < count; ++i)
        if (status[i] == MPIRG_OK && rhist_len[i] == 0)
          status[i] = st;
    }
  }
  for (auto &t : pool)
    t.join();
  double ms = 0.0;
  for (int w = 0; w < W; ++w)
  {
    float m = 0.0f;
    if (cudaEventElapsedTime(&m, start, ends[w]) == cudaSuccess)
      ms = std::max(ms, (double)m);
  }
  cudaGetLastError();
  if (device_ms)
    *device_ms = ms;
  cleanup();
  if (err)
    *err = first == MPIRG_OK ? mpirg_error{} : first_err;
  if (first == MPIRG_OK)
    fill_err(err, MPIRG_OK, "");
  return first;
}

int mpirg_batch_ir_solve(int count, int n, const mpirg_config *cfg, const void *a, const void *b,
                         int on_device, const mpirg_term_params *tp, void *sol, double *rhist,
                         double *dhist, int hist_capacity, int *rhist_len, int *reason,
                         int *status, double *device_ms, mpirg_error *err)
{
  if (count <= 0)
  {
    if (device_ms)
      *device_ms = 0.0;
    fill_err(err, MPIRG_OK, "");
    return MPIRG_OK;
  }
  int dev = 0;
  if (cfg->device >= 0)
    cudaSetDevice(cfg->device);
  cudaGetDevice(&dev);
  const int W = batch_workers(count, n);
  const size_t tw = elem_size(cfg->tw);
  std::atomic<int> next{0};
  std::mutex emu;
  int first = MPIRG_OK;
  mpirg_error first_err{};
  auto note = [&](int st, const mpirg_error &e) {
    std::lock_guard<std::mutex> lk(emu);
    if (first == MPIRG_OK && st != MPIRG_OK)
    {
      first = st;
      first_err = e;
    }
  };
  cudaEvent_t start = nullptr;
  std::vector<cudaEvent_t> ends(W, nullptr);
  std::vector<int> used(W, 0);
  {
    mpirg_error e{};
    const int st = guarded(&e, [&] {
      MPIRG_CUDA_CHECK(cudaEventCreate(&start));
      for (auto &ev : ends)
        MPIRG_CUDA_CHECK(cudaEventCreate(&ev));
      MPIRG_CUDA_CHECK(cudaEventRecord(start, 0));
    });
    if (st != MPIRG_OK)
    {
      if (err)
        *err = e;
      return st;
    }
  }
  // Pinned host inputs: stage the batch through HBM on a copy stream in
  // chunks of systems, issued up front. The workers take systems in index
  // order, so the copies run ahead of the solves and overlap them, instead of
  // one small synchronous copy per system. Solutions come back in one copy.
  BatchStage stage;
  if (!on_device)
    stage.make(count, n, tw, a, b);
  const bool staged = stage.ok;
  if ((on_device || staged) && batch_fast_ok(*cfg, n))
  {
    cudaEventDestroy(start);
    for (auto &ev : ends)
      cudaEventDestroy(ev);
    const int st = batch_ir_solve_fast(
        count, n, *cfg, static_cast<const char *>(staged ? stage.a : a),
        static_cast<const char *>(staged ? stage.b : b),
        static_cast<char *>(staged ? stage.sol : sol), staged ? &stage : nullptr, tp, rhist, dhist,
        hist_capacity, rhist_len, reason, status, device_ms, err, dev);
    if (staged)
    {
      // runs of solved systems only: a failed system's slice of `sol` stays untouched
      for (int lo = 0; lo < count;)
      {
        if (status[lo] != MPIRG_OK)
        {
          ++lo;
          continue;
        }
        int hi = lo;
        while (hi < count && status[hi] == MPIRG_OK)
          ++hi;
        const size_t off = (size_t)lo * n * tw;
        cudaMemcpy(static_cast<char *>(sol) + off, static_cast<char *>(stage.sol) + off,
                   (size_t)(hi - lo) * n * tw, cudaMemcpyDeviceToHost);
        lo = hi;
      }
      stage.release();
    }
    return st;
  }
  const void *a_src = staged ? stage.a : a;
  const void *b_src = staged ? stage.b : b;
  void *sol_dst = staged ? stage.sol : sol;
  const int src_on_device = staged ? 1 : on_device;
  auto worker = [&](int w) {
    cudaSetDevice(dev);
    mpirg_config c = *cfg;
    c.device = dev;
    mpirg_error e{};
    mpirg_factorization *f = nullptr;
    struct NoPartition  // the batch's handles share the whole GPU (lu.cu)
    {
      NoPartition() { lu_partition_allowed(false); }
      ~NoPartition() { lu_partition_allowed(true); }
    } no_partition;
    int st = mpirg_factorization_create(&f, n, &c, nullptr, src_on_device, &e);
    if (st != MPIRG_OK)
    {
      note(st, e);
      for (int sidx; (sidx = next.fetch_add(1)) < count;)
        status[sidx] = st;
      return;
    }
    cudaStreamWaitEvent(f->stream, start, 0);
    for (int sidx; (sidx = next.fetch_add(1)) < count;)
    {
      const char *as = static_cast<const char *>(a_src) + (size_t)sidx * n * n * tw;
      const char *bs = static_cast<const char *>(b_src) + (size_t)sidx * n * tw;
      rhist_len[sidx] = 0;
      reason[sidx] = MPIRG_ITERATION_LIMIT;
      if (staged)
        cudaStreamWaitEvent(f->stream, stage.ready[sidx / stage.per], 0);
      st = mpirg_factorization_refactor(f, as, src_on_device, &e);
      if (st == MPIRG_OK)
      {
        mpirg_report rep{};
        rep.sol = static_cast<char *>(sol_dst) + (size_t)sidx * n * tw;
        rep.sol_on_device = src_on_device;
        rep.rhist = rhist + (size_t)sidx * hist_capacity;
        rep.dhist = dhist + (size_t)sidx * hist_capacity;
        rep.hist_capacity = hist_capacity;
        st = mpirg_ir_solve(f, bs, src_on_device, tp, &rep, &e);
        rhist_len[sidx] = rep.rhist_len;
        reason[sidx] = rep.reason;
      }
      status[sidx] = st;
      note(st, e);
    }
    cudaEventRecord(ends[w], f->stream);
    cudaEventSynchronize(ends[w]);
    used[w] = 1;
    mpirg_factorization_destroy(f);
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < W; ++w)
    pool.emplace_back(worker, w);
  worker(0);
  for (auto &t : pool)
    t.join();
  if (staged)
  {
    // runs of solved systems only: a failed system's slice of `sol` stays
    // untouched, as on the non-staged path
    bool copied = true;
    for (int lo = 0; lo < count && copied;)
    {
      if (status[lo] != MPIRG_OK)
      {
        ++lo;
        continue;
      }
      int hi = lo;
      while (hi < count && status[hi] == MPIRG_OK)
        ++hi;
      const size_t off = (size_t)lo * n * tw;
      copied = cudaMemcpy(static_cast<char *>(sol) + off, static_cast<char *>(stage.sol) + off,
                          (size_t)(hi - lo) * n * tw, cudaMemcpyDeviceToHost) == cudaSuccess;
      lo = hi;
    }
    if (!copied && first == MPIRG_OK)
    {
      first = MPIRG_ERR_CUDA;
      fill_err(&first_err, MPIRG_ERR_CUDA, "batch: copy of the solutions to the host failed");
    }
  }
  stage.release();
  double ms = 0.0;
  for (int w = 0; w < W; ++w)
  {
    float m = 0.0f;
    if (used[w] && cudaEventElapsedTime(&m, start, ends[w]) == cudaSuccess)
      ms = std::max(ms, (double)m);
    cudaEventDestroy(ends[w]);
  }
  cudaEventDestroy(start);
  if (device_ms)
    *device_ms = ms;
  if (err)
    *err = first == MPIRG_OK ? mpirg_error{} : first_err;
  if (first == MPIRG_OK)
    fill_err(err, MPIRG_OK, "");
  return first;
}

}  // extern "C"


// ---------------------------------------------------------------------------
// Externally factored handles + the per-rank distributed LU (config 5a)
// ---------------------------------------------------------------------------
int mpirg_factorization_cast(mpirg_factorization *f, const void *a, int a_on_device,
                             mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(f->device));
    if (a)
      MPIRG_CUDA_CHECK(cudaMemcpyAsync(f->a_high, a, (size_t)f->n * f->n * f->tw_bytes(),
                                       a_on_device ? cudaMemcpyDeviceToDevice
                                                   : cudaMemcpyHostToDevice,
                                       f->stream));
    if (f->n > 0)
      f->refactor(false);
  });
}

int mpirg_factorization_buffers(mpirg_factorization *f, void **a_low, int **ipiv, int **perm,
                                void **stream)
{
  if (a_low)
    *a_low = f->a_low;
  if (ipiv)
    *ipiv = f->ipiv;
  if (perm)
    *perm = f->perm;
  if (stream)
    *stream = f->stream;
  return MPIRG_OK;
}

int mpirg_factorization_set_factored(mpirg_factorization *f, int singular_col, mpirg_error *err)
{
  return guarded(err, [&] {
    if (singular_col >= 0 && singular_col < f->n)
      throw ApiError{MPIRG_ERR_SINGULAR, "pivot column is exactly zero", singular_col};
  });
}

struct mpirg_dlu
{
  DluPlan plan;
  int device = 0;
  int nb = 0, np = 0, block_cols = 0;
  DevInfo *info = nullptr;
  int *hdr = nullptr;  // scratch for a received header
  void *msg[2] = {nullptr, nullptr};  // step messages of mpirg_dlu_factor (two slots)
  cudaEvent_t packed[2] = {nullptr, nullptr};
};

namespace
{
size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
struct MsgLayout
{
  size_t ipiv, moves, panel, total;
};
MsgLayout msg_layout(const mpirg_dlu *h, int p)
{
  const int n = h->plan.n, k0 = p * h->nb, jb = std::min(h->nb, n - k0);
  MsgLayout m;
  m.ipiv = 16;
  m.moves = al16(m.ipiv + sizeof(int) * (size_t)jb);
  m.panel = al16(m.moves + sizeof(int2) * 2 * (size_t)h->nb);
  m.total = al16(m.panel + elem_size(h->plan.prec) * (size_t)(n - k0) * jb);
  return m;
}
void check_step(const mpirg_dlu *h, int p)
{
  if (p < 0 || p >= h->np)
    throw ApiError{MPIRG_ERR_INVALID_PARAM, "panel index out of range"};
}
}  // namespace

int mpirg_dlu_create(mpirg_dlu **out, int prec, int n, int nb, int nranks, int rank,
                     int block_cols, int device, mpirg_error *err)
{
  *out = nullptr;
  return guarded(err, [&] {
    if (n <= 0)
      throw ApiError{MPIRG_ERR_INVALID_SIZE, "distributed LU needs n > 0"};
    if (prec != B64 && prec != B32 && prec != B16)
      throw ApiError{MPIRG_ERR_INVALID_CONFIG, "unknown factor precision"};
    if (nranks < 1 || rank < 0 || rank >= nranks)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "rank must lie in [0, nranks)"};
    require_gpu();
    if (device >= 0)
      MPIRG_CUDA_CHECK(cudaSetDevice(device));
    const int b = lu_choose_nb(prec, n, nb);
    int bc = block_cols > 0 ? block_cols : std::max(512, b);  // north_star: block 512
    if ((bc & (bc - 1)) != 0 || bc % b != 0)
      throw ApiError{MPIRG_ERR_INVALID_PARAM,
                     "block_cols must be a power of two and a multiple of nb"};
    auto *h = new mpirg_dlu;
    try
    {
      MPIRG_CUDA_CHECK(cudaGetDevice(&h->device));
      dlu_alloc(h->plan, prec, n, b, nranks, rank, bc);
      h->nb = b;
      h->np = h->plan.ws.npanels;
      h->block_cols = bc;
      h->info = dalloc<DevInfo>(1);
      h->hdr = dalloc<int>(4);
    }
    catch (...)
    {
      dlu_free(h->plan);
      if (h->info)
        cudaFree(h->info);
      delete h;
      throw;
    }
    *out = h;
  });
}

void mpirg_dlu_destroy(mpirg_dlu *h)
{
  if (!h)
    return;
  cudaSetDevice(h->device);
  dlu_free(h->plan);
  if (h->info)
    cudaFree(h->info);
  if (h->hdr)
    cudaFree(h->hdr);
  for (int i = 0; i < 2; ++i)
  {
    if (h->msg[i])
      cudaFree(h->msg[i]);
    if (h->packed[i])
      cudaEventDestroy(h->packed[i]);
  }
  delete h;
}

int mpirg_dlu_nb(const mpirg_dlu *h) { return h->nb; }
int mpirg_dlu_npanels(const mpirg_dlu *h) { return h->np; }
int mpirg_dlu_block_cols(const mpirg_dlu *h) { return h->block_cols; }
int mpirg_dlu_owner(const mpirg_dlu *h, int p)
{
  return ((p * h->nb) / h->block_cols) % h->plan.G;
}
size_t mpirg_dlu_msg_bytes(const mpirg_dlu *h, int p) { return msg_layout(h, p).total; }

int mpirg_dlu_begin(mpirg_dlu *h, int *perm, void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    auto s = static_cast<cudaStream_t>(stream);
    reset_info(h->info, s);
    dlu_begin(h->plan, perm, s);
  });
}

int mpirg_dlu_panel(mpirg_dlu *h, void *a, int p, int *ipiv, void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    check_step(h, p);
    if (mpirg_dlu_owner(h, p) != h->plan.r)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "this rank does not own the panel"};
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    dlu_panel(h->plan, a, p, ipiv, h->info, static_cast<cudaStream_t>(stream));
  });
}

// Step message: [nmoves, singular_col | ipiv[jb] | moves[2 nb] | panel rows k0..n-1 x jb].
static void pack_on(mpirg_dlu *h, const void *a, int p, const int *ipiv, void *msg,
                    cudaStream_t s)
{
  const MsgLayout L = msg_layout(h, p);
  const int n = h->plan.n, k0 = p * h->nb, jb = std::min(h->nb, n - k0);
  const size_t es = elem_size(h->plan.prec);
  char *m = static_cast<char *>(msg);
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(m, h->plan.ws.nmoves + p, sizeof(int),
                                   cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(m + 4, &h->info->singular_col, sizeof(int),
                                   cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(m + L.ipiv, ipiv + k0, sizeof(int) * jb,
                                   cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(m + L.moves, h->plan.ws.moves + (size_t)p * 2 * h->nb,
                                   sizeof(int2) * 2 * h->nb, cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpy2DAsync(m + L.panel, (n - k0) * es,
                                     static_cast<const char *>(a) + ((size_t)k0 * n + k0) * es,
                                     (size_t)n * es, (n - k0) * es, jb,
                                     cudaMemcpyDeviceToDevice, s));
}

static void unpack_on(mpirg_dlu *h, void *a, int p, int *ipiv, const void *msg, cudaStream_t s)
{
  const MsgLayout L = msg_layout(h, p);
  const int n = h->plan.n, k0 = p * h->nb, jb = std::min(h->nb, n - k0);
  const size_t es = elem_size(h->plan.prec);
  const char *m = static_cast<const char *>(msg);
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(h->plan.ws.nmoves + p, m, sizeof(int),
                                   cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(h->hdr, m + 4, sizeof(int), cudaMemcpyDeviceToDevice, s));
  dlu_merge_singular(&h->info->singular_col, h->hdr, s);
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(ipiv + k0, m + L.ipiv, sizeof(int) * jb,
                                   cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(h->plan.ws.moves + (size_t)p * 2 * h->nb, m + L.moves,
                                   sizeof(int2) * 2 * h->nb, cudaMemcpyDeviceToDevice, s));
  MPIRG_CUDA_CHECK(cudaMemcpy2DAsync(static_cast<char *>(a) + ((size_t)k0 * n + k0) * es,
                                     (size_t)n * es, m + L.panel, (n - k0) * es,
                                     (n - k0) * es, jb, cudaMemcpyDeviceToDevice, s));
}

int mpirg_dlu_pack(mpirg_dlu *h, const void *a, int p, const int *ipiv, void *msg,
                   void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    check_step(h, p);
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    pack_on(h, a, p, ipiv, msg, static_cast<cudaStream_t>(stream));
  });
}

int mpirg_dlu_unpack(mpirg_dlu *h, void *a, int p, int *ipiv, const void *msg, void *stream,
                     mpirg_error *err)
{
  return guarded(err, [&] {
    check_step(h, p);
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    unpack_on(h, a, p, ipiv, msg, static_cast<cudaStream_t>(stream));
  });
}

// The whole distributed LU of one rank, driven from here so that no host
// round trip sits between a panel and its broadcast: per panel p the owner
// factors it on the critical stream, packs it and the communication stream
// broadcasts it (NCCL over NVLink through `bcast`; the other ranks unpack it
// on their communication stream), then every rank updates its own columns.
// binary32 factors at nb = 64 run the single-GPU LU's paired TMA schedule
// (dlu_f32_*, lu.cu); other precisions the per-step schedule of
// mpirg_dlu_update with the same look-ahead as dist.factor.
int mpirg_dlu_factor(mpirg_dlu *h, void *a, int *ipiv, int *perm, mpirg_bcast_fn bcast,
                     void *ctx, void *stream, int *singular_col, mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    auto caller = static_cast<cudaStream_t>(stream);
    DluPlan &d = h->plan;
    const int np = h->np, G = d.G, r = d.r;
    if (G > 1 && !bcast)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "a multi-rank LU needs a broadcast hook"};
    if (G > 1 && !h->msg[0])
      for (int i = 0; i < 2; ++i)
      {
        h->msg[i] = dalloc_bytes(msg_layout(h, 0).total);  // panel 0 is the tallest
        MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&h->packed[i], cudaEventDisableTiming));
      }
    auto bc = [&](void *msg, int p, int owner, cudaStream_t s) {
      if (bcast(ctx, msg, msg_layout(h, p).total, owner, s) != 0)
        throw ApiError{MPIRG_ERR_NCCL, "broadcast of a factored panel failed"};
    };
    reset_info(h->info, caller);
    if (dlu_f32_supported(d, a))
    {
      dlu_f32_begin(d, a, perm, caller);
      cudaStream_t crit = dlu_f32_crit(d), comm = dlu_f32_comm(d);
      cudaEvent_t *slot_free = static_cast<cudaEvent_t *>(d.cevents);
      for (int p = 0; p < np; ++p)
      {
        const int owner = mpirg_dlu_owner(h, p), sl = p & 1;
        if (owner == r)
        {
          dlu_panel(d, a, p, ipiv, h->info, crit);
          dlu_f32_panel_ready(d, p, crit);
          if (G > 1)
          {
            MPIRG_CUDA_CHECK(cudaStreamWaitEvent(crit, slot_free[sl], 0));
            pack_on(h, a, p, ipiv, h->msg[sl], crit);
            MPIRG_CUDA_CHECK(cudaEventRecord(h->packed[sl], crit));
            MPIRG_CUDA_CHECK(cudaStreamWaitEvent(comm, h->packed[sl], 0));
            bc(h->msg[sl], p, owner, comm);
            MPIRG_CUDA_CHECK(cudaEventRecord(slot_free[sl], comm));
          }
        }
        else
        {
          bc(h->msg[sl], p, owner, comm);
          unpack_on(h, a, p, ipiv, h->msg[sl], comm);
          dlu_f32_panel_ready(d, p, comm);
          MPIRG_CUDA_CHECK(cudaEventRecord(slot_free[sl], comm));
        }
        dlu_f32_step(d, p, perm, owner == r);
      }
      dlu_f32_end(d, caller);
    }
    else
    {
      dlu_begin(d, perm, caller);
      bool early = false;  // panel p was factored during step p-1 (look-ahead)
      for (int p = 0; p < np; ++p)
      {
        const int owner = mpirg_dlu_owner(h, p);
        if (owner == r)
        {
          if (!early)
            dlu_panel(d, a, p, ipiv, h->info, caller);
          if (G > 1)
            pack_on(h, a, p, ipiv, h->msg[0], caller);
        }
        if (G > 1)
        {
          bc(h->msg[0], p, owner, caller);
          if (owner != r)
            unpack_on(h, a, p, ipiv, h->msg[0], caller);
        }
        early = false;
        if (p + 1 < np && mpirg_dlu_owner(h, p + 1) == r)
        {
          dlu_update(d, a, p, 1, perm, caller);
          dlu_panel(d, a, p + 1, ipiv, h->info, caller);
          early = true;
          dlu_update(d, a, p, 2, perm, caller);
        }
        else
          dlu_update(d, a, p, 2, perm, caller);
      }
      dlu_end(d, caller);
    }
    int sc = INT_MAX;
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(&sc, &h->info->singular_col, sizeof(int),
                                     cudaMemcpyDeviceToHost, caller));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(caller));
    if (singular_col)
      *singular_col = sc == INT_MAX ? -1 : sc;
  });
}

int mpirg_dlu_update(mpirg_dlu *h, void *a, int p, int part, int *perm, void *stream,
                     mpirg_error *err)
{
  return guarded(err, [&] {
    check_step(h, p);
    if (part < 0 || part > 2)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "part must be 0, 1 or 2"};
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    dlu_update(h->plan, a, p, part, perm, static_cast<cudaStream_t>(stream));
  });
}

int mpirg_dlu_end(mpirg_dlu *h, void *stream, int *singular_col, mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(h->device));
    auto s = static_cast<cudaStream_t>(stream);
    dlu_end(h->plan, s);
    int sc = INT_MAX;
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(&sc, &h->info->singular_col, sizeof(int),
                                     cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    if (singular_col)
      *singular_col = sc == INT_MAX ? -1 : sc;
  });
}

int mpirg_tc_update(int n, void *a, int k0, int cb, int ce, void *stream, mpirg_error *err)
{
  return guarded(err, [&] {
    if (!tc_update_supported(n, 64) || k0 < 0 || k0 + 64 > n || cb < k0 + 64 || ce > n)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "unsupported TC update geometry"};
    require_gpu();
    TcPlan plan;
    tc_plan_make(plan, a, n);
    launch_gemm_tc(plan, k0, cb, ce, static_cast<cudaStream_t>(stream));
  });
}

int mpirg_tc_gemm(int n, void *a, int r0, int r1, int cb, int ce, int k0, int K, void *stream,
                  mpirg_error *err)
{
  return guarded(err, [&] {
    if (!tc_update_supported(n, 64) || K <= 0 || K % 64 || k0 < 0 || k0 + K > r0 ||
        k0 + K > cb || r1 > n || ce > n || r0 > r1 || cb > ce)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "unsupported TC update geometry"};
    require_gpu();
    TcPlan plan;
    tc_plan_make(plan, a, n);
    tc_gemm(plan, r0, r1, cb, ce, k0, K, static_cast<cudaStream_t>(stream));
  });
}

// GMRES-IR (krylov_ir.hpp; MPFactorization's KrylovKind / basissize arguments,
// mp_structures.hpp:108-151): attaches the Krylov workspace to a handle; every
// later mpirg_ir_solve takes its corrections from the preconditioned GMRES
// instead of the plain substitution (krylov_ir_solve_report).
int mpirg_factorization_enable_krylov(mpirg_factorization *f, int kind, int basissize,
                                      mpirg_error *err)
{
  return guarded(err, [&] {
    MPIRG_CUDA_CHECK(cudaSetDevice(f->device));
    if (kind == MPIRG_KRYLOV_NONE)
    {
      f->free_krylov();
      return;
    }
    if (basissize < 1)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "Krylov basis budget must be at least 1"};
    if (kind != MPIRG_KRYLOV_GMRES && kind != MPIRG_KRYLOV_BICGSTAB)
      throw ApiError{MPIRG_ERR_INVALID_PARAM, "unknown Krylov kind"};
    f->enable_krylov(kind, basissize);
  });
}

int mpirg_factorization_last_khist(const mpirg_factorization *f, int *khist, int capacity,
                                   int *len, int *breakdown)
{
  const int k = (int)f->khist.size();
  for (int i = 0; i < k && i < capacity; ++i)
    khist[i] = f->khist[i];
  if (len)
    *len = k;
  if (breakdown)
    *breakdown = f->kry_breakdown ? 1 : 0;
  return MPIRG_OK;
}
