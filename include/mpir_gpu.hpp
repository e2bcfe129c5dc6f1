// mpir_gpu.hpp -- header-only C++ twin of the reference API over the C-ABI.
//
// Same names and semantics as the reference (arxiv/paper_2311_14616, proj/):
//   mpir::gpu::MPFactorization<TW,TF,TR>  <- mpir::MPFactorization   mp_structures.hpp:97-213
//   mpir::gpu::mp_lu / mp_refactor        <- mp_structures.hpp:215-237
//   mpir::gpu::ir_solve_report / ir_solve <- ir_engine.hpp:291-304
//   mpir::gpu::residual_tr                <- ir_engine.hpp:277-287
//   TermParams / update_parms / StopReason / SolveReport / FactorOptions
//   exception types                       <- errors.hpp:14-94
// A reference user switches by changing the namespace (and linking
// libmpir_gpu.so). Results are bit-identical to the reference's.
// Element types: double, float, and mpir::gpu::Half (binary16 bits).
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "mpir_gpu.h"

// With MPIR_GPU_USE_REFERENCE_TYPES defined (and the reference's proj/include
// on the include path, -std=c++20) the twin uses the reference's own Matrix,
// Half, TermParams / update_parms, StopReason, FactorOptions, PrecisionConfig
// and exception classes instead of the restatements below, so a reference
// program passes its mpir::Matrix objects straight in and catches the very
// same exception types; only the device-backed classes remain here.
#ifdef MPIR_GPU_USE_REFERENCE_TYPES
#include "mpir/errors.hpp"
#include "mpir/half.hpp"
#include "mpir/ir_engine.hpp"
#include "mpir/matrix.hpp"
#include "mpir/mp_structures.hpp"
#include "mpir/precision.hpp"
#endif

namespace mpir::gpu
{

#ifdef MPIR_GPU_USE_REFERENCE_TYPES
using ::mpir::DimensionMismatch;
using ::mpir::Error;
using ::mpir::FactorOptions;
using ::mpir::Half;
using ::mpir::InvalidConfig;
using ::mpir::InvalidParameter;
using ::mpir::InvalidSize;
using ::mpir::KrylovKind;
using ::mpir::Matrix;
using ::mpir::NonFiniteResult;
using ::mpir::OverflowDetected;
using ::mpir::Precision;
using ::mpir::PrecisionConfig;
using ::mpir::SingularPivot;
using ::mpir::StopReason;
using ::mpir::TermParams;
using ::mpir::update_parms;
#else
// ---- exceptions (errors.hpp) ------------------------------------------------
struct Error : std::runtime_error
{
  using std::runtime_error::runtime_error;
};
struct OverflowDetected : Error
{
  using Error::Error;
};
struct SingularPivot : Error
{
  SingularPivot(const std::string &m, int c) : Error(m), column(c) {}
  int column;
};
struct NonFiniteResult : Error
{
  NonFiniteResult(const std::string &m, std::vector<double> r, std::vector<double> d,
                  std::vector<int> k = {})
    : Error(m), rhist(std::move(r)), dhist(std::move(d)), khist(std::move(k))
  {
  }
  std::vector<double> rhist, dhist;
  std::vector<int> khist;
};
struct DimensionMismatch : Error
{
  using Error::Error;
};
struct InvalidConfig : Error
{
  using Error::Error;
};
struct InvalidParameter : Error
{
  using Error::Error;
};
struct InvalidSize : Error
{
  using Error::Error;
};
#endif
struct CudaError : Error
{
  using Error::Error;
};

inline void throw_status(int st, const mpirg_error &e, std::vector<double> rh = {},
                         std::vector<double> dh = {})
{
  const std::string m(e.message);
  switch (st)
  {
    case MPIRG_OK:
      return;
    case MPIRG_ERR_OVERFLOW:
      throw OverflowDetected(m);
    case MPIRG_ERR_SINGULAR:
      throw SingularPivot(m, e.column);
    case MPIRG_ERR_NONFINITE:
      throw NonFiniteResult(m, std::move(rh), std::move(dh), std::vector<int>{});
    case MPIRG_ERR_DIMENSION:
      throw DimensionMismatch(m);
    case MPIRG_ERR_INVALID_CONFIG:
      throw InvalidConfig(m);
    case MPIRG_ERR_INVALID_PARAM:
      throw InvalidParameter(m);
    case MPIRG_ERR_INVALID_SIZE:
      throw InvalidSize(m);
    default:
      throw CudaError(m);
  }
}

// ---- element types ------------------------------------------------------------
#ifndef MPIR_GPU_USE_REFERENCE_TYPES
struct Half
{
  std::uint16_t bits = 0;
};
#endif
template <typename T> struct prec_code;
template <> struct prec_code<double> : std::integral_constant<int, MPIRG_B64> {};
template <> struct prec_code<float> : std::integral_constant<int, MPIRG_B32> {};
template <> struct prec_code<Half> : std::integral_constant<int, MPIRG_B16> {};

#ifndef MPIR_GPU_USE_REFERENCE_TYPES
// ---- Matrix (matrix.hpp:19-61): column-major --------------------------------------
template <typename T>
class Matrix
{
public:
  Matrix() = default;
  Matrix(int rows, int cols) : rows_(rows), cols_(cols), data_(std::size_t(rows) * cols, T{})
  {
    if (rows < 0 || cols < 0)
      throw InvalidSize("matrix dimensions must be nonnegative");
  }
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  bool square() const { return rows_ == cols_; }
  T &operator()(int i, int j) { return data_[std::size_t(j) * rows_ + i]; }
  const T &operator()(int i, int j) const { return data_[std::size_t(j) * rows_ + i]; }
  T *data() { return data_.data(); }
  const T *data() const { return data_.data(); }
  std::size_t size() const { return data_.size(); }

private:
  int rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

// ---- termination (ir_engine.hpp:29-105) ------------------------------------------
struct TermParams
{
  double cr = 1.0, ce = 1.0, rmax = 0.5;
  int litmax = 10;
};
inline TermParams update_parms(std::optional<double> cr = {}, std::optional<double> ce = {},
                               std::optional<double> rmax = {}, std::optional<int> litmax = {})
{
  TermParams t;
  if (cr)
    t.cr = *cr;
  if (ce)
    t.ce = *ce;
  if (rmax)
    t.rmax = *rmax;
  if (litmax)
    t.litmax = *litmax;
  if (!(t.cr > 0.0) || !std::isfinite(t.cr))
    throw InvalidParameter("cr must be positive and finite");
  if (!(t.ce > 0.0) || !std::isfinite(t.ce))
    throw InvalidParameter("ce must be positive and finite");
  if (!(t.rmax > 0.0) || !(t.rmax <= 1.0))
    throw InvalidParameter("rmax must lie in (0, 1]");
  if (t.litmax < 1)
    throw InvalidParameter("litmax must be at least 1");
  return t;
}

enum class StopReason
{
  SmallResidual,
  SmallBackwardError,
  ResidualStagnation,
  CorrectionStagnation,
  IterationLimit
};

struct FactorOptions
{
  bool resid_term = true;
  std::optional<bool> on_the_fly;
};

// mpir::Precision (precision.hpp:20-25), PrecisionConfig (precision.hpp:210-231),
// KrylovKind (mp_structures.hpp)
enum class Precision
{
  B64,
  B32,
  B16
};
struct PrecisionConfig
{
  Precision tw = Precision::B64;
  Precision tf = Precision::B32;
  Precision tr = Precision::B64;
  bool on_the_fly = false;
  Precision ts() const { return on_the_fly ? tw : tf; }
  void validate() const
  {
    // a smaller code is a wider format
    if (static_cast<int>(tw) > static_cast<int>(tf))
      throw InvalidConfig("factorization precision must not exceed the working precision");
    if (static_cast<int>(tr) > static_cast<int>(tw))
      throw InvalidConfig("residual precision must be at least the working precision");
    if (tf == tw && !on_the_fly)
      throw InvalidConfig("equal-precision factors require on-the-fly solves");
  }
};
enum class KrylovKind
{
  None,
  Gmres,
  Bicgstab
};
#endif

#ifdef MPIR_GPU_USE_REFERENCE_TYPES
template <typename TW>
struct SolveReport : ::mpir::SolveReport<TW>
{
  double device_ms = 0.0;
};
#else
template <typename TW>
struct SolveReport
{
  std::vector<TW> sol;
  std::vector<double> rhist, dhist;
  std::vector<int> khist;
  StopReason reason = StopReason::IterationLimit;
  bool breakdown = false;
  double device_ms = 0.0;
};
#endif

// ---- MPFactorization (mp_structures.hpp:97-213) ------------------------------------
template <typename TW, typename TF, typename TR = TW>
class MPFactorization
{
public:
  using working_type = TW;
  using factor_type = TF;
  using residual_type = TR;

  explicit MPFactorization(const Matrix<TW> &a, FactorOptions opts = {}, int device = -1)
  {
    if (!a.square())
      throw DimensionMismatch("matrix must be square");
    mpirg_config c{};
    c.tw = prec_code<TW>::value;
    c.tf = prec_code<TF>::value;
    c.tr = prec_code<TR>::value;
    c.on_the_fly = opts.on_the_fly ? int(*opts.on_the_fly) : -1;
    c.resid_term = opts.resid_term ? 1 : 0;
    c.lu_mode = MPIRG_LU_EXACT;
    c.nb = 0;
    c.device = device;
    mpirg_error e{};
    throw_status(mpirg_factorization_create(&h_, a.rows(), &c, a.data(), 0, &e), e);
  }
  MPFactorization(const MPFactorization &) = delete;
  MPFactorization &operator=(const MPFactorization &) = delete;
  MPFactorization(MPFactorization &&o) noexcept : h_(o.h_), krylov_(o.krylov_) { o.h_ = nullptr; }
  ~MPFactorization() { mpirg_factorization_destroy(h_); }

  // refactor (mp_structures.hpp:155-169): every device buffer is reused.
  MPFactorization &refactor(const Matrix<TW> &a)
  {
    if (a.rows() != n() || a.cols() != n())
      throw DimensionMismatch("refactor matrix has a different shape");
    mpirg_error e{};
    throw_status(mpirg_factorization_refactor(h_, a.data(), 0, &e), e);
    return *this;
  }

  int n() const { return mpirg_factorization_n(h_); }
  mpirg_config config() const
  {
    mpirg_config c{};
    mpirg_factorization_config(h_, &c);
    return c;
  }
  bool on_the_fly() const { return config().on_the_fly != 0; }
  bool resid_term() const { return config().resid_term != 0; }
  double a_norm1() const { return mpirg_factorization_a_norm1(h_); }
  bool demotion_underflowed() const { return mpirg_factorization_demotion_underflowed(h_); }
  std::size_t matrix_bytes() const { return mpirg_factorization_matrix_bytes(h_); }
  double last_factor_ms() const { return mpirg_factorization_last_factor_ms(h_); }

  // Host mirrors of device state (lazy device->host copies).
  Matrix<TF> packed_lu() const
  {
    Matrix<TF> m(n(), n());
    mpirg_factorization_get_packed_lu(h_, m.data());
    return m;
  }
  Matrix<TW> a_high() const
  {
    Matrix<TW> m(n(), n());
    mpirg_factorization_get_a_high(h_, m.data());
    return m;
  }
  std::vector<int> ipiv() const
  {
    std::vector<int> v(n());
    mpirg_factorization_get_ipiv(h_, v.data());
    return v;
  }
  std::vector<int> pivots() const
  {
    std::vector<int> v(n());
    mpirg_factorization_get_pivots(h_, v.data());
    return v;
  }
  // Preallocated solver state (mp_structures.hpp:186-192) as stable DEVICE
  // pointers, n values each; the refinement loop owns them during a solve.
  // comp_buf is scratch only (the device residual keeps its compensation in
  // registers); low_buf and work_buf alias the one substitution scratch (a
  // configuration uses the scaled TF solve or the promoting TW solve, not both).
  TR *residual_buf() { return static_cast<TR *>(mpirg_factorization_residual_buf_device(h_)); }
  TR *sol_buf() { return static_cast<TR *>(mpirg_factorization_sol_buf_device(h_)); }
  TR *comp_buf() { return static_cast<TR *>(mpirg_factorization_comp_buf_device(h_)); }
  TF *low_buf() { return static_cast<TF *>(mpirg_factorization_low_buf_device(h_)); }
  TW *work_buf() { return static_cast<TW *>(mpirg_factorization_work_buf_device(h_)); }
  // Device views of the matrix copies (column-major n x n) and pivots.
  const TW *a_high_device() const
  {
    return static_cast<const TW *>(mpirg_factorization_a_high_device(h_));
  }
  const TF *packed_lu_device() const
  {
    return static_cast<const TF *>(mpirg_factorization_packed_lu_device(h_));
  }
  const int *ipiv_device() const { return mpirg_factorization_ipiv_device(h_); }
  // The Krylov workspace of mp_structures.hpp:134-151 (the reference passes
  // KrylovKind / basissize to the constructor; mp_glu below does the same).
  void enable_krylov(KrylovKind kind, int basissize)
  {
    mpirg_error e{};
    throw_status(mpirg_factorization_enable_krylov(h_, static_cast<int>(kind), basissize, &e), e);
    krylov_ = kind;
  }
  KrylovKind krylov_kind() const { return krylov_; }
  mpirg_factorization *handle() { return h_; }

private:
  mpirg_factorization *h_ = nullptr;
  KrylovKind krylov_ = KrylovKind::None;
};

template <typename TW, typename TF, typename TR = TW>
MPFactorization<TW, TF, TR> mp_lu(const Matrix<TW> &a, FactorOptions opts = {})
{
  return MPFactorization<TW, TF, TR>(a, opts);
}

template <typename TW, typename TF, typename TR>
MPFactorization<TW, TF, TR> &mp_refactor(MPFactorization<TW, TF, TR> &f, const Matrix<TW> &a)
{
  return f.refactor(a);
}

// ir_solve_report (ir_engine.hpp:291-297)
template <typename TW, typename TF, typename TR>
SolveReport<TW> ir_solve_report(MPFactorization<TW, TF, TR> &f, const std::vector<TW> &b,
                                const TermParams &tp = {})
{
  if (static_cast<int>(b.size()) != f.n())
    throw DimensionMismatch("right-hand side length does not match the matrix");
  SolveReport<TW> rep;
  rep.sol.resize(b.size());
  const int cap = tp.litmax + 1;
  rep.rhist.resize(cap);
  rep.dhist.resize(cap);
  mpirg_report r{};
  r.sol = rep.sol.data();
  r.sol_on_device = 0;
  r.rhist = rep.rhist.data();
  r.dhist = rep.dhist.data();
  r.hist_capacity = cap;
  const mpirg_term_params t{tp.cr, tp.ce, tp.rmax, tp.litmax};
  mpirg_error e{};
  const int st = mpirg_ir_solve(f.handle(), b.data(), 0, &t, &r, &e);
  rep.rhist.resize(r.rhist_len);
  rep.dhist.resize(r.dhist_len);
  throw_status(st, e, rep.rhist, rep.dhist);
  rep.reason = static_cast<StopReason>(r.reason);
  rep.device_ms = r.solve_ms;
  return rep;
}

template <typename TW, typename TF, typename TR>
std::vector<TW> ir_solve(MPFactorization<TW, TF, TR> &f, const std::vector<TW> &b,
                         const TermParams &tp = {})
{
  return ir_solve_report(f, b, tp).sol;
}

// mp_glu (mp_structures.hpp:221-225) and krylov_ir_solve_report
// (krylov_ir.hpp:297-318): GMRES corrections preconditioned by the factors.
template <typename TW, typename TF, typename TR = TW>
MPFactorization<TW, TF, TR> mp_glu(const Matrix<TW> &a, int basissize = 10,
                                   FactorOptions opts = {})
{
  MPFactorization<TW, TF, TR> f(a, opts);
  f.enable_krylov(KrylovKind::Gmres, basissize);
  return f;
}

template <typename TW, typename TF, typename TR>
SolveReport<TW> krylov_ir_solve_report(MPFactorization<TW, TF, TR> &f, const std::vector<TW> &b,
                                       const TermParams &tp = {})
{
  if (f.krylov_kind() == KrylovKind::None)
    throw InvalidConfig("factorization was built without a Krylov workspace");
  SolveReport<TW> rep = ir_solve_report(f, b, tp);
  std::vector<int> kh(tp.litmax + 1);
  int len = 0, brk = 0;
  mpirg_factorization_last_khist(f.handle(), kh.data(), static_cast<int>(kh.size()), &len, &brk);
  kh.resize(len < static_cast<int>(kh.size()) ? len : kh.size());
  rep.khist = kh;
  rep.breakdown = brk != 0;
  return rep;
}

// residual_tr (ir_engine.hpp:277-287)
template <typename TW, typename TF, typename TR>
std::vector<TR> residual_tr(MPFactorization<TW, TF, TR> &f, const std::vector<TW> &x,
                            const std::vector<TW> &b)
{
  if (static_cast<int>(x.size()) != f.n() || static_cast<int>(b.size()) != f.n())
    throw DimensionMismatch("vector length does not match the matrix");
  std::vector<TR> r(x.size());
  mpirg_error e{};
  throw_status(mpirg_residual_tr(f.handle(), x.data(), b.data(), r.data(), 0, &e), e);
  return r;
}

// ---- AnyFactorization (runtime.hpp:34-68, runtime.cpp:67-134) ----------------------
// The type-erased facade the reference's CLI and Python module call. The
// C-ABI is already type-erased, so one handle covers every supported
// precision combination. Input arrives in double and is rounded once into the
// working precision (runtime.cpp:23-28,56-63; demote_checked's overflow rule,
// precision.hpp:172-185).
struct RuntimeReport
{
  std::vector<double> sol, rhist, dhist;
  std::vector<int> khist;
  StopReason reason = StopReason::IterationLimit;
  bool breakdown = false;
  double seconds = 0.0;
};

namespace detail
{
inline std::vector<float> to_b32(const double *v, std::size_t count)
{
  std::vector<float> out(count);
  for (std::size_t i = 0; i < count; ++i)
  {
    const double x = v[i];
    if (std::isfinite(x) && std::fabs(x) > 3.4028234663852886e38)
      throw OverflowDetected("value " + std::to_string(x) +
                             " exceeds the largest finite b32 value");
    out[i] = static_cast<float>(x);
  }
  return out;
}
}  // namespace detail

class AnyFactorization
{
public:
  AnyFactorization(const Matrix<double> &a, const PrecisionConfig &cfg, bool resid_term = true,
                   KrylovKind kind = KrylovKind::None, int basissize = 10, int device = -1)
    : cfg_((cfg.validate(), cfg))  // validated before any allocation (runtime.cpp:69)
  {
    if (kind != KrylovKind::None && basissize < 1)
      throw InvalidParameter("Krylov basis budget must be at least 1");
    if (cfg.tw == Precision::B16)
      throw InvalidConfig("working precision must be b64 or b32");
    if (a.rows() != a.cols())
      throw DimensionMismatch("matrix must be square");
    mpirg_config c{};
    c.tw = static_cast<int>(cfg.tw);
    c.tf = static_cast<int>(cfg.tf);
    c.tr = static_cast<int>(cfg.tr);
    c.on_the_fly = cfg.on_the_fly ? 1 : 0;
    c.resid_term = resid_term ? 1 : 0;
    c.lu_mode = MPIRG_LU_EXACT;
    c.nb = 0;
    c.device = device;
    mpirg_error e{};
    if (cfg.tw == Precision::B64)
      throw_status(mpirg_factorization_create(&h_, a.rows(), &c, a.data(), 0, &e), e);
    else
    {
      const auto a32 = detail::to_b32(a.data(), a.size());
      throw_status(mpirg_factorization_create(&h_, a.rows(), &c, a32.data(), 0, &e), e);
    }
    if (kind != KrylovKind::None)
    {
      const int st = mpirg_factorization_enable_krylov(h_, static_cast<int>(kind), basissize, &e);
      if (st != MPIRG_OK)
      {
        mpirg_factorization_destroy(h_);
        h_ = nullptr;
        throw_status(st, e);
      }
      krylov_ = true;
    }
  }
  AnyFactorization(const AnyFactorization &) = delete;
  AnyFactorization &operator=(const AnyFactorization &) = delete;
  AnyFactorization(AnyFactorization &&o) noexcept : cfg_(o.cfg_), h_(o.h_), krylov_(o.krylov_)
  {
    o.h_ = nullptr;
  }
  ~AnyFactorization() { mpirg_factorization_destroy(h_); }

  int n() const { return mpirg_factorization_n(h_); }
  const PrecisionConfig &config() const { return cfg_; }

  // Iterative refinement (runtime.cpp:78-103).
  RuntimeReport solve(const std::vector<double> &b, const TermParams &tp = {})
  {
    if (static_cast<int>(b.size()) != n())
      throw DimensionMismatch("right-hand side length does not match the matrix");
    RuntimeReport out;
    const int cap = tp.litmax + 1;
    out.rhist.resize(cap > 0 ? cap : 1);
    out.dhist.resize(cap > 0 ? cap : 1);
    std::vector<float> b32, s32;
    out.sol.resize(b.size());
    const bool w64 = cfg_.tw == Precision::B64;
    if (!w64)
    {
      b32 = detail::to_b32(b.data(), b.size());
      s32.resize(b.size());
    }
    mpirg_report r{};
    r.sol = w64 ? static_cast<void *>(out.sol.data()) : static_cast<void *>(s32.data());
    r.sol_on_device = 0;
    r.rhist = out.rhist.data();
    r.dhist = out.dhist.data();
    r.hist_capacity = cap;
    const mpirg_term_params t{tp.cr, tp.ce, tp.rmax, tp.litmax};
    mpirg_error e{};
    const auto t0 = std::chrono::steady_clock::now();
    const int st = mpirg_ir_solve(h_, w64 ? static_cast<const void *>(b.data())
                                          : static_cast<const void *>(b32.data()),
                                  0, &t, &r, &e);
    const auto t1 = std::chrono::steady_clock::now();
    out.rhist.resize(r.rhist_len);
    out.dhist.resize(r.dhist_len);
    throw_status(st, e, out.rhist, out.dhist);
    if (!w64)
      for (std::size_t i = 0; i < s32.size(); ++i)
        out.sol[i] = s32[i];
    out.reason = static_cast<StopReason>(r.reason);
    out.seconds = std::chrono::duration<double>(t1 - t0).count();
    if (krylov_)
    {
      out.khist.resize(cap > 0 ? cap : 1);
      int len = 0, brk = 0;
      mpirg_factorization_last_khist(h_, out.khist.data(), static_cast<int>(out.khist.size()),
                                     &len, &brk);
      out.khist.resize(len < static_cast<int>(out.khist.size()) ? len : out.khist.size());
      out.breakdown = brk != 0;
    }
    return out;
  }

  // Krylov direct solves are outside the B200 hot path.
  std::vector<double> direct_solve(const std::vector<double> &, KrylovKind = KrylovKind::Gmres,
                                   int = 100, double = 1e-10, double * = nullptr)
  {
    throw InvalidParameter("Krylov direct solves are not part of the B200 IR hot path");
  }

  // Reuse the allocation for a new matrix of the same size (runtime.cpp:122-134).
  void refactor(const Matrix<double> &a)
  {
    if (a.rows() != n() || a.cols() != n())
      throw DimensionMismatch("refactor matrix has a different shape");
    mpirg_error e{};
    if (cfg_.tw == Precision::B64)
      throw_status(mpirg_factorization_refactor(h_, a.data(), 0, &e), e);
    else
    {
      const auto a32 = detail::to_b32(a.data(), a.size());
      throw_status(mpirg_factorization_refactor(h_, a32.data(), 0, &e), e);
    }
  }
  mpirg_factorization *handle() { return h_; }

private:
  PrecisionConfig cfg_;
  mpirg_factorization *h_ = nullptr;
  bool krylov_ = false;
};

}  // namespace mpir::gpu
