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

#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "mpir_gpu.h"

namespace mpir::gpu
{

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
  NonFiniteResult(const std::string &m, std::vector<double> r, std::vector<double> d)
    : Error(m), rhist(std::move(r)), dhist(std::move(d))
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
      throw NonFiniteResult(m, std::move(rh), std::move(dh));
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
struct Half
{
  std::uint16_t bits = 0;
};
template <typename T> struct precision_of;
template <> struct precision_of<double> : std::integral_constant<int, MPIRG_B64> {};
template <> struct precision_of<float> : std::integral_constant<int, MPIRG_B32> {};
template <> struct precision_of<Half> : std::integral_constant<int, MPIRG_B16> {};

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

struct FactorOptions
{
  bool resid_term = true;
  std::optional<bool> on_the_fly;
};

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
    c.tw = precision_of<TW>::value;
    c.tf = precision_of<TF>::value;
    c.tr = precision_of<TR>::value;
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
  MPFactorization(MPFactorization &&o) noexcept : h_(o.h_) { o.h_ = nullptr; }
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
  mpirg_factorization *handle() { return h_; }

private:
  mpirg_factorization *h_ = nullptr;
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

}  // namespace mpir::gpu
