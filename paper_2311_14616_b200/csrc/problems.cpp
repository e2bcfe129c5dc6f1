// Seeded input generators for the IR hot path (host side, libstdc++ RNG).
//
// These produce the byte-identical inputs that the GPU path, the C oracle and
// the compiled reference all consume. They are not on the timed path.
//
//  * Random matrices follow the reference test fixtures
//    (proj/tests/support/test_support.hpp:17-46): std::mt19937_64(seed) feeding
//    a <random> distribution over doubles, filled column-major (j outer, i
//    inner).
//  * The Green's operator A = I - alpha*G restates proj/src/greens.cpp:11-59
//    (kernel, pinned grid endpoint, trapezoid column weights, assembly in
//    double). Every operation is a lone multiply/subtract/add, so there is no
//    contraction freedom and the result is bitwise the reference's.
//  * matvec_compensated restates proj/include/mpir/matrix.hpp:173-195 in the
//    form GCC emits under the reference flags (-O3 -march=native, FMA
//    contraction): the product feeding two_sum (matrix.hpp:158-164) is
//    contracted into both of its uses.
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/mpir_gpu.h"

extern "C" {

void mpirg_gen_uniform_matrix(int rows, int cols, uint64_t seed, double lo, double hi,
                              double *out)
{
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i)
      out[j * rows + i] = dist(rng);
}

void mpirg_gen_normal_matrix(int rows, int cols, uint64_t seed, double *out)
{
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i)
      out[j * rows + i] = dist(rng);
}

// test_support.hpp:29-36: uniform(-1,1) then a_ii += shift (the reference
// fixture uses shift = 2n; BASELINE config 5b uses shift = n).
void mpirg_gen_diag_dominant(int n, uint64_t seed, double shift, double *out)
{
  mpirg_gen_uniform_matrix(n, n, seed, -1.0, 1.0, out);
  for (int64_t i = 0; i < n; ++i)
    out[i * n + i] = out[i * n + i] + shift;
}

// greens.cpp:11-14
static inline double greens_kernel(double x, double y)
{
  return x > y ? y * (1.0 - x) : x * (1.0 - y);
}

// greens.cpp:16-26 (grid) + 28-43 (matrix) + 48-59 (operator).
void mpirg_gen_greens_operator(int n, double alpha, double *out)
{
  const double h = 1.0 / (n - 1);
  std::vector<double> x(n);
  for (int i = 0; i < n; ++i)
    x[i] = i * h;
  x[n - 1] = 1.0;
  for (int64_t j = 0; j < n; ++j)
  {
    const double w = (j == 0 || j == n - 1) ? 0.5 * h : h;
    double *c = out + j * n;
    for (int64_t i = 0; i < n; ++i)
    {
      const double g = greens_kernel(x[i], x[j]) * w;
      c[i] = -alpha * g;
    }
    c[j] += 1.0;
  }
}

// greens.cpp:61-68
void mpirg_gen_integral_rhs(int n, double alpha, double *out)
{
  const double h = 1.0 / (n - 1);
  for (int i = 0; i < n; ++i)
  {
    const double x = (i == n - 1) ? 1.0 : i * h;
    out[i] = 1.0 - alpha * x * (1.0 - x) * 0.5;
  }
}

// matrix.hpp:173-195, y = A x compensated, FMA-contracted form.
void mpirg_gen_matvec_compensated_f64(int n, const double *a, const double *x, double *y)
{
  std::vector<double> comp(n, 0.0);
  for (int i = 0; i < n; ++i)
    y[i] = 0.0;
  for (int64_t j = 0; j < n; ++j)
  {
    const double *c = a + j * n;
    const double xj = x[j];
    for (int i = 0; i < n; ++i)
    {
      const double s = y[i];
      const double t = std::fma(c[i], xj, s);
      const double z = t - s;
      const double e = (s - (t - z)) + std::fma(c[i], xj, -z);
      comp[i] += e;
      y[i] = t;
    }
  }
  for (int i = 0; i < n; ++i)
    y[i] += comp[i];
}

}  // extern "C"
