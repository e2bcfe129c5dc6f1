// Scalar part of the GMRES correction (proj/include/mpir/krylov_ir.hpp:112-160):
// the Givens rotations on one new Hessenberg column and the back substitution
// of the small triangular system, in the working precision on the host.
//
// "Bitwise equal to the reference" means equal to the reference as its own
// build compiles it (GCC, -O3 -march=x86-64-v3, contraction on; oracle/Makefile
// is the source of truth). For these mixed product/sum expressions that build
// makes specific choices, read off its object code and spelled out here with
// explicit fma() so that this file does not depend on compiler flags:
//   t           = fma(cs_i, h_i, sn_i * h_{i+1})
//   h_{i+1}     = fma(-sn_i, h_i, cs_i * h_{i+1})
//   h_jj        = fma(cs_j, ha, sn_j * hb)
//   g_j, g_{j+1} = cs_j * g_j, (-sn_j) * g_j
//   s -= h_il y_l: the loop is vectorised as a fold-left reduction -- rounded
//                 products subtracted in order for the vector part (4 doubles /
//                 8 floats, then a half vector if that many remain), fused
//                 fnmadd for the scalar tail.
// tests/test_gpu_krylov.py holds the whole GPU path against the compiled
// reference bit for bit; reduction_unfused() is shared with the device dot
// products, which follow the same rule (krylov.cu).
#include <cmath>

#include "krylov_host.h"

namespace mpirg
{

int reduction_unfused(int count, int elem_bytes, bool half_step)
{
  const int v = elem_bytes == 8 ? 4 : 8;
  const int rem = count % v;
  int nv = count - rem;
  if (half_step && rem >= v / 2)
    nv += v / 2;
  return nv;
}

template <typename T>
double gmres_rotate(T *hess, int ld, T *cs, T *sn, T *g, int j)
{
  T *col = hess + (size_t)j * ld;  // hess(i, j) = col[i]
  for (int i = 0; i < j; ++i)
  {
    const T h0 = col[i], h1 = col[i + 1];
    col[i] = std::fma(cs[i], h0, sn[i] * h1);
    col[i + 1] = std::fma(-sn[i], h0, cs[i] * h1);
  }
  const T ha = col[j];
  const T hb = col[j + 1];
  const T rr = std::hypot(ha, hb);
  if (rr == T{})
  {
    cs[j] = T(1.0f);
    sn[j] = T{};
  }
  else
  {
    cs[j] = ha / rr;
    sn[j] = hb / rr;
  }
  col[j] = std::fma(cs[j], ha, sn[j] * hb);
  col[j + 1] = T{};
  const T gj = g[j];
  g[j] = cs[j] * gj;
  g[j + 1] = -sn[j] * gj;
  return std::fabs(static_cast<double>(g[j + 1]));
}

template <typename T>
bool gmres_backsolve(const T *hess, int ld, const T *g, T *y, int k)
{
  bool brk = false;
  for (int i = k - 1; i >= 0; --i)
  {
    T s = g[i];
    const int cnt = k - 1 - i;
    const int nv = reduction_unfused(cnt, (int)sizeof(T), true);
    for (int q = 0; q < cnt; ++q)
    {
      const int l = i + 1 + q;
      const T h = hess[(size_t)l * ld + i];
      if (q < nv)
      {
        const volatile T p = h * y[l];  // rounded product, then the subtraction
        s = s - p;
      }
      else
        s = std::fma(-h, y[l], s);
    }
    if (hess[(size_t)i * ld + i] == T{})
    {
      y[i] = T{};
      brk = true;
    }
    else
      y[i] = s / hess[(size_t)i * ld + i];
  }
  return brk;
}

template <typename T>
T host_sqrt(T v)
{
  return std::sqrt(v);
}

template <typename T>
T host_recip(T v)
{
  return T(1.0f) / v;
}

template double gmres_rotate<double>(double *, int, double *, double *, double *, int);
template double gmres_rotate<float>(float *, int, float *, float *, float *, int);
template bool gmres_backsolve<double>(const double *, int, const double *, double *, int);
template bool gmres_backsolve<float>(const float *, int, const float *, float *, int);
template double host_sqrt<double>(double);
template float host_sqrt<float>(float);
template double host_recip<double>(double);
template float host_recip<float>(float);

}  // namespace mpirg
