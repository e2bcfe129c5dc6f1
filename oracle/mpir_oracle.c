/*
 * oracle/mpir_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's mixed-precision IR hot path
 * (arxiv/paper_2311_14616, proj/include/mpir/*.hpp), used as the parity
 * checker for the CUDA path. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * library (paper_2311_14616_b200/libmpir_gpu.so) never links or calls it.
 *
 * Arithmetic order. The reference is built with -O3 -std=gnu++20
 * -march=native (proj/CMakeLists.txt:7-27), under which GCC contracts
 * c - a*b into one fused multiply-add. This file is compiled with
 * -ffp-contract=off and spells every contraction the reference build performs
 * as an explicit fma()/fmaf(); everything else is a single IEEE operation.
 * The restatement is pinned bitwise against the compiled reference
 * (oracle/_ref, built from /root/reference by oracle/Makefile) and the
 * committed golden vectors in tests/golden/.
 *
 * Precision codes: 0 = binary64, 1 = binary32, 2 = binary16 (uint16 bits),
 * as mpir::Precision (precision.hpp:20-25).
 * Status codes: 0 ok, 1 OverflowDetected, 2 SingularPivot, 3 NonFiniteResult,
 * 4 DimensionMismatch, 5 InvalidConfig, 6 InvalidParameter (errors.hpp).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { B64 = 0, B32 = 1, B16 = 2 };
enum { ST_OK = 0, ST_OVERFLOW = 1, ST_SINGULAR = 2, ST_NONFINITE = 3, ST_DIM = 4,
       ST_CONFIG = 5, ST_PARAM = 6 };
enum { R_SMALL_RESIDUAL = 0, R_SMALL_BACKWARD = 1, R_RESID_STAG = 2, R_CORR_STAG = 3,
       R_ITER_LIMIT = 4 };

/* ------------------------------------------------------------------------ */
/* binary16 (half.hpp)                                                       */
/* ------------------------------------------------------------------------ */

static uint32_t f_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint64_t d_bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

/* half.hpp:323-359 (from_float_sw; equals the F16C path by test_precision.cpp:67-92) */
uint16_t orc_f2h(float f)
{
  const uint32_t x = f_bits(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u)
  {
    if (ax > 0x7f800000u)
      return (uint16_t)(sign | 0x7e00u | ((ax >> 13) & 0x3ffu));
    return (uint16_t)(sign | 0x7c00u);
  }
  int e = (int)(ax >> 23) - 127 + 15;
  uint32_t m = ax & 0x7fffffu;
  if (e >= 31)
    return (uint16_t)(sign | 0x7c00u);
  if (e <= 0)
  {
    if (e < -10)
      return (uint16_t)sign;
    m |= 0x800000u;
    const int shift = 14 - e;
    const uint32_t frac = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    uint16_t h = (uint16_t)(sign | frac);
    if (rem > halfway || (rem == halfway && (frac & 1u)))
      ++h;
    return h;
  }
  const uint32_t frac = m >> 13;
  const uint32_t rem = m & 0x1fffu;
  uint16_t h = (uint16_t)(sign | ((uint32_t)e << 10) | frac);
  if (rem > 0x1000u || (rem == 0x1000u && (frac & 1u)))
    ++h;
  return h;
}

/* half.hpp:361-387 */
float orc_h2f(uint16_t h)
{
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1fu;
  uint32_t m = h & 0x3ffu;
  uint32_t out;
  if (e == 31)
    out = sign | 0x7f800000u | (m << 13);
  else if (e == 0)
  {
    if (m == 0)
      out = sign;
    else
    {
      uint32_t e32 = 113;
      while (!(m & 0x400u))
      {
        m <<= 1;
        --e32;
      }
      out = sign | (e32 << 23) | ((m & 0x3ffu) << 13);
    }
  }
  else
    out = sign | ((e + 112) << 23) | (m << 13);
  return bits_f(out);
}

/* half.hpp:389-423 (single rounding from double) */
uint16_t orc_d2h(double d)
{
  const uint64_t x = d_bits(d);
  const uint16_t sign = (uint16_t)((x >> 48) & 0x8000u);
  const uint64_t ax = x & 0x7fffffffffffffffull;
  if (ax >= 0x7ff0000000000000ull)
  {
    if (ax > 0x7ff0000000000000ull)
      return (uint16_t)(sign | 0x7e00u | ((ax >> 42) & 0x3ffu));
    return (uint16_t)(sign | 0x7c00u);
  }
  if (ax == 0)
    return sign;
  int e = (int)(ax >> 52) - 1023 + 15;
  uint64_t m = ax & 0xfffffffffffffull;
  if (e >= 31)
    return (uint16_t)(sign | 0x7c00u);
  int shift = 42;
  if (e <= 0)
  {
    if (e < -10)
      return sign;
    m |= 1ull << 52;
    shift = 43 - e;
    e = 0;
  }
  const uint64_t frac = m >> shift;
  const uint64_t rem = m & ((1ull << shift) - 1ull);
  const uint64_t halfway = 1ull << (shift - 1);
  uint16_t h = (uint16_t)(sign | ((uint32_t)e << 10) | (uint32_t)frac);
  if (rem > halfway || (rem == halfway && (frac & 1ull)))
    ++h;
  return h;
}

/* half.hpp:285-288: widen to binary32, operate, round back. */
static inline uint16_t hsub(uint16_t a, uint16_t b) { return orc_f2h(orc_h2f(a) - orc_h2f(b)); }
static inline uint16_t hadd(uint16_t a, uint16_t b) { return orc_f2h(orc_h2f(a) + orc_h2f(b)); }
static inline uint16_t hmul(uint16_t a, uint16_t b) { return orc_f2h(orc_h2f(a) * orc_h2f(b)); }
static inline uint16_t hdiv(uint16_t a, uint16_t b) { return orc_f2h(orc_h2f(a) / orc_h2f(b)); }
static inline uint16_t habs(uint16_t a) { return (uint16_t)(a & 0x7fffu); }
static inline int hfinite(uint16_t a) { return (a & 0x7c00u) != 0x7c00u; }

static size_t esize(int p) { return p == B64 ? 8 : (p == B32 ? 4 : 2); }

/* Value of element i of an array of precision p, widened exactly to double. */
static inline double ld(int p, const void *v, size_t i)
{
  if (p == B64)
    return ((const double *)v)[i];
  if (p == B32)
    return (double)((const float *)v)[i];
  return (double)orc_h2f(((const uint16_t *)v)[i]);
}

/* precision.hpp:43-67 */
double orc_machine_eps(int p) { return p == B64 ? 0x1p-52 : (p == B32 ? 0x1p-23 : 0x1p-10); }
static double max_finite(int p) { return p == B64 ? DBL_MAX : (p == B32 ? (double)FLT_MAX : 65504.0); }

/* ------------------------------------------------------------------------ */
/* Demotion: demote_matrix_into (matrix.hpp:74-85) + demote_checked          */
/* (precision.hpp:172-185).                                                  */
/* ------------------------------------------------------------------------ */
int orc_demote(int from, int to, size_t count, const void *src, void *dst, int *underflow,
               double *bad_value)
{
  int uf = underflow ? *underflow : 0;
  for (size_t i = 0; i < count; ++i)
  {
    const double x = ld(from, src, i);
    if (isfinite(x) && fabs(x) > max_finite(to))
    {
      if (bad_value)
        *bad_value = x;
      if (underflow)
        *underflow = uf;
      return ST_OVERFLOW;
    }
    double y;
    if (to == from)
    {
      memcpy((char *)dst + i * esize(to), (const char *)src + i * esize(from), esize(to));
      y = x;
    }
    else if (to == B32)
    {
      const float f = (float)((const double *)src)[i]; /* from must be B64 */
      ((float *)dst)[i] = f;
      y = f;
    }
    else /* to == B16 */
    {
      const uint16_t h = from == B64 ? orc_d2h(((const double *)src)[i])
                                     : orc_f2h(((const float *)src)[i]);
      ((uint16_t *)dst)[i] = h;
      y = orc_h2f(h);
    }
    if (!uf && y == 0.0 && x != 0.0)
      uf = 1;
  }
  if (underflow)
    *underflow = uf;
  return ST_OK;
}

/* matrix_one_norm<T> (mp_structures.hpp:22-36): column sums in T. */
double orc_one_norm(int p, int rows, int cols, const void *a)
{
  double best = 0.0;
  for (int64_t j = 0; j < cols; ++j)
  {
    double s_d = 0.0;
    if (p == B64)
    {
      const double *c = (const double *)a + j * rows;
      double s = 0.0;
      for (int i = 0; i < rows; ++i)
        s += fabs(c[i]);
      s_d = s;
    }
    else if (p == B32)
    {
      const float *c = (const float *)a + j * rows;
      float s = 0.0f;
      for (int i = 0; i < rows; ++i)
        s += fabsf(c[i]);
      s_d = s;
    }
    else
    {
      const uint16_t *c = (const uint16_t *)a + j * rows;
      uint16_t s = 0;
      for (int i = 0; i < rows; ++i)
        s = hadd(s, habs(c[i]));
      s_d = orc_h2f(s);
    }
    best = (best < s_d) ? s_d : best; /* std::max(best, s) */
  }
  return best;
}

/* ------------------------------------------------------------------------ */
/* LU: detail::lu_inplace (dense_lu.hpp:50-109). Block/worker counts only    */
/* change traversal order of independent columns, so one sequential form    */
/* covers lu_factor and lu_factor_half.                                      */
/* ------------------------------------------------------------------------ */
#define DEFINE_LU(NAME, T, ABSD, DIV, UPD)                                          \
  static int NAME(T *a, int n, int *ipiv, int *perm, int *singular_col)            \
  {                                                                                \
    for (int i = 0; i < n; ++i)                                                    \
    {                                                                              \
      ipiv[i] = 0;                                                                 \
      if (perm)                                                                    \
        perm[i] = i;                                                               \
    }                                                                              \
    for (int k = 0; k < n; ++k)                                                    \
    {                                                                              \
      T *ck = a + (int64_t)k * n;                                                  \
      int p = k;                                                                   \
      double best = ABSD(ck[k]);                                                   \
      for (int i = k + 1; i < n; ++i)                                              \
      {                                                                            \
        const double v = ABSD(ck[i]);                                              \
        if (v > best)                                                              \
        {                                                                          \
          best = v;                                                                \
          p = i;                                                                   \
        }                                                                          \
      }                                                                            \
      if (best == 0.0)                                                             \
      {                                                                            \
        if (singular_col)                                                          \
          *singular_col = k;                                                       \
        return ST_SINGULAR;                                                        \
      }                                                                            \
      ipiv[k] = p;                                                                 \
      if (p != k)                                                                  \
      {                                                                            \
        for (int64_t j = 0; j < n; ++j)                                            \
        {                                                                          \
          T t = a[j * n + k];                                                      \
          a[j * n + k] = a[j * n + p];                                             \
          a[j * n + p] = t;                                                        \
        }                                                                          \
        if (perm)                                                                  \
        {                                                                          \
          int t = perm[k];                                                         \
          perm[k] = perm[p];                                                       \
          perm[p] = t;                                                             \
        }                                                                          \
      }                                                                            \
      const T piv = ck[k];                                                         \
      for (int i = k + 1; i < n; ++i)                                              \
        ck[i] = DIV(ck[i], piv);                                                   \
      for (int64_t j = k + 1; j < n; ++j)                                          \
      {                                                                            \
        T *cj = a + j * n;                                                         \
        const T ukj = cj[k];                                                       \
        for (int i = k + 1; i < n; ++i)                                            \
          cj[i] = UPD(cj[i], ck[i], ukj);                                          \
      }                                                                            \
    }                                                                              \
    return ST_OK;                                                                  \
  }

#define ABS_D64(x) fabs(x)
#define ABS_D32(x) fabs((double)(x))
#define ABS_D16(x) fabs((double)orc_h2f(x))
#define DIV_NATIVE(a, b) ((a) / (b))
/* c - l*u, contracted by the reference build (dense_lu.hpp:105) */
#define UPD_F64(c, l, u) fma(-(l), (u), (c))
#define UPD_F32(c, l, u) fmaf(-(l), (u), (c))
/* Half: r16(c - r16(l*u)) (half.hpp:285-288) */
#define UPD_F16(c, l, u) hsub((c), hmul((l), (u)))

DEFINE_LU(lu_f64, double, ABS_D64, DIV_NATIVE, UPD_F64)
DEFINE_LU(lu_f32, float, ABS_D32, DIV_NATIVE, UPD_F32)
DEFINE_LU(lu_f16, uint16_t, ABS_D16, hdiv, UPD_F16)

int orc_lu(int p, int n, void *a, int *ipiv, int *perm, int *singular_col)
{
  if (singular_col)
    *singular_col = -1;
  if (p == B64)
    return lu_f64((double *)a, n, ipiv, perm, singular_col);
  if (p == B32)
    return lu_f32((float *)a, n, ipiv, perm, singular_col);
  return lu_f16((uint16_t *)a, n, ipiv, perm, singular_col);
}

/* ------------------------------------------------------------------------ */
/* Blocked building blocks of the 1-D block-cyclic LU (config 5a), used only */
/* by the multi-process CPU tests of the distributed schedule. Restated from */
/* lu_inplace (dense_lu.hpp:63-107) in its blocked right-looking form, whose */
/* per-element FMA order equals the unblocked loop.         */
/*   panel: the column loop restricted to columns [k0, k0+jb); the row swaps */
/*          touch only those columns; the composed swaps are returned as a   */
/*          gather list new[dst] = old[src] (<= 2 jb entries).               */
/*   update: that gather on owned columns outside the panel, then for owned  */
/*          trailing columns U12 = L11^-1 A12 (k ascending) and              */
/*          A22 = fma(-L21, U12, A22) (k ascending).                         */
/* A zero pivot column is recorded (first one) and the step continues with   */
/* p = k, as the device panel does.                                          */
/* ------------------------------------------------------------------------ */
#define DEFINE_DLU(SUF, T, ABSD, DIV, UPD)                                         \
  static void dlu_panel_##SUF(T *a, int n, int k0, int jb, int *ipiv, int *moves,  \
                              int *nmoves, int *singular)                          \
  {                                                                                \
    const int m = n - k0;                                                          \
    int *pp = (int *)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));               \
    for (int i = 0; i < m; ++i)                                                    \
      pp[i] = k0 + i;                                                              \
    for (int k = k0; k < k0 + jb; ++k)                                             \
    {                                                                              \
      T *ck = a + (int64_t)k * n;                                                  \
      int p = k;                                                                   \
      double best = ABSD(ck[k]);                                                   \
      for (int i = k + 1; i < n; ++i)                                              \
      {                                                                            \
        const double v = ABSD(ck[i]);                                              \
        if (v > best)                                                              \
        {                                                                          \
          best = v;                                                                \
          p = i;                                                                   \
        }                                                                          \
      }                                                                            \
      if (best == 0.0 && *singular < 0)                                            \
        *singular = k;                                                             \
      ipiv[k] = p;                                                                 \
      if (p != k)                                                                  \
      {                                                                            \
        for (int64_t j = k0; j < k0 + jb; ++j)                                     \
        {                                                                          \
          T t = a[j * n + k];                                                      \
          a[j * n + k] = a[j * n + p];                                             \
          a[j * n + p] = t;                                                        \
        }                                                                          \
        int t = pp[k - k0];                                                        \
        pp[k - k0] = pp[p - k0];                                                   \
        pp[p - k0] = t;                                                            \
      }                                                                            \
      const T piv = ck[k];                                                         \
      for (int i = k + 1; i < n; ++i)                                              \
        ck[i] = DIV(ck[i], piv);                                                   \
      for (int64_t j = k + 1; j < k0 + jb; ++j)                                    \
      {                                                                            \
        T *cj = a + j * n;                                                         \
        const T ukj = cj[k];                                                       \
        for (int i = k + 1; i < n; ++i)                                            \
          cj[i] = UPD(cj[i], ck[i], ukj);                                          \
      }                                                                            \
    }                                                                              \
    int e = 0;                                                                     \
    for (int i = 0; i < m; ++i)                                                    \
      if (pp[i] != k0 + i)                                                         \
      {                                                                            \
        moves[2 * e] = k0 + i;                                                     \
        moves[2 * e + 1] = pp[i];                                                  \
        ++e;                                                                       \
      }                                                                            \
    *nmoves = e;                                                                   \
    free(pp);                                                                      \
  }                                                                                \
  static void gather_##SUF(T *col, const int *moves, int nm, T *tmp)               \
  {                                                                                \
    for (int e = 0; e < nm; ++e)                                                   \
      tmp[e] = col[moves[2 * e + 1]];                                              \
    for (int e = 0; e < nm; ++e)                                                   \
      col[moves[2 * e]] = tmp[e];                                                  \
  }                                                                                \
  static void dlu_update_##SUF(T *a, int n, int k0, int jb, const int *moves,      \
                               int nm, int G, int r, int sh, int cb, int ce,       \
                               int left)                                           \
  {                                                                                \
    T tmp[256];                                                                    \
    for (int64_t c = 0; c < n; ++c)                                                \
    {                                                                              \
      if (G > 1 && ((int)(c >> sh) % G) != r)                                      \
        continue;                                                                  \
      T *cc = a + c * n;                                                           \
      if (left && c < k0)                                                          \
        gather_##SUF(cc, moves, nm, tmp);                                          \
      if (c < cb || c >= ce)                                                       \
        continue;                                                                  \
      gather_##SUF(cc, moves, nm, tmp);                                            \
      for (int kk = 0; kk < jb; ++kk)                                              \
      {                                                                            \
        const T *lk = a + (int64_t)(k0 + kk) * n;                                  \
        const T x = cc[k0 + kk];                                                   \
        for (int i = k0 + kk + 1; i < k0 + jb; ++i)                                \
          cc[i] = UPD(cc[i], lk[i], x);                                            \
      }                                                                            \
      for (int kk = 0; kk < jb; ++kk)                                              \
      {                                                                            \
        const T *lk = a + (int64_t)(k0 + kk) * n;                                  \
        const T u = cc[k0 + kk];                                                   \
        for (int i = k0 + jb; i < n; ++i)                                          \
          cc[i] = UPD(cc[i], lk[i], u);                                            \
      }                                                                            \
    }                                                                              \
  }

DEFINE_DLU(f64, double, ABS_D64, DIV_NATIVE, UPD_F64)
DEFINE_DLU(f32, float, ABS_D32, DIV_NATIVE, UPD_F32)

int orc_dlu_panel(int p, int n, void *a, int k0, int jb, int *ipiv, int *moves, int *nmoves,
                  int *singular)
{
  if (p == B64)
    dlu_panel_f64((double *)a, n, k0, jb, ipiv, moves, nmoves, singular);
  else if (p == B32)
    dlu_panel_f32((float *)a, n, k0, jb, ipiv, moves, nmoves, singular);
  else
    return ST_CONFIG;
  return ST_OK;
}

/* Owned columns (block 2^sh, block b on rank b mod G) in [cb, ce) get the
 * step's gather + U12 + A22 update; left != 0 also gathers owned columns
 * < k0; perm (optional) is gathered too. */
int orc_dlu_update(int p, int n, void *a, int k0, int jb, const int *moves, int nmoves, int G,
                   int r, int sh, int cb, int ce, int left, int *perm)
{
  if (nmoves > 256)
    return ST_CONFIG;
  if (perm && left)
  {
    int tmp[256];
    for (int e = 0; e < nmoves; ++e)
      tmp[e] = perm[moves[2 * e + 1]];
    for (int e = 0; e < nmoves; ++e)
      perm[moves[2 * e]] = tmp[e];
  }
  if (p == B64)
    dlu_update_f64((double *)a, n, k0, jb, moves, nmoves, G, r, sh, cb, ce, left);
  else if (p == B32)
    dlu_update_f32((float *)a, n, k0, jb, moves, nmoves, G, r, sh, cb, ce, left);
  else
    return ST_CONFIG;
  return ST_OK;
}

/* detail::apply_pivots (dense_lu.hpp:37-44) */
#define DEFINE_PIV(NAME, T)                                                        \
  static void NAME(const int *ipiv, int n, T *x)                                   \
  {                                                                                \
    for (int k = 0; k < n; ++k)                                                    \
      if (ipiv[k] != k)                                                            \
      {                                                                            \
        T t = x[k];                                                                \
        x[k] = x[ipiv[k]];                                                         \
        x[ipiv[k]] = t;                                                            \
      }                                                                            \
  }
DEFINE_PIV(piv_f64, double)
DEFINE_PIV(piv_f32, float)
DEFINE_PIV(piv_f16, uint16_t)

/* ------------------------------------------------------------------------ */
/* Triangular solves trsv_lower_unit / trsv_upper<TS,TF>                     */
/* (dense_lu.hpp:112-137). TS float/double: x_i = fma(-TS(l), x_k, x_i),    */
/* x_k = x_k / TS(u_kk). TS = TF = Half: r16 arithmetic.                     */
/* ------------------------------------------------------------------------ */
#define DEFINE_TRSV(NAME, TS, TF, PROM, FMA)                                       \
  static void NAME(const TF *lu, int n, TS *x)                                     \
  {                                                                                \
    for (int k = 0; k < n; ++k)                                                    \
    {                                                                              \
      const TF *ck = lu + (int64_t)k * n;                                          \
      const TS xk = x[k];                                                          \
      for (int i = k + 1; i < n; ++i)                                              \
        x[i] = FMA(-PROM(ck[i]), xk, x[i]);                                        \
    }                                                                              \
    for (int k = n - 1; k >= 0; --k)                                               \
    {                                                                              \
      const TF *ck = lu + (int64_t)k * n;                                          \
      x[k] = x[k] / PROM(ck[k]);                                                   \
      const TS xk = x[k];                                                          \
      for (int i = 0; i < k; ++i)                                                  \
        x[i] = FMA(-PROM(ck[i]), xk, x[i]);                                        \
    }                                                                              \
  }
#define PROM_ID(v) (v)
#define PROM_D(v) ((double)(v))
#define PROM_H2F(v) orc_h2f(v)
#define PROM_H2D(v) ((double)orc_h2f(v))
DEFINE_TRSV(trsv_d_d, double, double, PROM_ID, fma)
DEFINE_TRSV(trsv_d_f, double, float, PROM_D, fma)
DEFINE_TRSV(trsv_d_h, double, uint16_t, PROM_H2D, fma)
DEFINE_TRSV(trsv_f_f, float, float, PROM_ID, fmaf)
DEFINE_TRSV(trsv_f_h, float, uint16_t, PROM_H2F, fmaf)

static void trsv_h_h(const uint16_t *lu, int n, uint16_t *x)
{
  for (int k = 0; k < n; ++k)
  {
    const uint16_t *ck = lu + (int64_t)k * n;
    const uint16_t xk = x[k];
    for (int i = k + 1; i < n; ++i)
      x[i] = hsub(x[i], hmul(ck[i], xk));
  }
  for (int k = n - 1; k >= 0; --k)
  {
    const uint16_t *ck = lu + (int64_t)k * n;
    x[k] = hdiv(x[k], ck[k]);
    const uint16_t xk = x[k];
    for (int i = 0; i < k; ++i)
      x[i] = hsub(x[i], hmul(ck[i], xk));
  }
}

static int finite_all(int p, const void *x, int n)
{
  for (int i = 0; i < n; ++i)
  {
    if (p == B16)
    {
      if (!hfinite(((const uint16_t *)x)[i]))
        return 0;
    }
    else if (!isfinite(ld(p, x, i)))
      return 0;
  }
  return 1;
}

/* solve_mps_into<TS,TF> (dense_lu.hpp:175-182) */
int orc_solve_mps(int ts, int tf, int n, const void *packed, const int *ipiv, void *x)
{
  if (ts == B64)
  {
    piv_f64(ipiv, n, (double *)x);
    if (tf == B64)
      trsv_d_d((const double *)packed, n, (double *)x);
    else if (tf == B32)
      trsv_d_f((const float *)packed, n, (double *)x);
    else
      trsv_d_h((const uint16_t *)packed, n, (double *)x);
  }
  else if (ts == B32)
  {
    piv_f32(ipiv, n, (float *)x);
    if (tf == B32)
      trsv_f_f((const float *)packed, n, (float *)x);
    else
      trsv_f_h((const uint16_t *)packed, n, (float *)x);
  }
  else
  {
    piv_f16(ipiv, n, (uint16_t *)x);
    trsv_h_h((const uint16_t *)packed, n, (uint16_t *)x);
  }
  return finite_all(ts, x, n) ? ST_OK : ST_NONFINITE;
}

/* solve_lps_into<TW,TF> (dense_lu.hpp:204-232). scratch: n values of TF. */
int orc_solve_lps(int tw, int tf, int n, const void *packed, const int *ipiv, void *r_to_d,
                  void *scratch, int *underflow)
{
  double rho;
  if (tw == B64)
  {
    double *r = (double *)r_to_d;
    double m = 0.0;
    for (int i = 0; i < n; ++i)
    {
      const double a = r[i] < 0.0 ? -r[i] : r[i];
      if (a > m)
        m = a;
    }
    if (m == 0.0)
    {
      for (int i = 0; i < n; ++i)
        r[i] = 0.0;
      return ST_OK;
    }
    rho = m;
    int uf = underflow ? *underflow : 0;
    for (int i = 0; i < n; ++i)
    {
      const double s = r[i] / m;
      double y;
      if (tf == B32)
      {
        ((float *)scratch)[i] = (float)s;
        y = ((float *)scratch)[i];
      }
      else
      {
        ((uint16_t *)scratch)[i] = orc_d2h(s);
        y = orc_h2f(((uint16_t *)scratch)[i]);
      }
      if (!uf && y == 0.0 && s != 0.0)
        uf = 1;
    }
    if (underflow)
      *underflow = uf;
  }
  else /* tw == B32, tf == B16 */
  {
    float *r = (float *)r_to_d;
    float m = 0.0f;
    for (int i = 0; i < n; ++i)
    {
      const float a = r[i] < 0.0f ? -r[i] : r[i];
      if (a > m)
        m = a;
    }
    if (m == 0.0f)
    {
      for (int i = 0; i < n; ++i)
        r[i] = 0.0f;
      return ST_OK;
    }
    rho = m;
    int uf = underflow ? *underflow : 0;
    for (int i = 0; i < n; ++i)
    {
      const float s = r[i] / m;
      ((uint16_t *)scratch)[i] = orc_f2h(s);
      if (!uf && orc_h2f(((uint16_t *)scratch)[i]) == 0.0f && s != 0.0f)
        uf = 1;
    }
    if (underflow)
      *underflow = uf;
  }
  if (tf == B32)
  {
    piv_f32(ipiv, n, (float *)scratch);
    trsv_f_f((const float *)packed, n, (float *)scratch);
  }
  else
  {
    piv_f16(ipiv, n, (uint16_t *)scratch);
    trsv_h_h((const uint16_t *)packed, n, (uint16_t *)scratch);
  }
  if (tw == B64)
  {
    double *r = (double *)r_to_d;
    for (int i = 0; i < n; ++i)
      r[i] = ld(tf, scratch, i) * rho;
  }
  else
  {
    float *r = (float *)r_to_d;
    const float rf = (float)rho;
    for (int i = 0; i < n; ++i)
      r[i] = orc_h2f(((uint16_t *)scratch)[i]) * rf;
  }
  return finite_all(tw, r_to_d, n) ? ST_OK : ST_NONFINITE;
}

/* ------------------------------------------------------------------------ */
/* Residual: detail::residual_into<TW,TR> (ir_engine.hpp:115-139) with the   */
/* two_sum of matrix.hpp:158-164 as contracted by the reference build:       */
/*   t = fma(-a, x, s); z = t - s; e = (s - (t - z)) + fma(-a, x, -z).       */
/* ------------------------------------------------------------------------ */
static void residual_dd(int n, const double *a, const double *x, const double *b, double *r,
                        double *comp)
{
  for (int i = 0; i < n; ++i)
  {
    r[i] = b[i];
    comp[i] = 0.0;
  }
  for (int64_t j = 0; j < n; ++j)
  {
    const double xj = x[j];
    const double *c = a + j * n;
    for (int i = 0; i < n; ++i)
    {
      const double s = r[i];
      const double t = fma(-c[i], xj, s);
      const double z = t - s;
      const double e = (s - (t - z)) + fma(-c[i], xj, -z);
      comp[i] += e;
      r[i] = t;
    }
  }
  for (int i = 0; i < n; ++i)
    r[i] += comp[i];
}

static void residual_fd(int n, const float *a, const double *x, const float *b, double *r,
                        double *comp)
{
  for (int i = 0; i < n; ++i)
  {
    r[i] = (double)b[i];
    comp[i] = 0.0;
  }
  for (int64_t j = 0; j < n; ++j)
  {
    const double xj = x[j];
    const float *c = a + j * n;
    for (int i = 0; i < n; ++i)
    {
      const double s = r[i];
      const double av = (double)c[i];
      const double t = fma(-av, xj, s);
      const double z = t - s;
      const double e = (s - (t - z)) + fma(-av, xj, -z);
      comp[i] += e;
      r[i] = t;
    }
  }
  for (int i = 0; i < n; ++i)
    r[i] += comp[i];
}

static void residual_ff(int n, const float *a, const float *x, const float *b, float *r,
                        float *comp)
{
  for (int i = 0; i < n; ++i)
  {
    r[i] = b[i];
    comp[i] = 0.0f;
  }
  for (int64_t j = 0; j < n; ++j)
  {
    const float xj = x[j];
    const float *c = a + j * n;
    for (int i = 0; i < n; ++i)
    {
      const float s = r[i];
      const float t = fmaf(-c[i], xj, s);
      const float z = t - s;
      const float e = (s - (t - z)) + fmaf(-c[i], xj, -z);
      comp[i] += e;
      r[i] = t;
    }
  }
  for (int i = 0; i < n; ++i)
    r[i] += comp[i];
}

int orc_residual(int tw, int tr, int n, const void *a, const void *x, const void *b, void *r)
{
  void *comp = malloc((size_t)n * esize(tr));
  if (tw == B64)
    residual_dd(n, (const double *)a, (const double *)x, (const double *)b, (double *)r,
                (double *)comp);
  else if (tr == B64)
    residual_fd(n, (const float *)a, (const double *)x, (const float *)b, (double *)r,
                (double *)comp);
  else
    residual_ff(n, (const float *)a, (const float *)x, (const float *)b, (float *)r,
                (float *)comp);
  free(comp);
  return ST_OK;
}

/* norm_inf (matrix.hpp:95-106): NaN sticks. */
double orc_norm_inf(int p, const void *v, int n)
{
  double m = 0.0;
  for (int i = 0; i < n; ++i)
  {
    const double a = fabs(ld(p, v, i));
    if (a > m || isnan(a))
      m = a;
  }
  return m;
}

/* ------------------------------------------------------------------------ */
/* Refinement: MPFactorization ctor/refactor (mp_structures.hpp:108-169),   */
/* plain_correction (ir_engine.hpp:144-181), refine_loop (186-271).          */
/* a and b are TW arrays; sol receives TW; packed (optional) receives TF.   */
/* ------------------------------------------------------------------------ */
static int valid_config(int tw, int tf, int tr, int otf)
{
  /* precision.hpp:222-230 with at_least_as_wide = (code <= code) */
  if (!(tw <= tf))
    return 0;
  if (!(tr <= tw))
    return 0;
  if (tf == tw && !otf)
    return 0;
  return 1;
}

int orc_ir(int tw, int tf, int tr, int on_the_fly, int resid_term, int n, const void *a,
           const void *b, double cr, double ce, double rmax, int litmax, void *sol,
           double *rhist, double *dhist, int *rhist_len, int *reason, int *ipiv,
           void *packed, double *a_norm1, int *underflowed, int *singular_col,
           double *bad_value)
{
  *rhist_len = 0;
  if (tw == B16)
    return ST_CONFIG;
  int otf = on_the_fly < 0 ? (tf == B16 || tf == tw) : on_the_fly;
  if (tf == tw)
    otf = 1;
  if (!valid_config(tw, tf, tr, otf))
    return ST_CONFIG;
  if (!(cr > 0.0) || !isfinite(cr) || !(ce > 0.0) || !isfinite(ce) || !(rmax > 0.0) ||
      !(rmax <= 1.0) || litmax < 1)
    return ST_PARAM;

  /* refactor: one-norm in TW, demote into TF, LU in place. */
  const size_t nn = (size_t)n * n;
  void *low = packed ? packed : malloc(nn * esize(tf));
  *a_norm1 = orc_one_norm(tw, n, n, a);
  int uf = 0;
  int st = orc_demote(tw, tf, nn, a, low, &uf, bad_value);
  *underflowed = uf;
  if (st != ST_OK)
  {
    if (!packed)
      free(low);
    return st;
  }
  int *piv = ipiv ? ipiv : (int *)malloc(sizeof(int) * n);
  st = orc_lu(tf, n, low, piv, NULL, singular_col);
  if (st != ST_OK)
  {
    if (!packed)
      free(low);
    if (!ipiv)
      free(piv);
    return st;
  }

  /* refine_loop */
  const int ext = tr != tw;
  const size_t rs = esize(tr);
  void *x = calloc((size_t)n, rs);
  void *r = malloc((size_t)n * rs);
  void *w = malloc((size_t)n * esize(tw));
  void *scr = malloc((size_t)n * esize(tf));
  for (int i = 0; i < n; ++i)
  {
    if (tr == B64)
      ((double *)r)[i] = ld(tw, b, i);
    else
      ((float *)r)[i] = ((const float *)b)[i];
  }
  const double bnorm = orc_norm_inf(tr, r, n);
  int nr = 0, nd = 0;
  rhist[nr++] = bnorm;
  st = ST_OK;
  if (!isfinite(bnorm))
  {
    st = ST_NONFINITE;
    goto done;
  }
  const double eps_w = orc_machine_eps(tw);
  double rnorm = bnorm;
  for (;;)
  {
    double dnorm;
    /* plain_correction */
    if (!ext)
    {
      if (otf)
        st = orc_solve_mps(tw, tf, n, low, piv, r);
      else
        st = orc_solve_lps(tw, tf, n, low, piv, r, scr, NULL);
      if (st != ST_OK)
        goto done;
      if (tr == B64)
        for (int i = 0; i < n; ++i)
          ((double *)x)[i] += ((double *)r)[i];
      else
        for (int i = 0; i < n; ++i)
          ((float *)x)[i] += ((float *)r)[i];
      dnorm = orc_norm_inf(tr, r, n);
    }
    else if (otf)
    {
      /* tr = B64, tw = B32 */
      for (int i = 0; i < n; ++i)
        ((float *)w)[i] = (float)((double *)r)[i];
      st = orc_solve_mps(tw, tf, n, low, piv, w);
      if (st != ST_OK)
        goto done;
      for (int i = 0; i < n; ++i)
        ((double *)x)[i] += (double)((float *)w)[i];
      dnorm = orc_norm_inf(tw, w, n);
    }
    else
    {
      st = orc_solve_lps(tr, tf, n, low, piv, r, scr, NULL);
      if (st != ST_OK)
        goto done;
      for (int i = 0; i < n; ++i)
        ((double *)x)[i] += ((double *)r)[i];
      dnorm = orc_norm_inf(tr, r, n);
    }
    dhist[nd++] = dnorm;
    orc_residual(tw, tr, n, a, x, b, r);
    const double rnew = orc_norm_inf(tr, r, n);
    rhist[nr++] = rnew;
    if (!isfinite(rnew) || !isfinite(dnorm))
    {
      st = ST_NONFINITE;
      goto done;
    }
    if (!ext)
    {
      const int small = resid_term
                            ? rnew <= cr * eps_w * bnorm
                            /* GCC contracts bnorm + a_norm1*||x|| under the reference's
                               flags (verified on the -O3 -march build): one fma */
                            : rnew <= ce * eps_w * fma(*a_norm1, orc_norm_inf(tr, x, n), bnorm);
      if (small)
      {
        *reason = resid_term ? R_SMALL_RESIDUAL : R_SMALL_BACKWARD;
        break;
      }
      if (rnew >= rmax * rnorm)
      {
        *reason = R_RESID_STAG;
        break;
      }
    }
    else if (nd >= 2 && dhist[nd - 1] >= rmax * dhist[nd - 2])
    {
      *reason = R_CORR_STAG;
      break;
    }
    if (nr >= litmax)
    {
      *reason = R_ITER_LIMIT;
      break;
    }
    rnorm = rnew;
  }
  for (int i = 0; i < n; ++i)
  {
    if (tw == B64)
      ((double *)sol)[i] = ((double *)x)[i];
    else if (tr == B64)
      ((float *)sol)[i] = (float)((double *)x)[i];
    else
      ((float *)sol)[i] = ((float *)x)[i];
  }
done:
  *rhist_len = nr;
  free(x);
  free(r);
  free(w);
  free(scr);
  if (!packed)
    free(low);
  if (!ipiv)
    free(piv);
  return st;
}
