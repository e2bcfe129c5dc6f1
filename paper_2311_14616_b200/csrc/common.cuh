// Shared device helpers for the B200 IR hot path (sm_100a).
//
// Arithmetic contract: every kernel reproduces the per-element operation order
// of the reference as compiled with its own flags (GCC, -O3 -march=native:
// c - a*b contracts to one FMA). We therefore spell each such update as an
// explicit __fma_rn / __fmaf_rn and never rely on nvcc's own contraction; all
// other operations use the _rn intrinsics, which nvcc never fuses. binary16
// arithmetic follows half.hpp:285-288: widen to binary32, one binary32
// operation, round back to binary16 (RNE).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace mpirg
{

enum Prec : int
{
  B64 = 0,
  B32 = 1,
  B16 = 2
};

// binary16 storage type (bit pattern); arithmetic through binary32.
struct h16
{
  uint16_t bits;
};

__host__ __device__ inline size_t elem_size(int p) { return p == B64 ? 8 : (p == B32 ? 4 : 2); }

// ---------------------------------------------------------------------------
// binary16 conversions (RNE, subnormals preserved; matches _cvtss_sh / from_float_sw)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float h2f(h16 h) { return __half2float(__ushort_as_half(h.bits)); }
__device__ __forceinline__ h16 f2h(float f) { return h16{__half_as_ushort(__float2half_rn(f))}; }
// double -> binary16 with a single rounding (half.hpp:154-188, from_double_sw).
__device__ __forceinline__ h16 d2h(double d) { return h16{__half_as_ushort(__double2half(d))}; }

// Half ops (half.hpp:285-288).
__device__ __forceinline__ h16 hsub(h16 a, h16 b) { return f2h(__fsub_rn(h2f(a), h2f(b))); }
__device__ __forceinline__ h16 hadd(h16 a, h16 b) { return f2h(__fadd_rn(h2f(a), h2f(b))); }
__device__ __forceinline__ h16 hmul(h16 a, h16 b) { return f2h(__fmul_rn(h2f(a), h2f(b))); }
__device__ __forceinline__ h16 hdiv(h16 a, h16 b) { return f2h(__fdiv_rn(h2f(a), h2f(b))); }

// ---------------------------------------------------------------------------
// Type traits: widen-to-double, abs-as-double, finiteness.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double to_d(double v) { return v; }
__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(h16 v) { return (double)h2f(v); }

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite(float v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite(h16 v) { return (v.bits & 0x7c00u) != 0x7c00u; }

// Promotion of a factor entry into the solve type (precision.hpp:122-145).
template <typename TS, typename TF>
__device__ __forceinline__ TS promote(TF v);
template <> __device__ __forceinline__ double promote<double, double>(double v) { return v; }
template <> __device__ __forceinline__ double promote<double, float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double promote<double, h16>(h16 v) { return (double)h2f(v); }
template <> __device__ __forceinline__ float promote<float, float>(float v) { return v; }
template <> __device__ __forceinline__ float promote<float, h16>(h16 v) { return h2f(v); }
template <> __device__ __forceinline__ h16 promote<h16, h16>(h16 v) { return v; }

// Rounding conversion (demote_val, precision.hpp:156-164). Same type: identity.
template <typename To, typename From>
__device__ __forceinline__ To demote(From v);
template <> __device__ __forceinline__ double demote<double, double>(double v) { return v; }
template <> __device__ __forceinline__ float demote<float, double>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ h16 demote<h16, double>(double v) { return d2h(v); }
template <> __device__ __forceinline__ float demote<float, float>(float v) { return v; }
template <> __device__ __forceinline__ h16 demote<h16, float>(float v) { return f2h(v); }
template <> __device__ __forceinline__ h16 demote<h16, h16>(h16 v) { return v; }

// ---------------------------------------------------------------------------
// The elementary update c - l*u in the factor/solve type T:
//   double/float: one FMA (the reference build contracts it),
//   binary16:     r16(c - r16(l*u)).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double upd(double c, double l, double u) { return __fma_rn(-l, u, c); }
__device__ __forceinline__ float upd(float c, float l, float u) { return __fmaf_rn(-l, u, c); }
__device__ __forceinline__ h16 upd(h16 c, h16 l, h16 u) { return hsub(c, hmul(l, u)); }

__device__ __forceinline__ double divide(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float divide(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ h16 divide(h16 a, h16 b) { return hdiv(a, b); }

// ---------------------------------------------------------------------------
// IEEE division from a precomputed reciprocal, for divisions on a sequential
// critical path whose divisor is known early (the diagonal of U in the back
// substitution). With y = RN(1/b):
//   q0 = RN(a*y)
//   q1 = RN(q0 + RN(a - b*q0) * y)     (both residuals exact: one FMA each)
//   q2 = RN(q1 + RN(a - b*q1) * y)  =  RN(a/b)
// i.e. one multiply and four dependent FMAs instead of MUFU.RCP + the Newton
// sequence + FCHK of div.rn.
//
// Why q2 is the correctly rounded quotient (Markstein, "Computation of
// elementary functions on the IBM RISC System/6000 processor", IBM J. Res.
// Dev. 34(1), 1990, Theorem 1; the form used here is Cornea, Harrison and
// Tang, "Scientific Computing on Itanium-based Systems", 2002, ch. 8, and
// Muller et al., "Handbook of Floating-Point Arithmetic", 2nd ed., Theorem 4.8
// / section 4.7): if y is within one ulp of 1/b (here it is the correctly
// rounded reciprocal, error <= 1/2 ulp) and q is within one ulp of a/b, then
// r = RN(a - b*q) is computed exactly by one FMA and RN(q + r*y) is the
// correctly rounded quotient -- PROVIDED no intermediate underflows, overflows
// or loses bits to gradual underflow. q0 = RN(a*y) is within 3/2 ulp, q1 within
// one ulp, so the theorem applies to the last step. Preconditions as enforced
// here: b normal with |b| in [2^-60, 2^61) (binary32) / [2^-500, 2^501)
// (binary64), so y is normal and b*q cannot overflow; a nonzero with |a| in the
// same window, so a*y, a/b and the residuals a - b*q (which can be as small as
// |a| 2^-24 / 2^-53) stay normal. Zeros (signed-zero results), subnormals,
// infinities and NaN operands, and anything outside the windows take div.rn:
// the caller passes ok = rcp_ok(b) computed with y, div_rcp also checks a, and
// the TRSV diagonal solve redoes a whole block with div.rn when any operand of
// the block was outside (trsv.cu). The identity is additionally checked bit for
// bit against div.rn on 2 x 10^8 operand pairs per precision, including every
// exponent, near-power-of-two and all-ones significands
// (mpirg_check_fast_div, tests/test_gpu_kernels.py).
struct RcpF
{
  float y;
  bool ok;
};
struct RcpD
{
  double y;
  bool ok;
};
__device__ __forceinline__ bool exp_mid_f(float v)
{
  const unsigned e = (__float_as_uint(v) >> 23) & 0xffu;
  return e - 67u <= 120u;  // |v| in [2^-60, 2^61)
}
__device__ __forceinline__ bool exp_mid_d(double v)
{
  const unsigned e = (unsigned)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7ffu;
  return e - 523u <= 1000u;  // |v| in [2^-500, 2^501)
}
__device__ __forceinline__ RcpF make_rcp(float b) { return RcpF{__frcp_rn(b), exp_mid_f(b)}; }
__device__ __forceinline__ RcpD make_rcp(double b) { return RcpD{__drcp_rn(b), exp_mid_d(b)}; }
__device__ __forceinline__ float div_rcp(float a, float b, RcpF r)
{
  if (r.ok && exp_mid_f(a))
  {
    const float q0 = __fmul_rn(a, r.y);
    const float q1 = __fmaf_rn(__fmaf_rn(-b, q0, a), r.y, q0);
    return __fmaf_rn(__fmaf_rn(-b, q1, a), r.y, q1);
  }
  return __fdiv_rn(a, b);
}
__device__ __forceinline__ double div_rcp(double a, double b, RcpD r)
{
  if (r.ok && exp_mid_d(a))
  {
    const double q0 = __dmul_rn(a, r.y);
    const double q1 = __fma_rn(__fma_rn(-b, q0, a), r.y, q0);
    return __fma_rn(__fma_rn(-b, q1, a), r.y, q1);
  }
  return __ddiv_rn(a, b);
}

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }

template <typename T> __device__ __forceinline__ T zero_of();
template <> __device__ __forceinline__ double zero_of<double>() { return 0.0; }
template <> __device__ __forceinline__ float zero_of<float>() { return 0.0f; }
template <> __device__ __forceinline__ h16 zero_of<h16>() { return h16{0}; }

__device__ __forceinline__ double shfl_t(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ float shfl_t(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ h16 shfl_t(h16 v, int src)
{
  return h16{(uint16_t)__shfl_sync(0xffffffffu, (int)v.bits, src)};
}

// ---------------------------------------------------------------------------
// NaN-propagating max of non-negative doubles via the IEEE bit order:
// for x >= 0 (incl. +inf and positive NaN) the uint64 bit patterns are
// monotone and every NaN sorts above +inf. This is norm_inf's semantics
// (matrix.hpp:95-106): NaN sticks, otherwise the max.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long abs_bits(double v)
{
  return (unsigned long long)__double_as_longlong(fabs(v));
}
__device__ __forceinline__ void atomic_max_abs(unsigned long long *slot, double v)
{
  atomicMax(slot, abs_bits(v));
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
  {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// ---------------------------------------------------------------------------
// Acquire/release flag helpers (gpu scope) for sync-free producer/consumer
// kernels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int *p)
{
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_volatile_i32(const int *p)
{
  int v;
  asm volatile("ld.volatile.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v)
{
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Batched launches (config 5b): system z = blockIdx.z of a launch works on
// A + z*a, ipiv/perm + z*vec, moves + z*moves, nmoves + z*nm, info + z.
// All zero (the default) is the single-system launch.
struct BatchStride
{
  size_t a = 0;
  int vec = 0, moves = 0, nm = 0, info = 0;
};

// Device-side error record shared by the kernels of one handle.
struct DevInfo
{
  unsigned long long overflow_index;  // first offending element (storage order), ~0 = none
  int underflow;                      // sticky demotion underflow
  int singular_col;                   // first exactly-zero pivot column, INT_MAX = none
  int nonfinite;                      // substitution produced Inf/NaN
  int pad;
};

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may become resident while
// its predecessor in the stream still runs; pdl_wait() holds it until the
// predecessor has completed and its writes are visible (no-op for a plain
// launch), pdl_trigger() lets the successor become resident early.
__device__ __forceinline__ void pdl_wait()
{
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger()
{
  asm volatile("griddepcontrol.launch_dependents;");
}

}  // namespace mpirg

#define MPIRG_CUDA_CHECK(expr)                                                        \
  do                                                                                  \
  {                                                                                   \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw ::mpirg::CudaError(_e, #expr, __FILE__, __LINE__);                        \
  } while (0)
