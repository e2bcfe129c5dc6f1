// Microbenchmark (dev tool, not product): the 128 x 128 diagonal-tile solve of
// trsv.cu by one warp -- the current product scheme against the candidates --
// plus the latencies that bound it (SHFL, FFMA, LDS, VOTE, an L2 hand-off
// between two CTAs). Every variant is checked bit for bit against a one-thread
// sequential solve with div.rn (the reference's order, dense_lu.hpp:112-137).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false trsv_diag.cu -o trsv_diag
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

constexpr int TB = 128;

// ---------------------------------------------------------------- latencies
__global__ void lat_probe(float *out, long long *cyc, const float *gsrc)
{
  __shared__ float sm[1024];
  const int lane = threadIdx.x;
  sm[lane] = (float)((lane * 7 + 1) & 31);
  __syncwarp();
  const int iters = 4096;
  {
    float v = lane;
    int src = (lane * 7) & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      v = __shfl_sync(0xffffffffu, v, (src + i) & 31);
    long long t1 = clock64();
    if (lane == 0)
      cyc[0] = (t1 - t0) * 100 / iters;
    out[lane] = v;
  }
  {
    float v = lane, a = 1.0001f, b = 0.9999f;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i)
      v = __fmaf_rn(v, a, b);
    long long t1 = clock64();
    if (lane == 0)
      cyc[1] = (t1 - t0) * 100 / iters;
    out[32 + lane] = v;
  }
  {
    int idx = lane;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i)
      idx = (int)sm[idx];
    long long t1 = clock64();
    if (lane == 0)
      cyc[2] = (t1 - t0) * 100 / iters;
    out[64 + lane] = idx;
  }
  {
    int p = lane & 1;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i)
      p = __any_sync(0xffffffffu, p ^ (lane == (i & 31))) ? 1 : 0;
    long long t1 = clock64();
    if (lane == 0)
      cyc[3] = (t1 - t0) * 100 / iters;
    out[96 + lane] = p;
  }
  {
    double v = lane, a = 1.0001, b = 0.9999;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i)
      v = __fma_rn(v, a, b);
    long long t1 = clock64();
    if (lane == 0)
      cyc[4] = (t1 - t0) * 100 / iters;
    out[128 + lane] = (float)v;
  }
  {
    // FFMA -> SHFL (uniform source lane) -> FFMA round trip (what one round of the solve pays)
    float v = lane, a = 1.0001f, b = 0.9999f;
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < iters; ++i)
    {
      v = __fmaf_rn(v, a, b);
      v = __shfl_sync(0xffffffffu, v, (i >> 2) & 31);
      v = __fmaf_rn(v, b, a);
    }
    long long t1 = clock64();
    if (lane == 0)
      cyc[5] = (t1 - t0) * 100 / iters;
    out[160 + lane] = v;
  }
  {
    // dependent L2 loads (ld.relaxed.gpu), pointer chase through a zero array
    unsigned long long off = 0;
    const unsigned long long *g = reinterpret_cast<const unsigned long long *>(gsrc);
    long long t0 = clock64();
    for (int i = 0; i < 512; ++i)
    {
      unsigned long long w;
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(g + off + lane) : "memory");
      off = w;
    }
    long long t1 = clock64();
    if (lane == 0)
      cyc[6] = (t1 - t0) * 100 / 512;
    out[192 + lane] = (float)off;
  }
}

// Two CTAs bounce a tagged word through L2: one hand-off = store -> the
// other's polling load sees it. cyc = round trip / 2.
__global__ void pingpong(unsigned long long *w, int iters, long long *cyc)
{
  if (threadIdx.x != 0)
    return;
  const int me = blockIdx.x;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i)
  {
    if ((i & 1) == me)
    {
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(w), "l"((unsigned long long)i) : "memory");
    }
    else
    {
      unsigned long long v;
      do
      {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
      } while (v != (unsigned long long)i);
    }
  }
  long long t1 = clock64();
  if (me == 0)
    cyc[0] = (t1 - t0) * 100 / iters;
}

// ---------------------------------------------------------------- reference
// D[k * TB + i] = F[i][k] (column k, row i), the product's smem layout.
__global__ void ref_solve(const float *D, const float *rhs, float *xl, float *xu)
{
  float x[TB];
  for (int i = 0; i < TB; ++i)
    x[i] = rhs[i];
  for (int k = 0; k < TB; ++k)
    for (int i = k + 1; i < TB; ++i)
      x[i] = __fmaf_rn(-D[k * TB + i], x[k], x[i]);
  for (int i = 0; i < TB; ++i)
    xl[i] = x[i];
  for (int i = 0; i < TB; ++i)
    x[i] = rhs[i];
  for (int k = TB - 1; k >= 0; --k)
  {
    x[k] = __fdiv_rn(x[k], D[k * TB + k]);
    for (int i = k - 1; i >= 0; --i)
      x[i] = __fmaf_rn(-D[k * TB + i], x[k], x[i]);
  }
  for (int i = 0; i < TB; ++i)
    xu[i] = x[i];
}

// ---------------------------------------------------------------- variants
struct Smem
{
  float diag[TB][TB];
  float rhs[TB];
  float xq[TB];
  float xa[TB];
};

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// V0: the product's scheme (trsv.cu diag_solve, FULL, LPL = 4)
template <bool UPPER>
__device__ __forceinline__ void solve_v0(float (&a)[4], const float (*diag)[TB], int lane)
{
  constexpr int LPL = 4, NL = 32;
  float lt[LPL][LPL], ltn[LPL][LPL];
  auto load_lt = [&](int m, float (&dst)[LPL][LPL]) {
#pragma unroll
    for (int f = 0; f < LPL; ++f)
#pragma unroll
      for (int e = 0; e < LPL; ++e)
        dst[f][e] = diag[LPL * m + f][LPL * lane + e];
  };
  float ry[LPL];
#pragma unroll
  for (int e = 0; e < LPL; ++e)
    ry[e] = __frcp_rn(diag[LPL * lane + e][LPL * lane + e]);
  load_lt(UPPER ? NL - 1 : 0, lt);
#pragma unroll 2
  for (int rr = 0; rr < NL; ++rr)
  {
    const int m = UPPER ? NL - 1 - rr : rr;
    if (rr + 1 < NL)
      load_lt(UPPER ? m - 1 : m + 1, ltn);
    float s[LPL], xv[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e)
      s[e] = a[e];
    if constexpr (!UPPER)
    {
#pragma unroll
      for (int e = 0; e < LPL; ++e)
      {
#pragma unroll
        for (int f = 0; f < e; ++f)
          s[e] = __fmaf_rn(-lt[f][e], s[f], s[e]);
        xv[e] = __shfl_sync(0xffffffffu, s[e], m);
      }
    }
    else
    {
#pragma unroll
      for (int e = LPL - 1; e >= 0; --e)
      {
        const float b = lt[e][e], y = ry[e];
        const float q0 = __fmul_rn(s[e], y);
        const float q1 = __fmaf_rn(__fmaf_rn(-b, q0, s[e]), y, q0);
        s[e] = __fmaf_rn(__fmaf_rn(-b, q1, s[e]), y, q1);
#pragma unroll
        for (int f = 0; f < e; ++f)
          s[f] = __fmaf_rn(-lt[e][f], s[e], s[f]);
        xv[e] = __shfl_sync(0xffffffffu, s[e], m);
      }
    }
    const bool later = UPPER ? lane < m : lane > m;
#pragma unroll
    for (int e = 0; e < LPL; ++e)
    {
      float v = a[e];
      if constexpr (!UPPER)
      {
#pragma unroll
        for (int f = 0; f < LPL; ++f)
          v = __fmaf_rn(-lt[f][e], xv[f], v);
      }
      else
      {
#pragma unroll
        for (int f = LPL - 1; f >= 0; --f)
          v = __fmaf_rn(-lt[f][e], xv[f], v);
      }
      a[e] = later ? v : (lane == m ? s[e] : a[e]);
    }
#pragma unroll
    for (int f = 0; f < LPL; ++f)
#pragma unroll
      for (int e = 0; e < LPL; ++e)
        lt[f][e] = ltn[f][e];
  }
}

// V1 forward: no selects on the partial sums (finished lanes keep computing on
// dead values; the owner's results are captured), loads two rounds ahead.
__device__ __forceinline__ void fwd_v1(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
  float mine[4] = {a[0], a[1], a[2], a[3]};
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
    if (m + 1 < 32)
    {
      const float *nb = base + (4 * (m + 1)) * TB;
      n0 = ld4(nb);
      n1 = ld4(nb + TB);
      n2 = ld4(nb + 2 * TB);
      n3 = ld4(nb + 3 * TB);
    }
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = __shfl_sync(0xffffffffu, s0, m);
    const float x1 = __shfl_sync(0xffffffffu, s1, m);
    const float x2 = __shfl_sync(0xffffffffu, s2, m);
    const float x3 = __shfl_sync(0xffffffffu, s3, m);
    if (lane == m)
    {
      mine[0] = s0;
      mine[1] = s1;
      mine[2] = s2;
      mine[3] = s3;
    }
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mine[e];
}


// V3 forward: V1 with the factor entries loaded NS rounds ahead (ring of NS
// register sets, loop unrolled by NS so the ring index is a compile-time value).
template <int NS>
__device__ __forceinline__ void fwd_v3(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float4 c[NS][4];
#pragma unroll
  for (int j = 0; j < NS; ++j)
#pragma unroll
    for (int f = 0; f < 4; ++f)
      c[j][f] = ld4(base + (4 * j + f) * TB);
  float mine[4] = {a[0], a[1], a[2], a[3]};
  for (int m0 = 0; m0 < 32; m0 += NS)
  {
#pragma unroll
    for (int j = 0; j < NS; ++j)
    {
      const int m = m0 + j;
      const float4 c0 = c[j][0], c1 = c[j][1], c2 = c[j][2], c3 = c[j][3];
      const float s0 = a[0];
      const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
      const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
      const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
      const float x0 = __shfl_sync(0xffffffffu, s0, m);
      const float x1 = __shfl_sync(0xffffffffu, s1, m);
      const float x2 = __shfl_sync(0xffffffffu, s2, m);
      const float x3 = __shfl_sync(0xffffffffu, s3, m);
      if (m + NS < 32)
      {
        const float *nb = base + (4 * (m + NS)) * TB;
#pragma unroll
        for (int f = 0; f < 4; ++f)
          c[j][f] = ld4(nb + f * TB);
      }
      if (lane == m)
      {
        mine[0] = s0;
        mine[1] = s1;
        mine[2] = s2;
        mine[3] = s3;
      }
      a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
      a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
      a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
      a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mine[e];
}

// V4 forward: no factor loads at all inside the loop (every lane's entries
// preloaded is impossible: 512 registers), so as a bound: the chain alone with
// the entries of round 0 reused (WRONG results; timing floor only).
__device__ __forceinline__ void fwd_v4(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  const float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = __shfl_sync(0xffffffffu, s0, m);
    const float x1 = __shfl_sync(0xffffffffu, s1, m);
    const float x2 = __shfl_sync(0xffffffffu, s2, m);
    const float x3 = __shfl_sync(0xffffffffu, s3, m);
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
  }
}

// V5/V6: chain-only with NSH of the four broadcasts real (timing only)
template <int NSH>
__device__ __forceinline__ void fwd_v5(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  const float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = NSH >= 4 ? __shfl_sync(0xffffffffu, s0, m) : s0;
    const float x1 = NSH >= 2 ? __shfl_sync(0xffffffffu, s1, m) : s1;
    const float x2 = NSH >= 3 ? __shfl_sync(0xffffffffu, s2, m) : s2;
    const float x3 = __shfl_sync(0xffffffffu, s3, m);
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
  }
}

__device__ __forceinline__ bool exp_mid_f(float v)
{
  const unsigned e = (__float_as_uint(v) >> 23) & 0xffu;
  return e - 67u <= 120u;  // |v| in [2^-60, 2^61)
}

// V1 backward: the division on the chain is ONE fma after the numerator,
//   a = fma(-u, x, p)              (the reference's update: the numerator)
//   c = fma(-(u*yl), x, p*yl)      (alongside: ~ a*yl, the reciprocal's low part)
//   q = fma(a, yh, c)              (~ a*(yh+yl) = a/b to ~2^-47: RN(a/b) unless a/b
//                                   sits within that of a rounding boundary)
// and q is accepted only if one Markstein step leaves it unchanged,
//   fma(fma(-b, q, a), yh, q) == q   (=> q within 1 ulp => that step is RN(a/b)),
// checked per 32-row slice off the chain. Returns true when some quotient
// failed (the caller redoes the block with div.rn).
__device__ __forceinline__ bool bwd_v1(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float b[4], yh[4], yl[4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
  {
    b[e] = diag[4 * lane + e][4 * lane + e];
    yh[e] = __frcp_rn(b[e]);
    yl[e] = __fmul_rn(__fmaf_rn(-b[e], yh[e], 1.0f), yh[e]);
  }
  float4 c0 = ld4(base + (4 * 31) * TB), c1 = ld4(base + (4 * 31 + 1) * TB), c2 = ld4(base + (4 * 31 + 2) * TB),
         c3 = ld4(base + (4 * 31 + 3) * TB);
  float mq[4] = {1.f, 1.f, 1.f, 1.f}, ma[4] = {1.f, 1.f, 1.f, 1.f};
  float a3 = a[3], cc3 = __fmul_rn(a[3], yl[3]);
  bool bad = false;
#pragma unroll 4
  for (int m = 31; m >= 0; --m)
  {
    float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
    if (m > 0)
    {
      const float *nb = base + (4 * (m - 1)) * TB;
      n0 = ld4(nb);
      n1 = ld4(nb + TB);
      n2 = ld4(nb + 2 * TB);
      n3 = ld4(nb + 3 * TB);
    }
    // c_f = column 4m+f of my rows: c_f.x/y/z/w = rows 0..3
    // off-chain products for the triangle
    const float u23yl = __fmul_rn(c3.z, yl[2]);
    const float u12yl = __fmul_rn(c2.y, yl[1]);
    const float u01yl = __fmul_rn(c1.x, yl[0]);
    const float p2yl = __fmul_rn(a[2], yl[2]);
    const float q3 = __fmaf_rn(a3, yh[3], cc3);
    const float a2 = __fmaf_rn(-c3.z, q3, a[2]);
    const float cc2 = __fmaf_rn(-u23yl, q3, p2yl);
    const float p1 = __fmaf_rn(-c3.y, q3, a[1]);
    const float p0a = __fmaf_rn(-c3.x, q3, a[0]);
    const float q2 = __fmaf_rn(a2, yh[2], cc2);
    const float p1yl = __fmul_rn(p1, yl[1]);
    const float a1 = __fmaf_rn(-c2.y, q2, p1);
    const float cc1 = __fmaf_rn(-u12yl, q2, p1yl);
    const float p0 = __fmaf_rn(-c2.x, q2, p0a);
    const float q1 = __fmaf_rn(a1, yh[1], cc1);
    const float p0yl = __fmul_rn(p0, yl[0]);
    const float a0 = __fmaf_rn(-c1.x, q1, p0);
    const float cc0 = __fmaf_rn(-u01yl, q1, p0yl);
    const float q0 = __fmaf_rn(a0, yh[0], cc0);
    const float x3 = __shfl_sync(0xffffffffu, q3, m);
    const float x2 = __shfl_sync(0xffffffffu, q2, m);
    const float x1 = __shfl_sync(0xffffffffu, q1, m);
    const float x0 = __shfl_sync(0xffffffffu, q0, m);
    if (lane == m)
    {
      mq[0] = q0, mq[1] = q1, mq[2] = q2, mq[3] = q3;
      ma[0] = a0, ma[1] = a1, ma[2] = a2, ma[3] = a3;
    }
    // apply columns 4m+3 .. 4m to my rows (descending), row 3's last step in
    // both forms (numerator and low part)
    a[0] = __fmaf_rn(-c0.x, x0, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c3.x, x3, a[0]))));
    a[1] = __fmaf_rn(-c0.y, x0, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c3.y, x3, a[1]))));
    a[2] = __fmaf_rn(-c0.z, x0, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c3.z, x3, a[2]))));
    const float p3 = __fmaf_rn(-c1.w, x1, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c3.w, x3, a[3])));
    const float u30yl = __fmul_rn(c0.w, yl[3]);
    const float p3yl = __fmul_rn(p3, yl[3]);
    a3 = __fmaf_rn(-c0.w, x0, p3);
    cc3 = __fmaf_rn(-u30yl, x0, p3yl);
    a[3] = a3;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    if ((m & 7) == 0)
    {
      // verify the slice just finished (lanes m .. m+7)
      bool ok = true;
#pragma unroll
      for (int e = 0; e < 4; ++e)
      {
        const float r = __fmaf_rn(-b[e], mq[e], ma[e]);
        const float q2v = __fmaf_rn(r, yh[e], mq[e]);
        ok &= (q2v == mq[e]) && exp_mid_f(ma[e]) && exp_mid_f(b[e]);
      }
      bad |= (lane >= m && lane < m + 8) && !ok;
      if (__any_sync(0xffffffffu, bad))
        return true;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mq[e];
  return false;
}

// V2 backward: same as V1 with the 12-cycle division (q0 alongside the
// numerator, one correction on the chain) -- for comparison.
__device__ __forceinline__ bool bwd_v2(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float b[4], y[4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
  {
    b[e] = diag[4 * lane + e][4 * lane + e];
    y[e] = __frcp_rn(b[e]);
  }
  float4 c0 = ld4(base + (4 * 31) * TB), c1 = ld4(base + (4 * 31 + 1) * TB), c2 = ld4(base + (4 * 31 + 2) * TB),
         c3 = ld4(base + (4 * 31 + 3) * TB);
  float mq[4] = {1.f, 1.f, 1.f, 1.f}, ma[4] = {1.f, 1.f, 1.f, 1.f};
  float a3 = a[3], g3 = __fmul_rn(a[3], y[3]);
  bool bad = false;
  auto fin = [](float aa, float g, float bb, float yy) { return __fmaf_rn(__fmaf_rn(-bb, g, aa), yy, g); };
#pragma unroll 4
  for (int m = 31; m >= 0; --m)
  {
    float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
    if (m > 0)
    {
      const float *nb = base + (4 * (m - 1)) * TB;
      n0 = ld4(nb);
      n1 = ld4(nb + TB);
      n2 = ld4(nb + 2 * TB);
      n3 = ld4(nb + 3 * TB);
    }
    const float u23y = __fmul_rn(c3.z, y[2]);
    const float u12y = __fmul_rn(c2.y, y[1]);
    const float u01y = __fmul_rn(c1.x, y[0]);
    const float p2y = __fmul_rn(a[2], y[2]);
    const float q3 = fin(a3, g3, b[3], y[3]);
    const float a2 = __fmaf_rn(-c3.z, q3, a[2]);
    const float g2 = __fmaf_rn(-u23y, q3, p2y);
    const float p1 = __fmaf_rn(-c3.y, q3, a[1]);
    const float p0a = __fmaf_rn(-c3.x, q3, a[0]);
    const float q2 = fin(a2, g2, b[2], y[2]);
    const float p1y = __fmul_rn(p1, y[1]);
    const float a1 = __fmaf_rn(-c2.y, q2, p1);
    const float g1 = __fmaf_rn(-u12y, q2, p1y);
    const float p0 = __fmaf_rn(-c2.x, q2, p0a);
    const float q1 = fin(a1, g1, b[1], y[1]);
    const float p0y = __fmul_rn(p0, y[0]);
    const float a0 = __fmaf_rn(-c1.x, q1, p0);
    const float g0 = __fmaf_rn(-u01y, q1, p0y);
    const float q0 = fin(a0, g0, b[0], y[0]);
    const float x3 = __shfl_sync(0xffffffffu, q3, m);
    const float x2 = __shfl_sync(0xffffffffu, q2, m);
    const float x1 = __shfl_sync(0xffffffffu, q1, m);
    const float x0 = __shfl_sync(0xffffffffu, q0, m);
    if (lane == m)
    {
      mq[0] = q0, mq[1] = q1, mq[2] = q2, mq[3] = q3;
      ma[0] = a0, ma[1] = a1, ma[2] = a2, ma[3] = a3;
    }
    a[0] = __fmaf_rn(-c0.x, x0, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c3.x, x3, a[0]))));
    a[1] = __fmaf_rn(-c0.y, x0, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c3.y, x3, a[1]))));
    a[2] = __fmaf_rn(-c0.z, x0, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c3.z, x3, a[2]))));
    const float p3 = __fmaf_rn(-c1.w, x1, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c3.w, x3, a[3])));
    const float u30y = __fmul_rn(c0.w, y[3]);
    const float p3y = __fmul_rn(p3, y[3]);
    a3 = __fmaf_rn(-c0.w, x0, p3);
    g3 = __fmaf_rn(-u30y, x0, p3y);
    a[3] = a3;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    if ((m & 7) == 0)
    {
      bool ok = true;
#pragma unroll
      for (int e = 0; e < 4; ++e)
      {
        const float r = __fmaf_rn(-b[e], mq[e], ma[e]);
        const float q2v = __fmaf_rn(r, y[e], mq[e]);
        ok &= (q2v == mq[e]) && exp_mid_f(ma[e]) && exp_mid_f(b[e]);
      }
      bad |= (lane >= m && lane < m + 8) && !ok;
      if (__any_sync(0xffffffffu, bad))
        return true;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mq[e];
  return false;
}

// V4 backward: V1 with a minimal instruction count per round: per-row
// constants (yh, yl, u_{r,r+1}*yl_r) computed once and pinned in registers,
// the owner's quotients and numerators captured by two predicated STS.128
// (the verification reads them back per 32-row slice; the results are then
// already in shared memory), range check by min/max of |a|.
__device__ __forceinline__ void pin(float &v) { asm volatile("" : "+f"(v)); }
__device__ __forceinline__ bool bwd_v4(float (&a)[4], const float (*diag)[TB], float *xq, float *xa, int lane)
{
  const float *base = &diag[0][4 * lane];
  float b[4], yh[4], yl[4], uyl[4];
  bool bbad = false;
#pragma unroll
  for (int e = 0; e < 4; ++e)
  {
    b[e] = diag[4 * lane + e][4 * lane + e];
    yh[e] = __frcp_rn(b[e]);
    yl[e] = __fmul_rn(__fmaf_rn(-b[e], yh[e], 1.0f), yh[e]);
    const float un = (4 * lane + e + 1 < TB) ? diag[4 * lane + e + 1][4 * lane + e] : 0.0f;
    uyl[e] = __fmul_rn(un, yl[e]);
    bbad |= !exp_mid_f(b[e]);
    pin(yh[e]);
    pin(yl[e]);
    pin(uyl[e]);
  }
  float4 c0 = ld4(base + (4 * 31) * TB), c1 = ld4(base + (4 * 31 + 1) * TB), c2 = ld4(base + (4 * 31 + 2) * TB),
         c3 = ld4(base + (4 * 31 + 3) * TB);
  float a3 = a[3], cc3 = __fmul_rn(a[3], yl[3]);
  bool bad = false;
#pragma unroll 1
  for (int m8 = 24; m8 >= 0; m8 -= 8)
  {
#pragma unroll
    for (int j = 7; j >= 0; --j)
    {
      const int m = m8 + j;
      float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
      if (m > 0)
      {
        const float *nb = base + (4 * (m - 1)) * TB;
        n0 = ld4(nb);
        n1 = ld4(nb + TB);
        n2 = ld4(nb + 2 * TB);
        n3 = ld4(nb + 3 * TB);
      }
      const float p2yl = __fmul_rn(a[2], yl[2]);
      const float q3 = __fmaf_rn(a3, yh[3], cc3);
      const float a2 = __fmaf_rn(-c3.z, q3, a[2]);
      const float cc2 = __fmaf_rn(-uyl[2], q3, p2yl);
      const float p1 = __fmaf_rn(-c3.y, q3, a[1]);
      const float p0a = __fmaf_rn(-c3.x, q3, a[0]);
      const float q2 = __fmaf_rn(a2, yh[2], cc2);
      const float p1yl = __fmul_rn(p1, yl[1]);
      const float a1 = __fmaf_rn(-c2.y, q2, p1);
      const float cc1 = __fmaf_rn(-uyl[1], q2, p1yl);
      const float p0 = __fmaf_rn(-c2.x, q2, p0a);
      const float q1 = __fmaf_rn(a1, yh[1], cc1);
      const float p0yl = __fmul_rn(p0, yl[0]);
      const float a0 = __fmaf_rn(-c1.x, q1, p0);
      const float cc0 = __fmaf_rn(-uyl[0], q1, p0yl);
      const float q0 = __fmaf_rn(a0, yh[0], cc0);
      const float x3 = __shfl_sync(0xffffffffu, q3, m);
      const float x2 = __shfl_sync(0xffffffffu, q2, m);
      const float x1 = __shfl_sync(0xffffffffu, q1, m);
      const float x0 = __shfl_sync(0xffffffffu, q0, m);
      if (lane == m)
      {
        *reinterpret_cast<float4 *>(xq + 4 * lane) = make_float4(q0, q1, q2, q3);
        *reinterpret_cast<float4 *>(xa + 4 * lane) = make_float4(a0, a1, a2, a3);
      }
      a[0] = __fmaf_rn(-c0.x, x0, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c3.x, x3, a[0]))));
      a[1] = __fmaf_rn(-c0.y, x0, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c3.y, x3, a[1]))));
      a[2] = __fmaf_rn(-c0.z, x0, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c3.z, x3, a[2]))));
      const float p3 = __fmaf_rn(-c1.w, x1, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c3.w, x3, a[3])));
      const float p3yl = __fmul_rn(p3, yl[3]);
      a3 = __fmaf_rn(-c0.w, x0, p3);
      cc3 = __fmaf_rn(-uyl[3], x0, p3yl);
      a[3] = a3;
      c0 = n0;
      c1 = n1;
      c2 = n2;
      c3 = n3;
    }
    // verify the slice just finished (lanes m8 .. m8+7)
    __syncwarp();
    const bool mine = lane >= m8 && lane < m8 + 8;
    const int src = mine ? lane : m8;
    const float4 q = *reinterpret_cast<const float4 *>(xq + 4 * src);
    const float4 na = *reinterpret_cast<const float4 *>(xa + 4 * src);
    const float v0 = __fmaf_rn(__fmaf_rn(-b[0], q.x, na.x), yh[0], q.x);
    const float v1 = __fmaf_rn(__fmaf_rn(-b[1], q.y, na.y), yh[1], q.y);
    const float v2 = __fmaf_rn(__fmaf_rn(-b[2], q.z, na.z), yh[2], q.z);
    const float v3 = __fmaf_rn(__fmaf_rn(-b[3], q.w, na.w), yh[3], q.w);
    const float lo = fminf(fminf(fabsf(na.x), fabsf(na.y)), fminf(fabsf(na.z), fabsf(na.w)));
    const float hi = fmaxf(fmaxf(fabsf(na.x), fabsf(na.y)), fmaxf(fabsf(na.z), fabsf(na.w)));
    // (a NaN numerator fails q == v below)
    const bool ok = v0 == q.x && v1 == q.y && v2 == q.z && v3 == q.w && lo >= 0x1p-60f && hi < 0x1p61f && !bbad;
    bad |= mine && !ok;
    if (__any_sync(0xffffffffu, bad))
      return true;
  }
  const float4 q = *reinterpret_cast<const float4 *>(xq + 4 * lane);
  a[0] = q.x, a[1] = q.y, a[2] = q.z, a[3] = q.w;
  return false;
}

// V8 forward: V1 with the owner's results captured by one predicated STS.128
__device__ __forceinline__ void fwd_v8(float (&a)[4], const float (*diag)[TB], float *xq, int lane)
{
  const float *base = &diag[0][4 * lane];
  float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
    if (m + 1 < 32)
    {
      const float *nb = base + (4 * (m + 1)) * TB;
      n0 = ld4(nb);
      n1 = ld4(nb + TB);
      n2 = ld4(nb + 2 * TB);
      n3 = ld4(nb + 3 * TB);
    }
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = __shfl_sync(0xffffffffu, s0, m);
    const float x1 = __shfl_sync(0xffffffffu, s1, m);
    const float x2 = __shfl_sync(0xffffffffu, s2, m);
    const float x3 = __shfl_sync(0xffffffffu, s3, m);
    if (lane == m)
      *reinterpret_cast<float4 *>(xq + 4 * lane) = make_float4(s0, s1, s2, s3);
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  __syncwarp();
  const float4 q = *reinterpret_cast<const float4 *>(xq + 4 * lane);
  a[0] = q.x, a[1] = q.y, a[2] = q.z, a[3] = q.w;
}

// V9 forward: strips of 8 rounds with the strip's factor entries loaded up
// front into registers (128 per lane), no LDS inside the rounds. In the
// product the four strips would belong to four warps that preload before the
// chain reaches them; here one warp does all four (loads exposed per strip).
__device__ __forceinline__ void fwd_v9(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float mine[4] = {a[0], a[1], a[2], a[3]};
#pragma unroll 1
  for (int s8 = 0; s8 < 32; s8 += 8)
  {
    float4 c[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int f = 0; f < 4; ++f)
        c[j][f] = ld4(base + (4 * (s8 + j) + f) * TB);
#pragma unroll
    for (int j = 0; j < 8; ++j)
    {
      const int m = s8 + j;
      const float4 c0 = c[j][0], c1 = c[j][1], c2 = c[j][2], c3 = c[j][3];
      const float s0 = a[0];
      const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
      const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
      const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
      const float x0 = __shfl_sync(0xffffffffu, s0, m);
      const float x1 = __shfl_sync(0xffffffffu, s1, m);
      const float x2 = __shfl_sync(0xffffffffu, s2, m);
      const float x3 = __shfl_sync(0xffffffffu, s3, m);
      if (lane == m)
      {
        mine[0] = s0;
        mine[1] = s1;
        mine[2] = s2;
        mine[3] = s3;
      }
      a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
      a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
      a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
      a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mine[e];
}

// V10 forward: V1 with per-lane predicated loads (finished lanes load nothing:
// fewer shared-memory wavefronts competing with the shuffles)
__device__ __forceinline__ void fwd_v10(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
  float mine[4] = {a[0], a[1], a[2], a[3]};
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
    if (lane > m)
    {
      const float *nb = base + (4 * (m + 1)) * TB;
      n0 = ld4(nb);
      n1 = ld4(nb + TB);
      n2 = ld4(nb + 2 * TB);
      n3 = ld4(nb + 3 * TB);
    }
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = __shfl_sync(0xffffffffu, s0, m);
    const float x1 = __shfl_sync(0xffffffffu, s1, m);
    const float x2 = __shfl_sync(0xffffffffu, s2, m);
    const float x3 = __shfl_sync(0xffffffffu, s3, m);
    if (lane == m)
    {
      mine[0] = s0;
      mine[1] = s1;
      mine[2] = s2;
      mine[3] = s3;
    }
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mine[e];
}

// V11 forward: V1 with the next round's loads pinned (volatile asm) BEFORE the
// round's triangle and shuffles, so they are not queued behind/with the shuffles.
__device__ __forceinline__ float4 lds4v(const float *p)
{
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ float shflv(float v, int src)
{
  float r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=f"(r) : "f"(v), "r"(src));
  return r;
}
template <int MODE>
__device__ __forceinline__ void fwd_v11(float (&a)[4], const float (*diag)[TB], int lane)
{
  const float *base = &diag[0][4 * lane];
  float4 c0 = ld4(base), c1 = ld4(base + TB), c2 = ld4(base + 2 * TB), c3 = ld4(base + 3 * TB);
  float mine[4] = {a[0], a[1], a[2], a[3]};
#pragma unroll 4
  for (int m = 0; m < 32; ++m)
  {
    const float *nb = base + (4 * ((m + 1) & 31)) * TB;
    float4 n0, n1, n2, n3;
    if (MODE == 0)
    {
      n0 = lds4v(nb);
      n1 = lds4v(nb + TB);
      n2 = lds4v(nb + 2 * TB);
      n3 = lds4v(nb + 3 * TB);
    }
    const float s0 = a[0];
    const float s1 = __fmaf_rn(-c0.y, s0, a[1]);
    const float s2 = __fmaf_rn(-c1.z, s1, __fmaf_rn(-c0.z, s0, a[2]));
    const float s3 = __fmaf_rn(-c2.w, s2, __fmaf_rn(-c1.w, s1, __fmaf_rn(-c0.w, s0, a[3])));
    const float x0 = shflv(s0, m);
    const float x1 = shflv(s1, m);
    const float x2 = shflv(s2, m);
    const float x3 = shflv(s3, m);
    if (lane == m)
    {
      mine[0] = s0;
      mine[1] = s1;
      mine[2] = s2;
      mine[3] = s3;
    }
    a[0] = __fmaf_rn(-c3.x, x3, __fmaf_rn(-c2.x, x2, __fmaf_rn(-c1.x, x1, __fmaf_rn(-c0.x, x0, a[0]))));
    a[1] = __fmaf_rn(-c3.y, x3, __fmaf_rn(-c2.y, x2, __fmaf_rn(-c1.y, x1, __fmaf_rn(-c0.y, x0, a[1]))));
    a[2] = __fmaf_rn(-c3.z, x3, __fmaf_rn(-c2.z, x2, __fmaf_rn(-c1.z, x1, __fmaf_rn(-c0.z, x0, a[2]))));
    a[3] = __fmaf_rn(-c3.w, x3, __fmaf_rn(-c2.w, x2, __fmaf_rn(-c1.w, x1, __fmaf_rn(-c0.w, x0, a[3]))));
    if (MODE == 1)
    {
      // loads after the round's shuffle results were consumed
      n0 = lds4v(nb);
      n1 = lds4v(nb + TB);
      n2 = lds4v(nb + 2 * TB);
      n3 = lds4v(nb + 3 * TB);
    }
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    a[e] = mine[e];
}

template <int VAR>
__global__ void run_variant(const float *D, const float *rhs, float *xout, int reps, long long *cyc, int *nbad)
{
  extern __shared__ __align__(16) unsigned char raw[];
  Smem &sm = *reinterpret_cast<Smem *>(raw);
  for (int i = threadIdx.x; i < TB * TB; i += blockDim.x)
    (&sm.diag[0][0])[i] = D[i];
  for (int i = threadIdx.x; i < TB; i += blockDim.x)
    sm.rhs[i] = rhs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  float a[4];
  int bads = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
  {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      a[e] = sm.rhs[4 * lane + e];
    if constexpr (VAR == 0)
      solve_v0<false>(a, sm.diag, lane);
    else if constexpr (VAR == 1)
      fwd_v1(a, sm.diag, lane);
    else if constexpr (VAR == 2)
      fwd_v3<2>(a, sm.diag, lane);
    else if constexpr (VAR == 3)
      fwd_v3<4>(a, sm.diag, lane);
    else if constexpr (VAR == 4)
      fwd_v4(a, sm.diag, lane);
    else if constexpr (VAR == 5)
      fwd_v5<1>(a, sm.diag, lane);
    else if constexpr (VAR == 6)
      fwd_v5<2>(a, sm.diag, lane);
    else if constexpr (VAR == 7)
      fwd_v5<3>(a, sm.diag, lane);
    else if constexpr (VAR == 10)
      solve_v0<true>(a, sm.diag, lane);
    else if constexpr (VAR == 11)
      bads += bwd_v1(a, sm.diag, lane) ? 1 : 0;
    else if constexpr (VAR == 14)
      bads += bwd_v4(a, sm.diag, sm.xq, sm.xa, lane) ? 1 : 0;
    else if constexpr (VAR == 8)
      fwd_v8(a, sm.diag, sm.xq, lane);
    else if constexpr (VAR == 9)
      fwd_v9(a, sm.diag, lane);
    else if constexpr (VAR == 20)
      fwd_v10(a, sm.diag, lane);
    else if constexpr (VAR == 21)
      fwd_v11<0>(a, sm.diag, lane);
    else if constexpr (VAR == 22)
      fwd_v11<1>(a, sm.diag, lane);
    else if constexpr (VAR == 12)
      bads += bwd_v2(a, sm.diag, lane) ? 1 : 0;
    // keep the loop body alive across reps
    if (a[0] == 12345.678f)
      sm.rhs[0] = a[1];
  }
  long long t1 = clock64();
  if (lane == 0)
  {
    cyc[0] = (t1 - t0) / reps;
    *nbad = bads;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    xout[4 * lane + e] = a[e];
}

// The verified quotient against div.rn on random operand triples
// (p, u, x -> a = fma(-u, x, p); b): counts rejected (sent to div.rn) and
// accepted-but-different (must be 0).
__global__ void check_div(unsigned long long seed, int per_thread, unsigned long long *counts)
{
  unsigned long long s = seed + 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  auto next = [&]() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
  };
  unsigned long long rej = 0, wrong = 0, rej12 = 0, wrong12 = 0;
  for (int i = 0; i < per_thread; ++i)
  {
    const unsigned long long r1 = next(), r2 = next();
    // significands random, exponents within +-20 of each other
    auto mk = [](unsigned bits, int e) {
      return __uint_as_float(((unsigned)(127 + e) << 23) | (bits & 0x7fffffu)) * ((bits >> 23) & 1 ? -1.f : 1.f);
    };
    const float p = mk((unsigned)r1, (int)((r1 >> 32) % 9) - 4);
    const float u = mk((unsigned)(r1 >> 20), (int)((r1 >> 40) % 9) - 4);
    const float x = mk((unsigned)r2, (int)((r2 >> 32) % 9) - 4);
    const float b = mk((unsigned)(r2 >> 20), (int)((r2 >> 40) % 41) - 20);
    const float a = __fmaf_rn(-u, x, p);
    const float want = __fdiv_rn(a, b);
    const float yh = __frcp_rn(b);
    const float yl = __fmul_rn(__fmaf_rn(-b, yh, 1.0f), yh);
    {
      const float c = __fmaf_rn(-__fmul_rn(u, yl), x, __fmul_rn(p, yl));
      const float q = __fmaf_rn(a, yh, c);
      const float qv = __fmaf_rn(__fmaf_rn(-b, q, a), yh, q);
      const bool ok = (qv == q) && exp_mid_f(a) && exp_mid_f(b);
      if (!ok)
        ++rej;
      else if (__float_as_uint(q) != __float_as_uint(want))
        ++wrong;
    }
    {
      const float g = __fmaf_rn(-__fmul_rn(u, yh), x, __fmul_rn(p, yh));
      const float q = __fmaf_rn(__fmaf_rn(-b, g, a), yh, g);
      const float qv = __fmaf_rn(__fmaf_rn(-b, q, a), yh, q);
      const bool ok = (qv == q) && exp_mid_f(a) && exp_mid_f(b);
      if (!ok)
        ++rej12;
      else if (__float_as_uint(q) != __float_as_uint(want))
        ++wrong12;
    }
  }
  atomicAdd(counts + 0, rej);
  atomicAdd(counts + 1, wrong);
  atomicAdd(counts + 2, rej12);
  atomicAdd(counts + 3, wrong12);
}

// ---------------------------------------------------------------- host
static void make_tile(std::vector<float> &D, std::vector<float> &rhs, unsigned seed, bool dominant)
{
  // packed LU (partial pivoting) of a random matrix, as the factor tile
  const int n = TB;
  std::vector<float> A(n * n);
  srand(seed);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      A[i * n + j] = (float)rand() / RAND_MAX * 2.f - 1.f + ((dominant && i == j) ? n * 0.25f : 0.f);
  for (int k = 0; k < n; ++k)
  {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (fabsf(A[i * n + k]) > fabsf(A[p * n + k]))
        p = i;
    if (p != k)
      for (int j = 0; j < n; ++j)
        std::swap(A[k * n + j], A[p * n + j]);
    for (int i = k + 1; i < n; ++i)
    {
      A[i * n + k] /= A[k * n + k];
      for (int j = k + 1; j < n; ++j)
        A[i * n + j] = fmaf(-A[i * n + k], A[k * n + j], A[i * n + j]);
    }
  }
  D.resize(n * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k)
      D[k * n + i] = A[i * n + k];
  rhs.resize(n);
  for (int i = 0; i < n; ++i)
    rhs[i] = (float)rand() / RAND_MAX * 2.f - 1.f;
}

template <int VAR>
static void run(const char *name, const float *dD, const float *drhs, const float *want, float *dx, long long *cyc,
                int *nbad)
{
  cudaFuncSetAttribute(run_variant<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  run_variant<VAR><<<1, 32, sizeof(Smem)>>>(dD, drhs, dx, 1, cyc, nbad);
  cudaDeviceSynchronize();
  float got[TB], ref[TB];
  cudaMemcpy(got, dx, sizeof(got), cudaMemcpyDeviceToHost);
  cudaMemcpy(ref, want, sizeof(ref), cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < TB; ++i)
    diff += memcmp(&got[i], &ref[i], 4) != 0;
  const int bad1 = *nbad;
  run_variant<VAR><<<1, 32, sizeof(Smem)>>>(dD, drhs, dx, 200, cyc, nbad);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s %6lld cyc/block (%5.1f per 4-row round)  mismatches %d  redo %d  %s\n", name, cyc[0], cyc[0] / 32.0,
         diff, bad1, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main()
{
  float *dD, *drhs, *dxl, *dxu, *dx, *out;
  long long *cyc;
  int *nbad;
  unsigned long long *w, *counts;
  cudaMalloc(&dD, TB * TB * 4);
  cudaMalloc(&drhs, TB * 4);
  cudaMalloc(&dxl, TB * 4);
  cudaMalloc(&dxu, TB * 4);
  cudaMalloc(&dx, TB * 4);
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&w, 1 << 20);
  cudaMemset(w, 0, 1 << 20);
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  cudaMallocManaged(&nbad, sizeof(int));
  cudaMallocManaged(&counts, 4 * sizeof(unsigned long long));
  for (int r = 0; r < 2; ++r)
  {
    lat_probe<<<1, 32>>>(out, cyc, reinterpret_cast<const float *>(w));
    cudaDeviceSynchronize();
  }
  printf("latency (cycles): shfl %.1f  ffma %.1f  lds %.1f  vote %.1f  dfma %.1f  ffma+shfl %.1f  L2 ld.relaxed %.1f\n",
         cyc[0] / 100.0, cyc[1] / 100.0, cyc[2] / 100.0, cyc[3] / 100.0, cyc[4] / 100.0, cyc[5] / 100.0,
         cyc[6] / 100.0);
  for (int r = 0; r < 2; ++r)
  {
    cudaMemset(w, 0, 8);
    pingpong<<<2, 32>>>(w, 2000, cyc);
    cudaDeviceSynchronize();
  }
  printf("L2 hand-off (store -> polling load on another SM): %.1f cycles\n", cyc[0] / 100.0);

  for (int dom = 0; dom < 1; ++dom)
  {
    std::vector<float> D, rhs;
    make_tile(D, rhs, 1234 + dom, dom == 1);
    cudaMemcpy(dD, D.data(), TB * TB * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(drhs, rhs.data(), TB * 4, cudaMemcpyHostToDevice);
    ref_solve<<<1, 1>>>(dD, drhs, dxl, dxu);
    cudaDeviceSynchronize();
    printf("tile: %s\n", dom ? "diagonally dominant" : "random, partial pivoting");
    run<0>("forward  V0 (product)", dD, drhs, dxl, dx, cyc, nbad);
    run<1>("forward  V1", dD, drhs, dxl, dx, cyc, nbad);
    run<2>("forward  V3 (2 ahead)", dD, drhs, dxl, dx, cyc, nbad);
    run<3>("forward  V3 (4 ahead)", dD, drhs, dxl, dx, cyc, nbad);
    run<4>("forward  chain only (wrong)", dD, drhs, dxl, dx, cyc, nbad);
    run<5>("forward  chain, 1 shfl (wrong)", dD, drhs, dxl, dx, cyc, nbad);
    run<6>("forward  chain, 2 shfl (wrong)", dD, drhs, dxl, dx, cyc, nbad);
    run<7>("forward  chain, 3 shfl (wrong)", dD, drhs, dxl, dx, cyc, nbad);
    run<10>("backward V0 (product)", dD, drhs, dxu, dx, cyc, nbad);
    run<11>("backward V1 (8-cycle div)", dD, drhs, dxu, dx, cyc, nbad);
    run<12>("backward V2 (12-cycle div)", dD, drhs, dxu, dx, cyc, nbad);
    run<14>("backward V4 (lean V1)", dD, drhs, dxu, dx, cyc, nbad);
    run<9>("forward  V9 (register strips)", dD, drhs, dxl, dx, cyc, nbad);
    run<20>("forward  V10 (predicated LDS)", dD, drhs, dxl, dx, cyc, nbad);
    run<21>("forward  V11 (loads pinned first)", dD, drhs, dxl, dx, cyc, nbad);
    run<22>("forward  V11 (loads pinned last)", dD, drhs, dxl, dx, cyc, nbad);
    run<8>("forward  V8 (STS capture)", dD, drhs, dxl, dx, cyc, nbad);
  }
  memset(counts, 0, 32);
  check_div<<<592, 256>>>(42, 2000, counts);
  cudaDeviceSynchronize();
  const double tot = 592.0 * 256 * 2000;
  printf("verified quotient vs div.rn on %.3g triples: 8-cycle form rejected %llu (%.2e) wrong %llu; "
         "12-cycle form rejected %llu (%.2e) wrong %llu\n",
         tot, counts[0], counts[0] / tot, counts[1], counts[2], counts[2] / tot, counts[3]);
  return 0;
}
