// GMRES-IR corrections on the device, bitwise equal to
// gmres_correction_into (proj/include/mpir/krylov_ir.hpp:62-171) as the
// reference build runs it:
//   v0 = M^-1 r, beta = ||v0||_2, v0 /= beta
//   for j < budget: w = M^-1 (A v_j); modified Gram-Schmidt against v_0..v_j;
//                   h_{j+1,j} = ||w||_2; Givens rotations; stop on the estimate
//   d = sum_l y_l v_l
// with M^-1 = U^-1 L^-1 P in the working precision, factor entries promoted
// term by term (solve_mps_into, dense_lu.hpp:175-182 -- the K6 kernels).
//
// What fixes the bits:
//  * dot / nrm2 (krylov_ir.hpp:24-37) are one sequential accumulation, i
//    ascending, which the reference build compiles as a vectorised fold-left
//    reduction: rounded products added in order for the vector part of the
//    range (4 doubles / 8 floats per step, plus a half vector when that many
//    remain -- not for the binary64 nrm2), s = fma(a_i, b_i, s) for the scalar
//    tail (read off the object code of oracle/_ref; krylov_host.cpp
//    reduction_unfused states the rule, tests pin it). dot_seq_kernel runs
//    exactly that chain in one thread, the operands staged through shared
//    memory by the rest of the CTA, so it costs about one add latency per
//    element;
//  * matvec_into (matrix.hpp:127-140) is a column sweep y_i = fma(c_ij, x_j, y_i),
//    j ascending: one lane per row (the residual's order without the TwoSum);
//  * the vector updates are single rounded operations per element
//    (w -= h v as one FMA, v *= 1/beta as one product with the host's quotient);
//  * the Givens / back-substitution scalars stay on the host with the
//    reference build's fused / unfused choices spelled out (krylov_host.cpp);
//    sqrt and hypot are the host's.
// One host synchronisation per inner iteration (the reference's convergence
// test needs h_{.,j} anyway).
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "krylov_host.h"

namespace mpirg
{
namespace
{
__device__ __forceinline__ double kfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float kfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// out[slot] = sum_i a_i b_i, accumulated sequentially from 0 in T.
constexpr int DOT_TILE = 1024;  // 2 x 2 x 1024 x 8 B = 32 KB of static shared memory
__device__ __forceinline__ double kmuladd(double a, double b, double s)
{
  return __dadd_rn(s, __dmul_rn(a, b));
}
__device__ __forceinline__ float kmuladd(float a, float b, float s)
{
  return __fadd_rn(s, __fmul_rn(a, b));
}

// nv: the leading elements whose products are rounded before the addition.
template <typename T>
__global__ void __launch_bounds__(256) dot_seq_kernel(const T *__restrict__ a,
                                                      const T *__restrict__ b, int n, int nv,
                                                      T *__restrict__ out)
{
  __shared__ T sa[2][DOT_TILE], sb[2][DOT_TILE];
  const int t = threadIdx.x;
  const int nt = (n + DOT_TILE - 1) / DOT_TILE;
  auto load = [&](int tile, int buf) {
    const int base = tile * DOT_TILE;
    for (int i = t; i < DOT_TILE; i += 256)
    {
      const int g = base + i;
      sa[buf][i] = g < n ? a[g] : T(0);
      sb[buf][i] = g < n ? b[g] : T(0);
    }
  };
  load(0, 0);
  __syncthreads();
  T s = T(0);
  for (int tile = 0; tile < nt; ++tile)
  {
    const int buf = tile & 1;
    if (t == 0)
    {
      const int base = tile * DOT_TILE;
      const int cnt = min(DOT_TILE, n - base);
      if (base + DOT_TILE <= nv)
      {
#pragma unroll 16
        for (int i = 0; i < DOT_TILE; ++i)
          s = kmuladd(sa[buf][i], sb[buf][i], s);
      }
      else
        for (int i = 0; i < cnt; ++i)
          s = base + i < nv ? kmuladd(sa[buf][i], sb[buf][i], s)
                            : kfma(sa[buf][i], sb[buf][i], s);
    }
    else if (tile + 1 < nt)
      load(tile + 1, buf ^ 1);  // thread 0's share of the tile is covered below
    __syncthreads();
    if (tile + 1 < nt)
    {
      // the elements thread 0 would have loaded (i = 0, 256, ...)
      if (t == 1)
      {
        const int base = (tile + 1) * DOT_TILE;
        for (int i = 0; i < DOT_TILE; i += 256)
        {
          const int g = base + i;
          sa[buf ^ 1][i] = g < n ? a[g] : T(0);
          sb[buf ^ 1][i] = g < n ? b[g] : T(0);
        }
      }
      __syncthreads();
    }
  }
  if (t == 0)
    *out = s;
}

// w_l = fma(-h, v_l, w_l), h read from device memory
template <typename T>
__global__ void axpy_neg_kernel(T *__restrict__ w, const T *__restrict__ v,
                                const T *__restrict__ h, int n)
{
  const T hv = *h;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    w[i] = kfma(-hv, v[i], w[i]);
}

template <typename T>
__global__ void scale_kernel(T *__restrict__ w, T s, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    if constexpr (sizeof(T) == 8)
      w[i] = __dmul_rn(w[i], s);
    else
      w[i] = __fmul_rn(w[i], s);
  }
}

// d_i = sum_l fma(y_l, v_l[i], d_i), l ascending, from d = 0 (krylov_ir.hpp:162-168)
template <typename T>
__global__ void combine_kernel(T *__restrict__ d, const T *__restrict__ basis, int n, int k,
                               const T *__restrict__ y)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    T s = T(0);
    for (int l = 0; l < k; ++l)
      s = kfma(y[l], basis[(size_t)l * n + i], s);
    d[i] = s;
  }
}

// y = A x, column sweep in T (matrix.hpp:127-140): one lane per row.
template <typename T>
__global__ void __launch_bounds__(32) matvec_kernel(const T *__restrict__ a, int n,
                                                    const T *__restrict__ x, T *__restrict__ y)
{
  const int row = blockIdx.x * 32 + threadIdx.x;
  const bool valid = row < n;
  const int rr = valid ? row : 0;
  T s = T(0);
  int j = 0;
  for (; j + 16 <= n; j += 16)
  {
    T v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      v[q] = __ldcs(a + (size_t)(j + q) * n + rr);
#pragma unroll
    for (int q = 0; q < 16; ++q)
      s = kfma(v[q], __ldg(x + j + q), s);
  }
  for (; j < n; ++j)
    s = kfma(__ldcs(a + (size_t)j * n + rr), __ldg(x + j), s);
  if (valid)
    y[row] = s;
}

// w = TW(r) (krylov_ir.hpp:307-308)
template <typename TW, typename TR>
__global__ void demote_vec_kernel(const TR *__restrict__ r, TW *__restrict__ w, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    w[i] = demote<TW, TR>(r[i]);
}

// x_i += TR(w_i); ||w||_inf and ||x||_inf (krylov_ir.hpp:315-317)
template <typename TW, typename TR>
__global__ void ir_update_kernel(const TW *__restrict__ w, TR *__restrict__ x, int n,
                                 unsigned long long *dnorm_bits, unsigned long long *xnorm_bits)
{
  unsigned long long db = 0, xb = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    const TW wv = w[i];
    const TR xn = add(x[i], (TR)wv);
    x[i] = xn;
    const unsigned long long a = abs_bits((double)wv), b = abs_bits((double)xn);
    db = a > db ? a : db;
    xb = b > xb ? b : xb;
  }
  db = warp_max_u64(db);
  xb = warp_max_u64(xb);
  if ((threadIdx.x & 31) == 0)
  {
    atomicMax(dnorm_bits, db);
    atomicMax(xnorm_bits, xb);
  }
}

int grid_for(int n) { return std::max(1, std::min(148 * 4, (n + 255) / 256)); }

template <typename T>
void gmres_t(GmresCtx &c, void *w_inout, int *iters, bool *breakdown)
{
  const int n = c.n, bs = c.bs, ld = bs + 1;
  cudaStream_t s = c.s;
  T *w = static_cast<T *>(w_inout);
  T *basis = static_cast<T *>(c.basis);
  T *tmp = static_cast<T *>(c.tmp);
  T *dots = static_cast<T *>(c.dots);
  T *hd = static_cast<T *>(c.h_dots);
  std::vector<T> hess((size_t)ld * bs, T(0)), cs(bs, T(0)), sn(bs, T(0)), g(bs + 1, T(0)),
      y(bs, T(0));
  auto precond = [&](const T *src, T *dst) {
    TrsvArgs a{};
    a.ts = c.tw;
    a.tf = c.tf;
    a.tin = c.tw;
    a.lps = 0;
    a.ir = 0;
    a.n = n;
    a.lu = c.a_low;
    a.perm = c.perm;
    a.rin = src;
    a.y = c.y;
    a.out = dst;
    a.info = c.info;
    launch_trsv(a, *c.tws, s);
  };
  // half_step: the reference's nrm2 in binary64 has no half-vector epilogue
  auto dot = [&](const T *a, const T *b, int slot, bool half_step = true) {
    dot_seq_kernel<T><<<1, 256, 0, s>>>(a, b, n, reduction_unfused(n, (int)sizeof(T), half_step),
                                        dots + slot);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  };
  constexpr bool nrm_half = sizeof(T) == 4;
  // reads `count` scalars + the error record; false if a substitution went non-finite
  auto fetch = [&](int count) {
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(hd, dots, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(
        cudaMemcpyAsync(c.h_info, c.info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    return c.h_info->nonfinite == 0;
  };
  *iters = 0;
  *breakdown = false;
  c.nonfinite = false;
  T *v0 = basis;
  precond(w, v0);
  dot(v0, v0, 0, nrm_half);
  if (!fetch(1))
  {
    c.nonfinite = true;
    return;
  }
  const T beta = host_sqrt<T>(hd[0]);
  MPIRG_CUDA_CHECK(cudaMemsetAsync(w, 0, sizeof(T) * n, s));  // d = 0
  if (beta == T(0))
    return;
  scale_kernel<T><<<grid_for(n), 256, 0, s>>>(v0, host_recip<T>(beta), n);
  g[0] = beta;
  const double target = c.rtol * static_cast<double>(beta);
  int k = 0;
  bool brk = false;
  for (int j = 0; j < bs; ++j)
  {
    T *vj = basis + (size_t)j * n, *wj = basis + (size_t)(j + 1) * n;
    matvec_kernel<T><<<(n + 31) / 32, 32, 0, s>>>(static_cast<const T *>(c.a_high), n, vj, tmp);
    MPIRG_CUDA_CHECK(cudaGetLastError());
    precond(tmp, wj);
    for (int i = 0; i <= j; ++i)
    {
      dot(wj, basis + (size_t)i * n, i);
      axpy_neg_kernel<T><<<grid_for(n), 256, 0, s>>>(wj, basis + (size_t)i * n, dots + i, n);
    }
    dot(wj, wj, j + 1, nrm_half);
    if (!fetch(j + 2))
    {
      c.nonfinite = true;
      return;
    }
    T *col = hess.data() + (size_t)j * ld;
    for (int i = 0; i <= j; ++i)
      col[i] = hd[i];
    const T hj1 = host_sqrt<T>(hd[j + 1]);
    col[j + 1] = hj1;
    if (hj1 > T(0))
      scale_kernel<T><<<grid_for(n), 256, 0, s>>>(wj, host_recip<T>(hj1), n);
    const double res = gmres_rotate<T>(hess.data(), ld, cs.data(), sn.data(), g.data(), j);
    k = j + 1;
    if (res <= target)
      break;
    if (hj1 == T(0))
    {
      brk = true;
      break;
    }
  }
  brk = gmres_backsolve<T>(hess.data(), ld, g.data(), y.data(), k) || brk;
  MPIRG_CUDA_CHECK(cudaMemcpyAsync(dots, y.data(), sizeof(T) * k, cudaMemcpyHostToDevice, s));
  combine_kernel<T><<<grid_for(n), 256, 0, s>>>(w, basis, n, k, dots);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));  // y (host vector) is read by the copy above
  *iters = k;
  *breakdown = brk;
}
// out_i = fma(sc, b_i, a_i) (out may alias a): the reference build fuses every
// "x +- scalar * y" of the BiCGSTAB vector updates into one FMA.
template <typename T>
__global__ void vfma_kernel(T *__restrict__ out, const T *a, const T *__restrict__ b, T sc, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = kfma(sc, b[i], a[i]);
}
// p_i = fma(beta, fma(-omega, v_i, p_i), rr_i) (krylov_ir.hpp:248-249)
template <typename T>
__global__ void bicg_p_kernel(T *__restrict__ p, const T *__restrict__ rr, const T *__restrict__ v,
                              T beta, T omega, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = kfma(beta, kfma(-omega, v[i], p[i]), rr[i]);
}

// bicgstab_correction_into (krylov_ir.hpp:173-254) as the reference build runs
// it: left-preconditioned BiCGSTAB on M^-1 A d = M^-1 r from d = 0, at most
// `bs` iterations, rtol 0.1. The dot products follow the same fold-left rule as
// the GMRES ones (dot: half-vector epilogue; the a == b instances -- nrm2 and
// t.t -- as nrm2 does); every vector update is one FMA per element; the five
// scalars per iteration (alpha, omega, beta from two quotients and a product)
// are computed on the host in the working precision. Workspace: seven vectors
// at the start of c.basis. Four host synchronisations per iteration.
template <typename T>
void bicgstab_t(GmresCtx &c, void *w_inout, int *iters, bool *breakdown)
{
  const int n = c.n;
  cudaStream_t s = c.s;
  T *w = static_cast<T *>(w_inout);
  T *z = static_cast<T *>(c.basis);
  T *rr = z + (size_t)n, *rhat = z + 2 * (size_t)n, *p = z + 3 * (size_t)n, *v = z + 4 * (size_t)n,
    *sv = z + 5 * (size_t)n, *tv = z + 6 * (size_t)n;
  T *tmp = static_cast<T *>(c.tmp);
  T *dots = static_cast<T *>(c.dots);
  T *hd = static_cast<T *>(c.h_dots);
  auto precond = [&](const T *src, T *dst) {
    TrsvArgs a{};
    a.ts = c.tw;
    a.tf = c.tf;
    a.tin = c.tw;
    a.lps = 0;
    a.ir = 0;
    a.n = n;
    a.lu = c.a_low;
    a.perm = c.perm;
    a.rin = src;
    a.y = c.y;
    a.out = dst;
    a.info = c.info;
    launch_trsv(a, *c.tws, s);
  };
  auto dot = [&](const T *a, const T *b, int slot, bool half_step = true) {
    dot_seq_kernel<T><<<1, 256, 0, s>>>(a, b, n, reduction_unfused(n, (int)sizeof(T), half_step),
                                        dots + slot);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  };
  constexpr bool nrm_half = sizeof(T) == 4;
  auto fetch = [&](int count) {
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(hd, dots, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(
        cudaMemcpyAsync(c.h_info, c.info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
    MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
    return c.h_info->nonfinite == 0;
  };
  auto matvec = [&](const T *x, T *y) {
    matvec_kernel<T><<<(n + 31) / 32, 32, 0, s>>>(static_cast<const T *>(c.a_high), n, x, y);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  };
  const int g = grid_for(n);
  *iters = 0;
  *breakdown = false;
  c.nonfinite = false;
  precond(w, z);
  dot(z, z, 0, nrm_half);
  if (!fetch(1))
  {
    c.nonfinite = true;
    return;
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(w, 0, sizeof(T) * n, s));  // d = 0
  const double znorm = static_cast<double>(host_sqrt<T>(hd[0]));
  if (znorm == 0.0)
    return;
  const double target = c.rtol * znorm;
  for (T *dst : {rr, rhat, p})
    MPIRG_CUDA_CHECK(cudaMemcpyAsync(dst, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  dot(rhat, rr, 0);
  if (!fetch(1))
  {
    c.nonfinite = true;
    return;
  }
  T rho = hd[0];
  int it = 0;
  bool brk = false;
  while (it < c.bs)
  {
    matvec(p, tmp);
    precond(tmp, v);
    dot(rhat, v, 0);
    if (!fetch(1))
    {
      c.nonfinite = true;
      return;
    }
    const T denom = hd[0];
    if (denom == T(0))
    {
      brk = true;
      break;
    }
    const T alpha = rho / denom;
    vfma_kernel<T><<<g, 256, 0, s>>>(sv, rr, v, -alpha, n);
    vfma_kernel<T><<<g, 256, 0, s>>>(w, w, p, alpha, n);
    ++it;
    dot(sv, sv, 0, nrm_half);
    if (!fetch(1))
    {
      c.nonfinite = true;
      return;
    }
    if (static_cast<double>(host_sqrt<T>(hd[0])) <= target)
      break;
    matvec(sv, tmp);
    precond(tmp, tv);
    dot(tv, tv, 0, nrm_half);
    dot(tv, sv, 1);
    if (!fetch(2))
    {
      c.nonfinite = true;
      return;
    }
    const T tt = hd[0];
    if (tt == T(0))
    {
      brk = true;
      break;
    }
    const T omega = hd[1] / tt;
    vfma_kernel<T><<<g, 256, 0, s>>>(w, w, sv, omega, n);
    vfma_kernel<T><<<g, 256, 0, s>>>(rr, sv, tv, -omega, n);
    dot(rr, rr, 0, nrm_half);
    dot(rhat, rr, 1);
    if (!fetch(2))
    {
      c.nonfinite = true;
      return;
    }
    if (static_cast<double>(host_sqrt<T>(hd[0])) <= target)
      break;
    const T rho_new = hd[1];
    if (rho_new == T(0) || omega == T(0))
    {
      brk = true;
      break;
    }
    const T beta = (rho_new / rho) * (alpha / omega);
    bicg_p_kernel<T><<<g, 256, 0, s>>>(p, rr, v, beta, omega, n);
    rho = rho_new;
  }
  MPIRG_CUDA_CHECK(cudaGetLastError());
  MPIRG_CUDA_CHECK(cudaStreamSynchronize(s));
  *iters = it;
  *breakdown = brk;
}
}  // namespace

void gmres_correction(GmresCtx &c, void *w, int *iters, bool *breakdown)
{
  if (c.tw == B64)
    gmres_t<double>(c, w, iters, breakdown);
  else
    gmres_t<float>(c, w, iters, breakdown);
}

void bicgstab_correction(GmresCtx &c, void *w, int *iters, bool *breakdown)
{
  if (c.tw == B64)
    bicgstab_t<double>(c, w, iters, breakdown);
  else
    bicgstab_t<float>(c, w, iters, breakdown);
}

void launch_demote_vec(int tw, int tr, int n, const void *r, void *w, cudaStream_t s)
{
  ProfScope ps(KC_VEC, s);
  const int g = grid_for(n);
  if (tw == B64 && tr == B64)
    demote_vec_kernel<double, double><<<g, 256, 0, s>>>((const double *)r, (double *)w, n);
  else if (tw == B32 && tr == B64)
    demote_vec_kernel<float, double><<<g, 256, 0, s>>>((const double *)r, (float *)w, n);
  else
    demote_vec_kernel<float, float><<<g, 256, 0, s>>>((const float *)r, (float *)w, n);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

void launch_ir_update(int tw, int tr, int n, const void *w, void *x, unsigned long long *dnorm,
                      unsigned long long *xnorm, cudaStream_t s)
{
  ProfScope ps(KC_VEC, s);
  const int g = grid_for(n);
  if (tw == B64 && tr == B64)
    ir_update_kernel<double, double><<<g, 256, 0, s>>>((const double *)w, (double *)x, n, dnorm,
                                                      xnorm);
  else if (tw == B32 && tr == B64)
    ir_update_kernel<float, double><<<g, 256, 0, s>>>((const float *)w, (double *)x, n, dnorm,
                                                     xnorm);
  else
    ir_update_kernel<float, float><<<g, 256, 0, s>>>((const float *)w, (float *)x, n, dnorm,
                                                    xnorm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace mpirg
