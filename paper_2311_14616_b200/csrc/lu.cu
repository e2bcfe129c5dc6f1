// K2-K5 -- blocked right-looking LU with partial pivoting, bitwise equal to
// detail::lu_inplace (proj/include/mpir/dense_lu.hpp:50-109).
//
// Why blocking keeps the reference's bits: lu_inplace updates every element
// a_ij once per elimination step k, in ascending k, with one rounding per
// update (an FMA for fp32/fp64 under the reference build; r16(c - r16(l*u))
// for binary16). A right-looking blocked LU performs exactly the same
// per-element sequence as long as (1) the panel applies its rank-1 updates in
// k order, (2) U12 = L11^{-1} A12 is a forward substitution in k order, and
// (3) the trailing GEMM initialises its accumulator from A22 and walks k in
// order with one FMA per term. Row swaps only move data, so deferring them to
// a gather per panel changes nothing. Pivot choice is the reference's: the
// first row (lowest index) maximising |a_ik| as a double, NaN never chosen,
// and a NaN on the diagonal keeps p = k (dense_lu.hpp:65-78).
//
// Kernels per panel step p (panel width nb, k0 = p*nb, c0 = k0 + nb):
//   lu_panel2_kernel     (lu_panel.cuh) one thread-block cluster factors the
//                        (n-k0) x nb panel in registers; st.async/mbarrier
//                        candidate exchange; emits ipiv + the row-move list.
//   lu_mt_kernel         applies the panel's row moves (a permutation of
//                        <= 2nb rows, as a gather) to trailing columns and
//                        solves U12 = L11^{-1} A12 for them (k order).
//   lu_gemm_kernel       A22 -= L21 U12, SIMT register-tiled FMA with the
//                        accumulator initialised from A22, k ascending (no
//                        TF32: that would change the factor precision).
//   lu_apply_moves_kernel  the same row moves for the columns left of the
//                        panel and for the accumulated permutation.
// Schedule (look-ahead): the main stream runs the critical chain
//   panel(p) -> mt(next nb columns) -> gemm(next nb columns) -> panel(p+1)
// while a side stream applies mt + gemm to the remaining columns and the
// left-column moves, overlapping the sequential panel chain.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <cstdlib>
#include <string>
#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "../../include/mpir_gpu.h"
#include "lu_f32.cuh"
#include "lu_panel.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace mpirg
{

namespace
{

// Column ownership of a rank under the 1-D block-cyclic distribution of
// BASELINE config 5a: global column blocks of 2^sh columns,
// block b on rank b mod G. Kernels walk the rank's columns by LOCAL index L
// (owned columns in ascending global order) and map L to the global column.
// G == 1 is the identity (single-GPU LU).
struct ColMap
{
  int G = 1, r = 0, sh = 30;
  __host__ __device__ __forceinline__ int g(int L) const
  {
    if (G == 1)
      return L;
    const int m = (1 << sh) - 1;
    return ((((L >> sh) * G) + r) << sh) | (L & m);
  }
  // number of owned columns with global index < c
  __host__ __device__ int lcount(int c) const
  {
    if (G == 1)
      return c;
    const int full = c >> sh;
    const int owned = full > r ? (full - 1 - r) / G + 1 : 0;
    return (owned << sh) + ((full % G) == r ? (c & ((1 << sh) - 1)) : 0);
  }
};

// Gather-apply the panel's row moves (new[dst] = old[src]) to the columns
// [cb, ce) -- one warp per column -- and to perm (block 0, warp 0).
template <typename T, int NB>
__global__ void __launch_bounds__(256) lu_apply_moves_kernel(T *__restrict__ A, int n, int cb,
                                                             int ce, ColMap map,
                                                             const int2 *__restrict__ moves,
                                                             const int *__restrict__ nmoves,
                                                             int *__restrict__ perm,
                                                             BatchStride bs = BatchStride{})
{
  constexpr int PER = (2 * NB + 31) / 32;
  A += (size_t)blockIdx.z * bs.a;
  moves += (size_t)blockIdx.z * bs.moves;
  nmoves += (size_t)blockIdx.z * bs.nm;
  if (perm)
    perm += (size_t)blockIdx.z * bs.vec;
  const int nm = *nmoves;
  if (nm == 0)
    return;
  const int lane = threadIdx.x & 31;
  int2 mv[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q)
  {
    const int e = lane + 32 * q;
    mv[q] = e < nm ? moves[e] : make_int2(-1, -1);
  }
  const int ncols = ce - cb;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x < 32 && perm)
  {
    int v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (mv[q].x >= 0)
        v[q] = perm[mv[q].y];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (mv[q].x >= 0)
        perm[mv[q].x] = v[q];
  }
  constexpr int UNR = 4;
  for (int c0 = gw * UNR; c0 < ncols; c0 += nw * UNR)
  {
    T v[UNR][PER];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (c0 + u < ncols)
      {
        const T *cp = A + (size_t)map.g(cb + c0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            v[u][q] = cp[mv[q].y];
      }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (c0 + u < ncols)
      {
        T *cp = A + (size_t)map.g(cb + c0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            cp[mv[q].x] = v[u][q];
      }
  }
}

// The row moves of several consecutive panels [pa, pb), applied in panel
// order to the columns [cb, ce) -- one warp per column, so a column's moves
// stay ordered without any grid-wide synchronisation (lu_run_tc applies a
// whole sub-tree's moves to the other half of its block in one launch).
template <typename T, int NB>
__global__ void __launch_bounds__(256) lu_apply_moves_multi_kernel(
    T *__restrict__ A, int n, int cb, int ce, const int2 *__restrict__ moves,
    const int *__restrict__ nmoves, int pa, int pb)
{
  constexpr int PER = (2 * NB + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = pa; p < pb; ++p)
  {
    const int nm = nmoves[p];
    if (nm == 0)
      continue;  // warp-uniform
    int2 mv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
    {
      const int e = lane + 32 * q;
      mv[q] = e < nm ? moves[(size_t)p * 2 * NB + e] : make_int2(-1, -1);
    }
    for (int c = cb + gw; c < ce; c += nw)
    {
      T *cp = A + (size_t)c * n;
      T v[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (mv[q].x >= 0)
          v[q] = cp[mv[q].y];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (mv[q].x >= 0)
          cp[mv[q].x] = v[q];
      __syncwarp();
    }
  }
}

// Row moves + U12 = L11^{-1} A12 for the trailing columns [cb, ce).
// CTA = 4 warps, 32 columns (8 per warp). Phase 1: each warp gathers the
// moves of its 8 columns (lanes over move entries). Phase 2: each warp solves
// its 8 columns at once -- lane owns panel rows (lane, lane+32), x_k is
// broadcast by shuffle, k ascending, one update per element per step, so the
// per-element chain is the reference's (dense_lu.hpp:91-107 restricted to
// the panel rows).
constexpr int MT_COLS = 32;
template <typename T, int NB>
__global__ void __launch_bounds__(128) lu_mt_kernel(T *__restrict__ A, int n, int k0, int jb,
                                                    int cb, int ce, ColMap map,
                                                    const int2 *__restrict__ moves,
                                                    const int *__restrict__ nmoves,
                                                    BatchStride bs = BatchStride{})
{
  constexpr int PER = (2 * NB + 31) / 32;
  constexpr int RL = (NB + 31) / 32;  // panel rows per lane
  __shared__ T L[NB][NB + 1];
  A += (size_t)blockIdx.z * bs.a;
  moves += (size_t)blockIdx.z * bs.moves;
  nmoves += (size_t)blockIdx.z * bs.nm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    // stage L11 with all loads in flight before the stores
    constexpr int PT = (NB * NB + 127) / 128;
    T tmp[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = threadIdx.x + u * 128;
      const int kk = idx / NB, i = idx % NB;
      tmp[u] = (kk < jb && i < jb) ? A[(size_t)(k0 + kk) * n + k0 + i] : T{};
    }
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = threadIdx.x + u * 128;
      const int kk = idx / NB, i = idx % NB;
      if (kk < NB)
        L[i][kk] = tmp[u];
    }
  }
  const int nm = *nmoves;
  const int col0 = cb + blockIdx.x * MT_COLS + warp * 8;
  // phase 1: gather the row moves for this warp's 8 columns
  if (nm > 0)
  {
    int2 mv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
    {
      const int e = lane + 32 * q;
      mv[q] = e < nm ? moves[e] : make_int2(-1, -1);
    }
    T v[8][PER];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (col0 + u < ce)
      {
        const T *cp = A + (size_t)map.g(col0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            v[u][q] = cp[mv[q].y];
      }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (col0 + u < ce)
      {
        T *cp = A + (size_t)map.g(col0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            cp[mv[q].x] = v[u][q];
      }
    __syncwarp();
  }
  __syncthreads();  // L staged; this warp's gathered values visible to itself
  // phase 2: forward substitution on the panel rows of 8 columns
  T x[8][RL];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      x[u][h] = (col0 + u < ce && i < jb) ? A[(size_t)map.g(col0 + u) * n + k0 + i] : T{};
    }
#pragma unroll 1
  for (int kk = 0; kk < jb; ++kk)
  {
    const int hk = kk >> 5, lk = kk & 31;
    T lv[RL];
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      lv[h] = (i > kk && i < jb) ? L[i][kk] : T{};
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
    {
      T src = x[u][0];
#pragma unroll
      for (int h = 1; h < RL; ++h)
        if (hk == h)
          src = x[u][h];
      const T xk = shfl_t(src, lk);
#pragma unroll
      for (int h = 0; h < RL; ++h)
      {
        const int i = lane + 32 * h;
        if (i > kk && i < jb)
          x[u][h] = upd(x[u][h], lv[h], xk);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      if (col0 + u < ce && i < jb)
        A[(size_t)map.g(col0 + u) * n + k0 + i] = x[u][h];
    }
}

// ---- trailing update A22 -= L21 * U12 ------------------------------------
// Compute type: binary16 values are held exactly in fp32 registers.
template <typename T> struct CType { using type = T; };
template <> struct CType<h16> { using type = float; };

__device__ __forceinline__ float to_c(h16 v) { return h2f(v); }
__device__ __forceinline__ float to_c(float v) { return v; }
__device__ __forceinline__ double to_c(double v) { return v; }
__device__ __forceinline__ void from_c(h16 &dst, float v) { dst = f2h(v); }
__device__ __forceinline__ void from_c(float &dst, float v) { dst = v; }
__device__ __forceinline__ void from_c(double &dst, double v) { dst = v; }

template <typename T>
__device__ __forceinline__ typename CType<T>::type gemm_upd(typename CType<T>::type c,
                                                            typename CType<T>::type l,
                                                            typename CType<T>::type u)
{
  if constexpr (std::is_same<T, h16>::value)
  {
    const float p = __half2float(__float2half_rn(__fmul_rn(l, u)));
    return __half2float(__float2half_rn(__fsub_rn(c, p)));
  }
  else
    return upd(c, l, u);
}

constexpr int GB = 128;       // C tile edge
constexpr int GPAD = 4;       // Bs row padding
template <typename T, int NB>
constexpr size_t gemm_smem_bytes()
{
  using C = typename CType<T>::type;
  return sizeof(C) * (size_t)NB * GB + sizeof(C) * (size_t)NB * (GB + GPAD);
}

// C = A[r0.., cb..ce) for rows >= c0; L21 = A[rows, k0..k0+jb); U12 = A[k0.., cols].
template <typename T, int NB>
__global__ void __launch_bounds__(256) lu_gemm_kernel(T *__restrict__ A, int n, int k0, int jb,
                                                      int cb, int ce, ColMap map)
{
  using C = typename CType<T>::type;
  extern __shared__ __align__(16) unsigned char gsm[];
  C *As = reinterpret_cast<C *>(gsm);                  // [NB][GB]
  C *Bs = As + (size_t)NB * GB;                        // [NB][GB+GPAD]
  const int c0 = k0 + jb;
  const int r0 = c0 + blockIdx.x * GB;
  const int cc0 = cb + blockIdx.y * GB;
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;

  {
    constexpr int PT = NB * GB / 256;  // elements per thread per operand
    C ta[PT], tb[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = t + u * 256;
      const int kk = idx / GB, m = idx % GB;
      const int row = r0 + m;
      ta[u] = (kk < jb && row < n) ? to_c(A[(size_t)(k0 + kk) * n + row]) : C(0);
      const int nn = idx / NB, kb = idx % NB;
      const int col = cc0 + nn;
      tb[u] = (kb < jb && col < ce) ? to_c(A[(size_t)map.g(col) * n + k0 + kb]) : C(0);
    }
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = t + u * 256;
      As[(idx / GB) * GB + idx % GB] = ta[u];
      Bs[(idx % NB) * (GB + GPAD) + idx / NB] = tb[u];
    }
  }

  C acc[8][8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
  {
    const int col = cc0 + (j < 4 ? ty * 4 + j : 64 + ty * 4 + (j - 4));
#pragma unroll
    for (int i = 0; i < 8; ++i)
    {
      const int row = r0 + (i < 4 ? tx * 4 + i : 64 + tx * 4 + (i - 4));
      acc[i][j] = (row < n && col < ce) ? to_c(A[(size_t)map.g(col) * n + row]) : C(0);
    }
  }
  __syncthreads();

  for (int kk = 0; kk < jb; ++kk)
  {
    C a[8], b[8];
    const C *ar = As + kk * GB;
    const C *br = Bs + kk * (GB + GPAD);
#pragma unroll
    for (int i = 0; i < 4; ++i)
    {
      a[i] = ar[tx * 4 + i];
      a[4 + i] = ar[64 + tx * 4 + i];
      b[i] = br[ty * 4 + i];
      b[4 + i] = br[64 + ty * 4 + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        acc[i][j] = gemm_upd<T>(acc[i][j], a[i], b[j]);
  }

#pragma unroll
  for (int j = 0; j < 8; ++j)
  {
    const int col = cc0 + (j < 4 ? ty * 4 + j : 64 + ty * 4 + (j - 4));
#pragma unroll
    for (int i = 0; i < 8; ++i)
    {
      const int row = r0 + (i < 4 ? tx * 4 + i : 64 + tx * 4 + (i - 4));
      if (row < n && col < ce)
        from_c(A[(size_t)map.g(col) * n + row], acc[i][j]);
    }
  }
}

// binary32 trailing update, vectorised (n % 4 == 0, 16-byte aligned A):
// BM x BN tile of C per CTA of 256 threads (16 x 16), each thread a
// (BM/16) x (BN/16) micro-tile made of 4-row x 4-column groups 64 apart, so
// every C access is a float4 along a column (coalesced 256 B per 16 lanes)
// and every operand read from shared memory is an LDS.128. Same arithmetic
// and per-element order as lu_gemm_kernel: the accumulator starts from A22
// and takes one FMA per k, k ascending.
template <int NB, int BM, int BN>
__global__ void __launch_bounds__(256, 2) lu_gemm_v4_kernel(float *__restrict__ A, int n, int k0,
                                                         int jb, int cb, int ce, ColMap map,
                                                         size_t batch_stride = 0)
{
  constexpr int TM = BM / 16, TN = BN / 16;
  A += (size_t)blockIdx.z * batch_stride;
  constexpr int BPAD = 4;
  extern __shared__ __align__(16) unsigned char gsm[];
  float *As = reinterpret_cast<float *>(gsm);  // [NB][BM]
  float *Bs = As + (size_t)NB * BM;            // [NB][BN + BPAD]
  const int c0 = k0 + jb;
  const int r0 = c0 + blockIdx.x * BM;
  const int cc0 = cb + blockIdx.y * BN;
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  {
    // A block: As[kk][m] = A[(k0+kk)*n + r0 + m], float4 along m
    constexpr int AV = NB * BM / 4 / 256;
    float4 ta[AV];
#pragma unroll
    for (int u = 0; u < AV; ++u)
    {
      const int idx = t + u * 256;
      const int kk = idx / (BM / 4), m4 = idx % (BM / 4);
      const int row = r0 + 4 * m4;
      ta[u] = (kk < jb && row < n)
                  ? __ldg(reinterpret_cast<const float4 *>(A + (size_t)(k0 + kk) * n + row))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // B block: Bs[kb][nn] = A[col(nn)*n + k0 + kb], float4 along kb
    constexpr int BV = NB * BN / 4 / 256;
    float4 tb[BV];
#pragma unroll
    for (int u = 0; u < BV; ++u)
    {
      const int idx = t + u * 256;
      const int nn = idx % BN, kq = idx / BN;
      const int col = cc0 + nn;
      tb[u] = (col < ce && 4 * kq < jb)
                  ? __ldg(reinterpret_cast<const float4 *>(A + (size_t)map.g(col) * n + k0 + 4 * kq))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < AV; ++u)
    {
      const int idx = t + u * 256;
      const int kk = idx / (BM / 4), m4 = idx % (BM / 4);
      reinterpret_cast<float4 *>(As + kk * BM)[m4] = ta[u];
    }
#pragma unroll
    for (int u = 0; u < BV; ++u)
    {
      const int idx = t + u * 256;
      const int nn = idx % BN, kq = idx / BN;
      // k beyond jb must not contribute: zero the lanes past jb
      const float v[4] = {tb[u].x, tb[u].y, tb[u].z, tb[u].w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        Bs[(4 * kq + e) * (BN + BPAD) + nn] = (4 * kq + e < jb) ? v[e] : 0.f;
    }
  }

  float acc[TM][TN];
#pragma unroll
  for (int gj = 0; gj < TN / 4; ++gj)
#pragma unroll
    for (int j = 0; j < 4; ++j)
    {
      const int col = cc0 + gj * 64 + ty * 4 + j;
#pragma unroll
      for (int gi = 0; gi < TM / 4; ++gi)
      {
        const int row = r0 + gi * 64 + tx * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < n && col < ce)
          v = *reinterpret_cast<const float4 *>(A + (size_t)map.g(col) * n + row);
        acc[gi * 4 + 0][gj * 4 + j] = v.x;
        acc[gi * 4 + 1][gj * 4 + j] = v.y;
        acc[gi * 4 + 2][gj * 4 + j] = v.z;
        acc[gi * 4 + 3][gj * 4 + j] = v.w;
      }
    }
  __syncthreads();

#pragma unroll 4
  for (int kk = 0; kk < jb; ++kk)
  {
    float a[TM], b[TN];
    const float *ar = As + kk * BM;
    const float *br = Bs + kk * (BN + BPAD);
#pragma unroll
    for (int gi = 0; gi < TM / 4; ++gi)
    {
      const float4 v = reinterpret_cast<const float4 *>(ar + gi * 64)[tx];
      a[gi * 4 + 0] = v.x;
      a[gi * 4 + 1] = v.y;
      a[gi * 4 + 2] = v.z;
      a[gi * 4 + 3] = v.w;
    }
#pragma unroll
    for (int gj = 0; gj < TN / 4; ++gj)
    {
      const float4 v = reinterpret_cast<const float4 *>(br + gj * 64)[ty];
      b[gj * 4 + 0] = v.x;
      b[gj * 4 + 1] = v.y;
      b[gj * 4 + 2] = v.z;
      b[gj * 4 + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        acc[i][j] = __fmaf_rn(-a[i], b[j], acc[i][j]);
  }

#pragma unroll
  for (int gj = 0; gj < TN / 4; ++gj)
#pragma unroll
    for (int j = 0; j < 4; ++j)
    {
      const int col = cc0 + gj * 64 + ty * 4 + j;
#pragma unroll
      for (int gi = 0; gi < TM / 4; ++gi)
      {
        const int row = r0 + gi * 64 + tx * 4;
        if (row < n && col < ce)
          *reinterpret_cast<float4 *>(A + (size_t)map.g(col) * n + row) =
              make_float4(acc[gi * 4 + 0][gj * 4 + j], acc[gi * 4 + 1][gj * 4 + j],
                          acc[gi * 4 + 2][gj * 4 + j], acc[gi * 4 + 3][gj * 4 + j]);
      }
    }
}

template <int NB, int BM, int BN>
constexpr size_t gemm_v4_smem()
{
  return sizeof(float) * ((size_t)NB * BM + (size_t)NB * (BN + 4));
}

__global__ void iota_kernel(int *p, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = i;
}

__global__ void perm_from_ipiv_kernel(const int *__restrict__ ipiv, int n, int *__restrict__ perm)
{
  // Sequential by construction (apply_pivots order); used only off the hot path.
  if (threadIdx.x != 0)
    return;
  for (int i = 0; i < n; ++i)
    perm[i] = i;
  for (int k = 0; k < n; ++k)
  {
    const int p = ipiv[k];
    if (p != k)
    {
      const int tmp = perm[k];
      perm[k] = perm[p];
      perm[p] = tmp;
    }
  }
}

// ---- host orchestration --------------------------------------------------
__global__ void iota_range_kernel(int *p, int lo, int hi)
{
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
    p[i] = i;
}

// Row-move list of a tall panel from its composed position map pp (rows of
// [lo, hi) whose content came from another row): new[i] = old[pp[i]].
__global__ void compact_moves_kernel(const int *__restrict__ pp, int lo, int hi,
                                     int2 *__restrict__ moves, int *__restrict__ nmoves)
{
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
  {
    const int src = pp[i];
    if (src != i)
      moves[atomicAdd(nmoves, 1)] = make_int2(i, src);
  }
}

__global__ void min_into_kernel(int *dst, const int *src) { *dst = min(*dst, *src); }

template <typename T, int NB, int RPT, int NTX, typename TG = T>
void configure_panel()
{
  static DeviceOnce done;
  if (!done.needed())
    return;
  auto k = panel2::lu_panel2_kernel<T, NB, RPT, NTX, TG>;
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)panel2::panel_dyn_smem<T, NB, RPT, NTX>()));
  done.done();
}

template <typename T, int NB>
void configure_gemm()
{
  static DeviceOnce done;
  if (!done.needed())
    return;
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_kernel<T, NB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)gemm_smem_bytes<T, NB>()));
  done.done();
}

// Speculative pivoting in the panel (lu_panel.cuh), a bit mask: 1 = per
// eight-column block, 2 = whole panel first. MPIRG_PANEL_SPEC=0 turns both off
// (every step then takes the cluster-wide exchange), MPIRG_PANEL_WHOLE=0 only
// the whole-panel pass, MPIRG_PANEL_WHOLE_BATCH=0 only for batched launches
// (measured on cfg 5b: 0.213 s with it, 0.227 s without -- the pass's shared
// memory already limits the kernel to one CTA per SM either way).
// Programmatic dependent launch along the binary32 LU's chain: level 1 (default)
// U12 solve -> update -> next panel, level 2 also panel -> U12 solve (no gain
// measured), MPIRG_LU_PDL=0 plain launches; same kernels, same results.
static int lu_pdl()
{
  static const int v = [] {
    const char *e = std::getenv("MPIRG_LU_PDL");
    return tool_attached() ? 0 : (e ? std::atoi(e) : 1);
  }();
  return v;
}

static int panel_spec(int ns)
{
  static const int base = [] {
    const char *e = std::getenv("MPIRG_PANEL_SPEC");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : 1;
  }();
  static const int whole = [] {
    const char *e = std::getenv("MPIRG_PANEL_WHOLE");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : 1;
  }();
  static const int whole_batch = [] {
    const char *e = std::getenv("MPIRG_PANEL_WHOLE_BATCH");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : 1;
  }();
  if (!base)
    return 0;
  return 1 | ((ns > 1 ? whole_batch : whole) ? 2 : 0);
}

template <typename T, int NB, int RPT, int NTX = panel2::NT, typename TG = T>
void launch_panel_rpt(int cs, TG *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm,
                      DevInfo *info, cudaStream_t s, int ns = 1, BatchStride bs = BatchStride{})
{
  configure_panel<T, NB, RPT, NTX, TG>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, ns);
  cfg.blockDim = dim3(NTX);
  const int spec = panel_spec(ns);
  // (the whole-panel pass needs more shared memory than the exchange algorithm)
  cfg.dynamicSmemBytes = (spec & 2) ? panel2::panel_dyn_smem<T, NB, RPT, NTX>()
                                    : panel2::panel_exact_smem<T, NB, RPT, NTX>();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (lu_pdl() && ns == 1)
  {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel2::lu_panel2_kernel<T, NB, RPT, NTX, TG>, a, n,
                                      k0, jb, ipiv, mv, nm, info, spec, bs));
}

// Largest rows-per-thread the shared memory allows for (T, NB) at 256 threads.
template <typename T, int NB>
constexpr int max_rpt()
{
  return panel2::panel_dyn_smem<T, NB, 4>() <= 180 * 1024
             ? 4
             : (panel2::panel_dyn_smem<T, NB, 2>() <= 180 * 1024 ? 2 : 1);
}

static int panel_max_cs()
{
  static const int v = [] {
    const char *e = std::getenv("MPIRG_PANEL_MAXCS");
    const int x = e ? std::atoi(e) : panel2::MAXCS;
    return std::max(1, std::min(panel2::MAXCS, x));
  }();
  return v;
}

// Rows-per-thread for an m-row panel on one cluster at NB (0 = does not fit).
template <typename T, int NB>
int panel_rpt(int m)
{
  int rpt = 1;
  while (rpt * panel2::NT * panel_max_cs() < m)
    rpt *= 2;
  return rpt <= max_rpt<T, NB>() ? rpt : 0;
}

template <typename T, int NB, typename TG = T>
void launch_panel(TG *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, DevInfo *info,
                  cudaStream_t s, int ns = 1, BatchStride bs = BatchStride{})
{
  const int m = n - k0;
  const int per_cta = panel2::NT;
  const int rpt = panel_rpt<T, NB>(m);
  if (rpt == 0)
    throw std::runtime_error("LU panel: n too large for a single-cluster panel at this nb");
  const int cs = std::max(1, (m + rpt * per_cta - 1) / (rpt * per_cta));
  prof_begin(KC_PANEL, s);
  if (rpt == 1)
    launch_panel_rpt<T, NB, 1, panel2::NT, TG>(cs, a, n, k0, jb, ipiv, mv, nm, info, s, ns, bs);
  else if (rpt == 2)
  {
    if constexpr (max_rpt<T, NB>() >= 2)
      launch_panel_rpt<T, NB, 2, panel2::NT, TG>(cs, a, n, k0, jb, ipiv, mv, nm, info, s, ns,
                                                 bs);
  }
  else
  {
    if constexpr (max_rpt<T, NB>() >= 4)
      launch_panel_rpt<T, NB, 4, panel2::NT, TG>(cs, a, n, k0, jb, ipiv, mv, nm, info, s, ns,
                                                 bs);
  }
  prof_end(KC_PANEL, s);
}

// Leaf of a tall panel: LEAF columns, 512 threads per CTA, up to 16 CTAs. The
// widest leaf whose rows fit the cluster's shared memory is used: 32 columns up
// to 16384 rows (binary32), 16 up to 32768, 8 beyond -- a 64-column panel of
// config 4 (n = 16384) is 2 leaves instead of 8.
constexpr int LEAF_NT = 512;
template <typename T, int LEAF>
constexpr int leaf_max_rpt()
{
  int r = 8;
  while (r > 1 && (sizeof(T) * (size_t)LEAF * r * LEAF_NT + 4096) > 180 * 1024)
    r /= 2;
  return r;
}

template <typename T, int LEAF>
int leaf_capacity()
{
  return leaf_max_rpt<T, LEAF>() * LEAF_NT * panel_max_cs();
}

template <typename T, int LEAF>
void launch_leaf(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, DevInfo *info,
                 cudaStream_t s)
{
  const int m = n - k0;
  prof_begin(KC_PANEL, s);
  if constexpr (LEAF == 8)
  {
    int rpt = 1;
    while (rpt * LEAF_NT * panel_max_cs() < m)
      rpt *= 2;
    if (rpt > leaf_max_rpt<T, LEAF>())
      throw std::runtime_error("LU panel: n too large for a single-cluster tall panel");
    const int cs = std::max(1, (m + rpt * LEAF_NT - 1) / (rpt * LEAF_NT));
    if (rpt == 1)
      launch_panel_rpt<T, LEAF, 1, LEAF_NT>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
    else if (rpt == 2)
      launch_panel_rpt<T, LEAF, 2, LEAF_NT>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
    else if (rpt == 4)
      launch_panel_rpt<T, LEAF, 4, LEAF_NT>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
    else
    {
      if constexpr (leaf_max_rpt<T, LEAF>() >= 8)
        launch_panel_rpt<T, LEAF, 8, LEAF_NT>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
    }
  }
  else
  {
    // wider leaves only exist at their largest rows-per-thread (they are
    // chosen when the panel is too tall for anything wider)
    constexpr int rpt = leaf_max_rpt<T, LEAF>();
    const int cs = std::max(1, (m + rpt * LEAF_NT - 1) / (rpt * LEAF_NT));
    launch_panel_rpt<T, LEAF, rpt, LEAF_NT>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
  }
  prof_end(KC_PANEL, s);
}

// Local column range [cb, ce) of a rank (global ranges when map is the identity).
template <typename T, int NB>
void launch_mt(T *a, int n, int k0, int jb, int cb, int ce, ColMap map, const int2 *mv,
               const int *nm, cudaStream_t s)
{
  if (ce <= cb)
    return;
  prof_begin(KC_TRSM, s);
  lu_mt_kernel<T, NB><<<(ce - cb + MT_COLS - 1) / MT_COLS, 128, 0, s>>>(a, n, k0, jb, cb, ce,
                                                                      map, mv, nm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_TRSM, s);
}

template <int NB, int BM, int BN>
void launch_gemm_v4_t(float *a, int n, int k0, int jb, int cb, int ce, ColMap map, cudaStream_t s)
{
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_v4_kernel<NB, BM, BN>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)gemm_v4_smem<NB, BM, BN>()));
    configured.done();
  }
  const int c0 = k0 + jb;
  const dim3 grid((n - c0 + BM - 1) / BM, (ce - cb + BN - 1) / BN);
  lu_gemm_v4_kernel<NB, BM, BN><<<grid, 256, gemm_v4_smem<NB, BM, BN>(), s>>>(a, n, k0, jb, cb,
                                                                              ce, map);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// MPIRG_GEMM=scalar forces the generic kernel (A/B measurements).
static bool gemm_v4_allowed()
{
  static const bool v = [] {
    const char *e = std::getenv("MPIRG_GEMM");
    return !(e && std::string(e) == "scalar");
  }();
  return v;
}

template <typename T, int NB>
void launch_gemm(T *a, int n, int k0, int jb, int cb, int ce, ColMap map, cudaStream_t s)
{
  const int c0 = k0 + jb;
  if (ce <= cb || c0 >= n)
    return;
  prof_begin(KC_GEMM, s);
  if constexpr (std::is_same<T, float>::value && NB >= 16)
  {
    if (n % 4 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0 && gemm_v4_allowed())
    {
      // 128 x 128 tiles while they fill the GPU twice over, else 64 x 64
      const long tiles128 = (long)((n - c0 + 127) / 128) * ((ce - cb + 127) / 128);
      if (tiles128 >= 2 * 148)
        launch_gemm_v4_t<NB, 128, 128>(a, n, k0, jb, cb, ce, map, s);
      else
        launch_gemm_v4_t<NB, 64, 64>(a, n, k0, jb, cb, ce, map, s);
      prof_end(KC_GEMM, s);
      return;
    }
  }
  configure_gemm<T, NB>();
  const dim3 grid((n - c0 + GB - 1) / GB, (ce - cb + GB - 1) / GB);
  lu_gemm_kernel<T, NB><<<grid, 256, gemm_smem_bytes<T, NB>(), s>>>(a, n, k0, jb, cb, ce, map);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_GEMM, s);
}

template <typename T, int NB>
void launch_moves(T *a, int n, int cb, int ce, ColMap map, const int2 *mv, const int *nm,
                  int *perm, cudaStream_t s)
{
  const int ncols = ce - cb;
  if (ncols <= 0 && !perm)
    return;
  prof_begin(KC_MOVES, s);
  const int warps_needed = std::max(1, (ncols + 3) / 4);
  const int grid = std::max(1, std::min((warps_needed + 7) / 8, 148 * 8));
  lu_apply_moves_kernel<T, NB><<<grid, 256, 0, s>>>(a, n, cb, std::max(cb, ce), map, mv, nm,
                                                    perm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_MOVES, s);
}

// A panel taller than one cluster holds at width NB: factor it as NB/8
// leaves of 8 columns (the same blocked right-looking order inside the
// panel: leaf, its moves on the panel's left columns, mt + gemm on the
// panel's right columns), composing the leaves' row moves in pp.
template <typename T, int NB, int LEAF>
void panel_tall_t(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, LuWorkspace &ws,
                  DevInfo *info, cudaStream_t s)
{
  const ColMap id{};
  const int m = n - k0;
  const int g = std::min(148 * 4, (m + 255) / 256);
  iota_range_kernel<<<g, 256, 0, s>>>(ws.pp, k0, n);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  const int nleaf = (jb + LEAF - 1) / LEAF;
  MPIRG_CUDA_CHECK(cudaMemsetAsync(ws.snm, 0, sizeof(int) * nleaf, s));
  for (int l = 0; l < nleaf; ++l)
  {
    const int ks = k0 + l * LEAF, w = std::min(LEAF, jb - l * LEAF);
    int2 *smv = ws.smv + (size_t)l * 2 * LEAF;
    int *snm = ws.snm + l;
    launch_leaf<T, LEAF>(a, n, ks, w, ipiv, smv, snm, info, s);
    launch_moves<T, LEAF>(a, n, k0, ks, id, smv, snm, ws.pp, s);
    launch_mt<T, LEAF>(a, n, ks, w, ks + w, k0 + jb, id, smv, snm, s);
    launch_gemm<T, LEAF>(a, n, ks, w, ks + w, k0 + jb, id, s);
  }
  compact_moves_kernel<<<g, 256, 0, s>>>(ws.pp, k0, n, mv, nm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// MPIRG_TALL_LEAF=8 keeps the 8-column leaves at every height (A/B runs).
static int tall_leaf_max()
{
  static const int v = [] {
    const char *e = std::getenv("MPIRG_TALL_LEAF");
    return e ? std::atoi(e) : 32;
  }();
  return v;
}

template <typename T, int NB>
void panel_tall(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, LuWorkspace &ws,
                DevInfo *info, cudaStream_t s)
{
  const int m = n - k0;
  if constexpr (NB >= 32)
    if (tall_leaf_max() >= 32 && m <= leaf_capacity<T, 32>())
    {
      panel_tall_t<T, NB, 32>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
      return;
    }
  if constexpr (NB >= 16)
    if (tall_leaf_max() >= 16 && m <= leaf_capacity<T, 16>())
    {
      panel_tall_t<T, NB, 16>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
      return;
    }
  panel_tall_t<T, NB, 8>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
}

template <typename T, int NB>
void panel_any(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, LuWorkspace &ws,
               DevInfo *info, cudaStream_t s)
{
  if (panel_rpt<T, NB>(n - k0) > 0)
    launch_panel<T, NB>(a, n, k0, jb, ipiv, mv, nm, info, s);
  else
    panel_tall<T, NB>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
}

// Trailing update of step k0 on columns [cb, ce): the tensor-core kernel when
// a TC plan is given (binary16, nb = 64, full panel), else the exact SIMT one.
template <typename T, int NB>
void trailing_update(T *a, int n, int k0, int jb, int cb, int ce, const TcPlan *tc,
                     cudaStream_t s)
{
  if constexpr (std::is_same<T, h16>::value && NB == 64)
  {
    if (tc && jb == NB)
    {
      launch_gemm_tc(*tc, k0, cb, ce, s);
      return;
    }
  }
  launch_gemm<T, NB>(a, n, k0, jb, cb, ce, ColMap{}, s);
}

template <typename T, int NB>
void lu_run(T *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info, cudaStream_t s,
            const TcPlan *tc = nullptr)
{
  const ColMap id{};
  cudaStream_t side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);  // [4][npanels]: P, N, R, F
  const int np = ws.npanels;
  if (perm)
  {
    ProfScope ps(KC_VEC, s);
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(perm, n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(ws.nmoves, 0, sizeof(int) * np, s));
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[0], s));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, ev[0], 0));
  for (int p = 0, k0 = 0; k0 < n; ++p, k0 += NB)
  {
    const int jb = std::min(NB, n - k0);
    const int c0 = k0 + jb;
    int2 *mv = ws.moves + (size_t)p * 2 * NB;
    int *nm = ws.nmoves + p;
    cudaEvent_t evP = ev[p], evN = ev[np + p], evR = ev[2 * np + p], evF = ev[3 * np + p];
    // main: the critical chain
    panel_any<T, NB>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
    MPIRG_CUDA_CHECK(cudaEventRecord(evP, s));
    const int cnext = std::min(n, c0 + NB);
    if (c0 < n)
    {
      // depth-2 look-ahead: wait only for step p-1's update of these columns
      // (issued first on the side stream), not for the whole of step p-1
      if (p > 0)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[3 * np + p - 1], 0));
      launch_mt<T, NB>(a, n, k0, jb, c0, cnext, id, mv, nm, s);
      trailing_update<T, NB>(a, n, k0, jb, c0, cnext, tc, s);
    }
    MPIRG_CUDA_CHECK(cudaEventRecord(evN, s));
    // side: the rest of this step's update + the left-column moves
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, evP, 0));
    if (cnext < n)
    {
      // the next panel's columns first: panel p+1's critical chain needs
      // only these (evF), the bulk of the update then overlaps panel p+1
      const int cnn = std::min(n, cnext + NB);
      launch_mt<T, NB>(a, n, k0, jb, cnext, cnn, id, mv, nm, side);
      trailing_update<T, NB>(a, n, k0, jb, cnext, cnn, tc, side);
      MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
      if (cnn < n)
      {
        launch_mt<T, NB>(a, n, k0, jb, cnn, n, id, mv, nm, side);
        trailing_update<T, NB>(a, n, k0, jb, cnn, n, tc, side);
      }
    }
    else
      MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
    launch_moves<T, NB>(a, n, 0, k0, id, mv, nm, perm, side);
    MPIRG_CUDA_CHECK(cudaEventRecord(evR, side));
  }
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2 * np + np - 1], 0));
}

// ---- binary16 tensor-core schedule (lu_mode TC): recursive LU ---------------
// factor(K0, w) factors columns [K0, K0 + w), rows [K0, n):
//   w <= 64:  one panel (cluster kernel), which records its row moves;
//   else:     factor the left half; apply its panels' row moves to the right
//             half; U12 = L11^-1 A12 (recursive: 64-row solves + tensor-core
//             updates); A22 -= L21 U12 on the tensor cores with K = w/2;
//             factor the right half; apply its row moves to the left half's L.
// Every update is one tcgen05 GEMM (lu_tc.cu) whose K doubles with each level:
// 7/8 of the 2n^3/3 flops run at K >= n/16, and the trailing matrix is read and
// written log2(n/64) times instead of n/64 times. The panels are factored in
// binary32 (the binary16 panel converted into a scratch buffer, the binary32
// cluster kernel, one rounding back): half the binary16 kernel's time, and no
// less accurate (the panel kernel widens on load and rounds once on store).
// Not bitwise (lu_mode EXACT is); pivots are the reference's
// whenever no near-tie is decided differently by the higher precision.
static bool tc_panel_f32()
{
  static const bool v = [] {
    const char *e = std::getenv("MPIRG_TC_PANEL");
    return !(e && std::string(e) == "f16");
  }();
  return v;
}

struct TcRun
{
  h16 *a;
  int n;
  int *ipiv, *perm;
  LuWorkspace *ws;
  DevInfo *info;
  cudaStream_t s;
  const TcPlan *tc;
};

static int tc_split(int w) { return ((w / 64 + 1) / 2) * 64; }

static void tc_panel(TcRun &R, int k0, int jb)
{
  LuWorkspace &ws = *R.ws;
  const int p = k0 / 64, n = R.n;
  int2 *mv = ws.moves + (size_t)p * 128;
  int *nm = ws.nmoves + p;
  if (tc_panel_f32() && panel_rpt<float, 64>(n - k0) > 0)
    launch_panel<float, 64, h16>(R.a, n, k0, jb, R.ipiv, mv, nm, R.info, R.s);
  else
    panel_any<h16, 64>(R.a, n, k0, jb, R.ipiv, mv, nm, ws, R.info, R.s);
  // the accumulated permutation follows on the side stream, off the chain
  if (R.perm)
  {
    cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);
    cudaStream_t side = static_cast<cudaStream_t>(ws.side);
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[p], R.s));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, ev[p], 0));
    launch_moves<h16, 64>(R.a, n, 0, 0, ColMap{}, mv, nm, R.perm, side);
  }
}

// row moves of panels [pa, pb), in order, on columns [cb, ce)
static void tc_moves(TcRun &R, int pa, int pb, int cb, int ce)
{
  if (ce <= cb || pb <= pa)
    return;
  prof_begin(KC_MOVES, R.s);
  const int grid = std::max(1, std::min((ce - cb + 7) / 8, 148 * 4));
  lu_apply_moves_multi_kernel<h16, 64><<<grid, 256, 0, R.s>>>(R.a, R.n, cb, ce, R.ws->moves,
                                                              R.ws->nmoves, pa, pb);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_MOVES, R.s);
}

// rows [K0, K0 + sz) of columns [cb, ce) <- L11^-1 (those rows), L11 unit lower at (K0, K0)
// U12 leaf of the tensor-core mode: rows [k0, k0 + jb) of columns [cb, ce)
// <- L11^-1 (those rows), jb <= LB, with the substitution in binary32
// (binary16 inputs, one FMA per term, one rounding back to binary16).
// lu_mt_kernel's layout -- 4 warps x 8 columns per CTA, lane owns rows
// lane + 32 h, x_k by shuffle -- without the per-term binary16 roundings the
// exact mode needs, and up to 256 rows per launch (L11 staged k-major as
// binary16 in shared memory), so the solve of a 256-row block is one launch
// instead of 4 leaves + 3 updates.
template <int LB>
__global__ void __launch_bounds__(256) tc_trsm_leaf_kernel(h16 *__restrict__ A, int n, int k0,
                                                           int jb, int cb, int ce,
                                                           const int2 *__restrict__ moves,
                                                           const int *__restrict__ nmoves, int pa,
                                                           int pb)
{
  constexpr int RL = LB / 32, CW = 4;  // 8 warps x 4 columns
  constexpr int PER = 4;               // 2 * 64 move entries over 32 lanes
  extern __shared__ __align__(16) unsigned char trsm_smem[];
  h16 *Ls = reinterpret_cast<h16 *>(trsm_smem);  // [kk][i], i contiguous
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // L11 (strictly lower part), 8 binary16 values per load (k0 is a multiple of 64)
  for (int idx = threadIdx.x * 8; idx < LB * LB; idx += 256 * 8)
  {
    const int kk = idx / LB, i = idx % LB;
    unsigned short e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (kk < jb && i < jb && i + 7 > kk)
    {
      if (i + 8 <= jb)
      {
        const uint4 w = *reinterpret_cast<const uint4 *>(A + (size_t)(k0 + kk) * n + k0 + i);
        const unsigned int ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
          e[q] = (unsigned short)(ww[q >> 1] >> (16 * (q & 1)));
      }
      else
      {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          e[q] = i + q < jb ? A[(size_t)(k0 + kk) * n + k0 + i + q].bits : (unsigned short)0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (i + q <= kk)
          e[q] = 0;  // only the strictly lower part: rows <= kk are final at step kk
    }
    const uint4 v = make_uint4(e[0] | ((unsigned)e[1] << 16), e[2] | ((unsigned)e[3] << 16),
                               e[4] | ((unsigned)e[5] << 16), e[6] | ((unsigned)e[7] << 16));
    *reinterpret_cast<uint4 *>(Ls + idx) = v;
  }
  const int col0 = cb + blockIdx.x * MT_COLS + warp * CW;
  // the row moves of panels [pa, pb), in order, on this warp's columns (the
  // columns of a block's right half take the left half's moves here instead
  // of in a launch of their own)
  for (int p = pa; p < pb; ++p)
  {
    const int nm = nmoves[p];
    if (nm == 0)
      continue;
    int2 mv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
    {
      const int e = lane + 32 * q;
      mv[q] = e < nm ? moves[(size_t)p * 128 + e] : make_int2(-1, -1);
    }
#pragma unroll
    for (int u = 0; u < CW; ++u)
      if (col0 + u < ce)
      {
        h16 *cp = A + (size_t)(col0 + u) * n;
        h16 v[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            v[q] = cp[mv[q].y];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            cp[mv[q].x] = v[q];
        __syncwarp();
      }
  }
  float x[CW][RL];
#pragma unroll
  for (int u = 0; u < CW; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      x[u][h] = (col0 + u < ce && i < jb) ? h2f(A[(size_t)(col0 + u) * n + k0 + i]) : 0.f;
    }
  __syncthreads();
#pragma unroll
  for (int hk = 0; hk < RL; ++hk)
  {
    if (32 * hk >= jb)
      break;
#pragma unroll 8
    for (int lk = 0; lk < 32; ++lk)
    {
      const int kk = 32 * hk + lk;  // rows above 32 hk are final: only slots h >= hk change
      float lv[RL];
#pragma unroll
      for (int h = hk; h < RL; ++h)
        lv[h] = h2f(Ls[kk * LB + lane + 32 * h]);  // 0 for rows <= kk and beyond jb
#pragma unroll
      for (int u = 0; u < CW; ++u)
      {
        const float xk = __shfl_sync(0xffffffffu, x[u][hk], lk);
#pragma unroll
        for (int h = hk; h < RL; ++h)
          x[u][h] = __fmaf_rn(-lv[h], xk, x[u][h]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CW; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      if (col0 + u < ce && i < jb)
        A[(size_t)(col0 + u) * n + k0 + i] = f2h(x[u][h]);
    }
}

template <int LB>
static void tc_trsm_leaf(TcRun &R, int K0, int sz, int cb, int ce, int pa, int pb)
{
  constexpr int smem = LB * LB * 2;
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(tc_trsm_leaf_kernel<LB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.done();
  }
  tc_trsm_leaf_kernel<LB><<<(ce - cb + MT_COLS - 1) / MT_COLS, 256, smem, R.s>>>(
      R.a, R.n, K0, sz, cb, ce, R.ws->moves, R.ws->nmoves, pa, pb);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// [pa, pb): panels whose row moves the first leaf applies to the columns (none: pa == pb)
static void tc_trsm(TcRun &R, int K0, int sz, int cb, int ce, int pa = 0, int pb = 0)
{
  if (sz <= 256)
  {
    if (ce <= cb)
      return;
    prof_begin(KC_TRSM, R.s);
    if (sz <= 64)
      tc_trsm_leaf<64>(R, K0, sz, cb, ce, pa, pb);
    else if (sz <= 128)
      tc_trsm_leaf<128>(R, K0, sz, cb, ce, pa, pb);
    else
      tc_trsm_leaf<256>(R, K0, sz, cb, ce, pa, pb);
    prof_end(KC_TRSM, R.s);
    return;
  }
  const int h = tc_split(sz);
  tc_trsm(R, K0, h, cb, ce, pa, pb);  // the moves go with the first leaf only
  tc_gemm(*R.tc, K0 + h, K0 + sz, cb, ce, K0, h, R.s, KC_TRSM);
  tc_trsm(R, K0 + h, sz - h, cb, ce);
}

static void tc_factor(TcRun &R, int K0, int w)
{
  if (w <= 64)
  {
    tc_panel(R, K0, w);
    return;
  }
  const int h = tc_split(w);
  tc_factor(R, K0, h);
  // the left half's row moves reach the right half inside the U12 solve's first leaf
  tc_trsm(R, K0, h, K0 + h, K0 + w, K0 / 64, (K0 + h) / 64);
  tc_gemm(*R.tc, K0 + h, R.n, K0 + h, K0 + w, K0, h, R.s);
  tc_factor(R, K0 + h, w - h);
  tc_moves(R, (K0 + h) / 64, (K0 + w + 63) / 64, K0, K0 + h);
}

static void lu_run_tc_body(h16 *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                           cudaStream_t s, const TcPlan &tc)
{
  cudaStream_t side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);
  const int np = ws.npanels;
  if (perm)
  {
    ProfScope ps(KC_VEC, s);
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(perm, n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(ws.nmoves, 0, sizeof(int) * np, s));
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[np], s));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, ev[np], 0));
  TcRun R{a, n, ipiv, perm, &ws, info, s, &tc};
  tc_factor(R, 0, n);
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[np + 1], side));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[np + 1], 0));
}

// ---- binary32 single-GPU schedule: TMA trailing update, paired steps ------
// MPIRG_GEMM=v4 keeps the one-step-per-pass schedule of lu_run (A/B runs).
static int f32_mode()
{
  static const int v = [] {
    const char *e = std::getenv("MPIRG_GEMM");
    if (e && (std::string(e) == "v4" || std::string(e) == "scalar"))
      return 0;
    return 1;
  }();
  return v;
}

struct F32Plan
{
  CUtensorMap a128, u128, a64, u64;  // L21 (over ls) and U12 (over ut) boxes
  float *a = nullptr, *ut = nullptr;
  const float *ls = nullptr;  // where the L factors are read (a, or the panel snapshots)
  int n = 0;
  // columns per warp of the critical next-panel U12 solve: 1 from device memory
  // (LU 4.01 -> 3.81 ms on cfg 2a), 2 inside the streamed refactor, whose late
  // chunks run beside the chain (there 1 measured slower: 4.85 vs 4.64 ms)
  int next_cpw = 2;
};

static void f32_encode(CUtensorMap *map, float *base, int inner, int outer, int box0)
{
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)f32u::GKC};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = tma_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims,
                                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed for the fp32 trailing update");
}

static void f32_plan_make(F32Plan &p, float *a, int n, float *ut, int ut_rows,
                          float *ls = nullptr)
{
  p.a = a;
  p.n = n;
  p.ut = ut;
  p.ls = ls ? ls : a;
  f32_encode(&p.a128, ls ? ls : a, n, n, 128);
  f32_encode(&p.a64, ls ? ls : a, n, n, 64);
  f32_encode(&p.u128, ut, n, ut_rows, 128);
  f32_encode(&p.u64, ut, n, ut_rows, 64);
}

template <int NB>
static void f32_mt(const F32Plan &P, int k0, int jb, int cb, int ce, const int2 *mv,
                   const int *nm, int kp, int ut_row, cudaStream_t s, bool chain = false)
{
  if (ce <= cb)
    return;
  prof_begin(KC_TRSM, s);
  if (ce - cb <= NB && P.next_cpw == 1 && chain && kp < 0 && lu_pdl() >= 2)
  {
    // right behind the panel in the chain's stream: programmatic launch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((ce - cb + 3) / 4);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, f32u::mt2_kernel<NB, false, 1>, P.a, P.n, k0, jb, cb,
                                        ce, mv, nm, 0, P.ut, ut_row, (const float *)P.ls,
                                        BatchStride{}, 0));
  }
  else if (ce - cb <= NB && P.next_cpw == 1)
  {
    // the critical chain's next-panel block: one column per warp
    const int g = (ce - cb + 3) / 4;
    if (kp >= 0)
      f32u::mt2_kernel<NB, true, 1><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, kp, P.ut,
                                                     ut_row, P.ls);
    else
      f32u::mt2_kernel<NB, false, 1><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, 0, P.ut,
                                                      ut_row, P.ls);
  }
  else if (ce - cb <= NB)
  {
    // the same block with two columns per warp
    const int g = (ce - cb + 7) / 8;
    if (kp >= 0)
      f32u::mt2_kernel<NB, true, 2><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, kp, P.ut,
                                                     ut_row, P.ls);
    else
      f32u::mt2_kernel<NB, false, 2><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, 0, P.ut,
                                                      ut_row, P.ls);
  }
  else
  {
    const int g = (ce - cb + f32u::MT_COLS - 1) / f32u::MT_COLS;
    if (kp >= 0)
      f32u::mt2_kernel<NB, true><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, kp, P.ut,
                                                  ut_row, P.ls);
    else
      f32u::mt2_kernel<NB, false><<<g, 128, 0, s>>>(P.a, P.n, k0, jb, cb, ce, mv, nm, 0, P.ut,
                                                   ut_row, P.ls);
  }
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_TRSM, s);
}

// The critical chain's next-column block in one fused launch (lu_f32.cuh
// next_kernel), opt-in with MPIRG_LU_NEXT=1. Bitwise equal to the two-launch
// form, but measured slower on B200 inside the 16-SM partition (cfg 2a LU
// 4.56 -> 4.75 ms, profiles/r01g_next_fused_experiment.txt), so the default
// stays mt2_kernel + gemm_tma_kernel.
static bool next_fused()
{
  static const bool v = [] {
    const char *e = std::getenv("MPIRG_LU_NEXT");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

template <int NB>
static bool f32_next(const F32Plan &P, int k0, int jb, int cb, int ce, const int2 *mv,
                     const int *nm, int ut_row, cudaStream_t s)
{
  if constexpr (NB != 64)
    return false;
  else
  {
    if (!next_fused() || P.ls != P.a || ce <= cb || ce - cb > NB)
      return false;
    static DeviceOnce configured;
    if (configured.needed())
    {
      MPIRG_CUDA_CHECK(cudaFuncSetAttribute(f32u::next_kernel<NB>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)f32u::next_smem<NB>()));
      MPIRG_CUDA_CHECK(cudaFuncSetAttribute(f32u::next_kernel<NB>,
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      configured.done();
    }
    const int ntile = (P.n - (k0 + jb) + f32u::NX_TM - 1) / f32u::NX_TM;
    const int cs = std::max(1, std::min(16, ntile));
    prof_begin(KC_GEMM, s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = f32u::next_smem<NB>();
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, f32u::next_kernel<NB>, P.a, P.n, k0, jb, cb, ce,
                                        mv, nm, P.ut, ut_row));
    prof_end(KC_GEMM, s);
    return true;
  }
}

template <int BM>
static void f32_gemm_t(const CUtensorMap &ma, const CUtensorMap &mu, const F32Plan &P, int k0,
                       int K, int ut_row, int cb, int ce, cudaStream_t s)
{
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(f32u::gemm_tma_kernel<BM>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)f32u::gemm_tma_smem<BM>()));
    configured.done();
  }
  const int c0 = k0 + K;
  const dim3 grid((P.n - c0 + BM - 1) / BM, (ce - cb + BM - 1) / BM);
  if (BM == 64 && lu_pdl() && ce - cb <= 64)
  {
    // the chain's update right behind its U12 solve in the same stream
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = f32u::gemm_tma_smem<BM>();
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, f32u::gemm_tma_kernel<BM>, ma, mu, P.a, P.n, k0, K,
                                        ut_row, cb, ce));
    return;
  }
  f32u::gemm_tma_kernel<BM><<<grid, 256, f32u::gemm_tma_smem<BM>(), s>>>(ma, mu, P.a, P.n, k0,
                                                                        K, ut_row, cb, ce);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// rows [k0 + K, n) x columns [cb, ce) -= L(:, k0 .. k0+K) U(k0 .. k0+K, :), U from ut rows
// [ut_row, ut_row + K)
static void f32_gemm(const F32Plan &P, int k0, int K, int ut_row, int cb, int ce, cudaStream_t s)
{
  const int c0 = k0 + K;
  if (ce <= cb || c0 >= P.n)
    return;
  prof_begin(KC_GEMM, s);
  const long tiles128 = (long)((P.n - c0 + 127) / 128) * ((ce - cb + 127) / 128);
  if (tiles128 >= 2 * 148)
    f32_gemm_t<128>(P.a128, P.u128, P, k0, K, ut_row, cb, ce, s);
  else
    f32_gemm_t<64>(P.a64, P.u64, P, k0, K, ut_row, cb, ce, s);
  prof_end(KC_GEMM, s);
}

// Same dependency structure as lu_run (critical chain on s, bulk on the side
// stream), plus pairing: an even step p whose far columns [c0 + 2nb, n) are
// not needed by the next panel only solves their U12 rows; the odd step p+1
// then applies its row moves to them and to panel p's L columns, the pending
// step-p update of its own panel rows (inside the U12 solve), and one K = 2nb
// update (lu_f32.cuh explains why the bits are unchanged).
// MPIRG_LU_TIMELINE=1: timing events along the critical chain of lu_run_f32,
// summarised on stderr (diagnostics only; synchronises at the end).
struct LuTimeline
{
  bool on = false;
  std::vector<cudaEvent_t> ev;  // [np][6]: panel start/end, mt end, gemm end, F end, R end
  int np = 0;
  void init(int n_panels)
  {
    static const bool env = std::getenv("MPIRG_LU_TIMELINE") != nullptr;
    on = env;
    if (!on)
      return;
    np = n_panels;
    ev.resize((size_t)np * 6);
    for (auto &e : ev)
      MPIRG_CUDA_CHECK(cudaEventCreate(&e));
  }
  void mark(int p, int i, cudaStream_t s)
  {
    if (on)
      MPIRG_CUDA_CHECK(cudaEventRecord(ev[(size_t)p * 6 + i], s));
  }
  void report()
  {
    if (!on)
      return;
    MPIRG_CUDA_CHECK(cudaDeviceSynchronize());
    auto t = [&](int p, int i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0], ev[(size_t)p * 6 + i]);
      return (double)ms * 1e3;
    };
    double sp = 0, sm = 0, sg = 0, sw = 0;
    for (int p = 0; p < np; ++p)
    {
      const double a = t(p, 0), b = t(p, 1), c = t(p, 2), d = t(p, 3);
      sp += b - a;
      sm += c - b;
      sg += d - c;
      if (p + 1 < np)
        sw += t(p + 1, 0) - d;
      if (p < 8 || p % 16 == 0 || p == np - 1)
        std::fprintf(stderr,
                     "step %3d start %9.1f panel %6.1f mt %5.1f gemm %5.1f | F %9.1f R %9.1f us\n",
                     p, a, b - a, c - b, d - c, t(p, 4), t(p, 5));
    }
    std::fprintf(stderr, "chain totals (us): panel %.0f mt %.0f gemm %.0f wait %.0f end %.0f\n",
                 sp, sm, sg, sw, t(np - 1, 5));
    for (auto &e : ev)
      cudaEventDestroy(e);
    ev.clear();
  }
};

// Snapshot of panel columns [k0, k0 + jb), rows [k0, n) (a kernel, not a
// DMA copy: the copy engines are busy with the host-to-device stream).
__global__ void panel_snapshot_kernel(const float *__restrict__ a, float *__restrict__ dst, int n,
                                      int k0, int jb)
{
  const int rows = n - k0;
  const int r4 = (rows + 3) / 4;
  const int tot = r4 * jb;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x)
  {
    const int c = i / r4, q = i - c * r4;
    const size_t base = (size_t)(k0 + c) * n + k0;
    const int r = 4 * q;
    if (((k0 & 3) == 0) && r + 3 < rows)
      *reinterpret_cast<float4 *>(dst + base + r) =
          *reinterpret_cast<const float4 *>(a + base + r);
    else
      for (int e = 0; e < 4 && r + e < rows; ++e)
        dst[base + r + e] = a[base + r + e];
  }
}

// Late-column resources of a workspace (launch_lu_late), allocated on first use.
struct LateRes
{
  float *lsnap;
  float *utl;
  cudaStream_t *st;
  cudaEvent_t *ev;  // [late_np] snapshot taken, then [MAXCH] chunk caught up
};

static LateRes late_res(LuWorkspace &ws, int n, int nb)
{
  const int np = (n + nb - 1) / nb;
  if (ws.late_n < n || ws.late_np < np)
  {
    if (ws.lsnap)
    {
      cudaFree(ws.lsnap);
      cudaFree(ws.utl);
      auto *st = static_cast<cudaStream_t *>(ws.lstreams);
      for (int i = 0; i < LuLate::MAXCH; ++i)
        cudaStreamDestroy(st[i]);
      delete[] st;
      auto *ev = static_cast<cudaEvent_t *>(ws.levents);
      for (int i = 0; i < ws.late_np + LuLate::MAXCH; ++i)
        cudaEventDestroy(ev[i]);
      delete[] ev;
    }
    MPIRG_CUDA_CHECK(cudaMalloc(&ws.lsnap, sizeof(float) * (size_t)n * n));
    MPIRG_CUDA_CHECK(cudaMalloc(&ws.utl, sizeof(float) * (size_t)LuLate::MAXCH * nb * n));
    auto *st = new cudaStream_t[LuLate::MAXCH];
    for (int i = 0; i < LuLate::MAXCH; ++i)
      st[i] = lu_bulk_stream_create();
    ws.lstreams = st;
    auto *ev = new cudaEvent_t[np + LuLate::MAXCH];
    for (int i = 0; i < np + LuLate::MAXCH; ++i)
      MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    ws.levents = ev;
    ws.late_n = n;
    ws.late_np = np;
  }
  return {static_cast<float *>(ws.lsnap), static_cast<float *>(ws.utl),
          static_cast<cudaStream_t *>(ws.lstreams), static_cast<cudaEvent_t *>(ws.levents)};
}

template <int NB>
void lu_run_f32_body(float *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                     cudaStream_t caller, const LuLate *late = nullptr)
{
  // the critical chain runs on the caller's stream, or on the critical SM
  // group's stream when the SMs are partitioned (MPIRG_LU_GREEN)
  cudaStream_t s = ws.crit ? static_cast<cudaStream_t>(ws.crit) : caller;
  cudaEvent_t *evx = static_cast<cudaEvent_t *>(ws.events);
  if (s != caller)
  {
    MPIRG_CUDA_CHECK(cudaEventRecord(evx[1], caller));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, evx[1], 0));
  }
  const ColMap id{};
  cudaStream_t side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);  // [4][npanels]: P, N, R, F
  const int np = ws.npanels;
  F32Plan P;
  f32_plan_make(P, a, n, static_cast<float *>(ws.ut), 2 * NB);
  {
    static const int forced = [] {
      const char *e = std::getenv("MPIRG_NEXT_CPW");
      return e ? std::atoi(e) : 0;
    }();
    P.next_cpw = forced ? forced : (late ? 2 : 1);
  }
  // late columns: chunk c (c >= 1) is updated on its own stream from panel
  // snapshots until step join[c]; the regular schedule's far columns end at
  // rlim(p) = the first column of the first chunk not yet joined
  const int nlate = late ? late->nch : 0;
  LateRes LR{};
  F32Plan PL[LuLate::MAXCH];
  int last_join = 0;
  if (nlate > 1)
  {
    LR = late_res(ws, n, NB);
    for (int c = 1; c < nlate; ++c)
    {
      f32_plan_make(PL[c], a, n, LR.utl + (size_t)c * NB * n, NB, LR.lsnap);
      last_join = std::max(last_join, late->join[c]);
    }
  }
  auto rlim = [&](int p) {
    int r = n;
    for (int c = 1; c < nlate; ++c)
      if (late->join[c] > p)
        r = std::min(r, late->lo[c]);
    return r;
  };
  if (perm)
  {
    ProfScope ps(KC_VEC, s);
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(perm, n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(ws.nmoves, 0, sizeof(int) * np, s));
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[0], s));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, ev[0], 0));
  bool prev_deferred = false;
  LuTimeline tl;
  tl.init(np);
  for (int p = 0, k0 = 0; k0 < n; ++p, k0 += NB)
  {
    const int jb = std::min(NB, n - k0);
    const int c0 = k0 + jb;
    const int cnext = std::min(n, c0 + NB);
    const int cnn = std::min(n, cnext + NB);
    const int ur = (p & 1) * NB;  // this step's rows of ut
    int2 *mv = ws.moves + (size_t)p * 2 * NB;
    int *nm = ws.nmoves + p;
    cudaEvent_t evP = ev[p], evN = ev[np + p], evR = ev[2 * np + p], evF = ev[3 * np + p];
    const bool pend = prev_deferred;  // step p-1 left its far-column update to this step
    const int rl = rlim(p);
    const bool defer = !pend && (p & 1) == 0 && cnn < rl && jb == NB;
    const int kp = k0 - NB;
    tl.mark(p, 0, s);
    panel_any<float, NB>(a, n, k0, jb, ipiv, mv, nm, ws, info, s);
    MPIRG_CUDA_CHECK(cudaEventRecord(evP, s));
    tl.mark(p, 1, s);
    if (c0 < n)
    {
      if (p > 0)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[3 * np + p - 1], 0));
      if (f32_next<NB>(P, k0, jb, c0, cnext, mv, nm, ur, s))
        tl.mark(p, 2, s);
      else
      {
        f32_mt<NB>(P, k0, jb, c0, cnext, mv, nm, -1, ur, s, true);
        tl.mark(p, 2, s);
        f32_gemm(P, k0, jb, ur, c0, cnext, s);
      }
    }
    else
      tl.mark(p, 2, s);
    tl.mark(p, 3, s);
    MPIRG_CUDA_CHECK(cudaEventRecord(evN, s));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, evP, 0));
    if (nlate > 1 && p < last_join)
    {
      // snapshot of panel p (rows k0.., as it left the panel) for the late chunks
      {
        const int tot = ((n - k0 + 3) / 4) * jb;
        panel_snapshot_kernel<<<std::min(148 * 2, (tot + 255) / 256), 256, 0, side>>>(
            a, LR.lsnap, n, k0, jb);
        MPIRG_CUDA_CHECK(cudaGetLastError());
      }
      MPIRG_CUDA_CHECK(cudaEventRecord(LR.ev[p], side));
      // one stream per late chunk (they wait for different host-to-device
      // chunks; CUDA_DEVICE_MAX_CONNECTIONS=32 keeps them off each other's
      // hardware queues, paper_2311_14616_b200/__init__.py)
      for (int c = 1; c < nlate; ++c)
      {
        if (late->join[c] <= p)
          continue;
        cudaStream_t ls = LR.st[c];
        if (p == 0)
          MPIRG_CUDA_CHECK(cudaStreamWaitEvent(ls, static_cast<cudaEvent_t>(late->ready[c]), 0));
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(ls, LR.ev[p], 0));
        f32_mt<NB>(PL[c], k0, jb, late->lo[c], late->hi[c], mv, nm, -1, 0, ls);
        f32_gemm(PL[c], k0, jb, 0, late->lo[c], late->hi[c], ls);
        if (p == late->join[c] - 1)
          MPIRG_CUDA_CHECK(cudaEventRecord(LR.ev[ws.late_np + c], ls));
      }
    }
    for (int c = 1; c < nlate; ++c)
      if (late->join[c] == p)  // chunk c joins the regular schedule at this step
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, LR.ev[ws.late_np + c], 0));
    if (pend)  // panel p-1's L rows follow this step's row moves before they are used
      launch_moves<float, NB>(a, n, kp, k0, id, mv, nm, nullptr, side);
    if (cnext < n)
    {
      if (pend)
      {
        f32_mt<NB>(P, k0, jb, cnext, cnn, mv, nm, kp, ur, side);
        f32_gemm(P, kp, NB + jb, 0, cnext, cnn, side);
      }
      else
      {
        f32_mt<NB>(P, k0, jb, cnext, cnn, mv, nm, -1, ur, side);
        f32_gemm(P, k0, jb, ur, cnext, cnn, side);
      }
      MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
      tl.mark(p, 4, side);
      if (cnn < rl)
      {
        if (pend)
        {
          f32_mt<NB>(P, k0, jb, cnn, rl, mv, nm, kp, ur, side);
          f32_gemm(P, kp, NB + jb, 0, cnn, rl, side);
        }
        else
        {
          f32_mt<NB>(P, k0, jb, cnn, rl, mv, nm, -1, ur, side);
          if (!defer)
            f32_gemm(P, k0, jb, ur, cnn, rl, side);
        }
      }
    }
    else
    {
      MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
      tl.mark(p, 4, side);
    }
    launch_moves<float, NB>(a, n, 0, pend ? kp : k0, id, mv, nm, perm, side);
    MPIRG_CUDA_CHECK(cudaEventRecord(evR, side));
    tl.mark(p, 5, side);
    prev_deferred = defer;
  }
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2 * np + np - 1], 0));
  if (s != caller)
  {
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[np + np - 1], s));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(caller, ev[np + np - 1], 0));
  }
  tl.report();
}

// The binary32 schedule issues ~6 launches per panel step across two streams;
// on the critical chain each dependent launch costs a few microseconds of
// launch latency. The whole schedule is therefore captured once per
// (matrix, workspace) into a CUDA graph and replayed (MPIRG_LU_GRAPH=0 turns
// this off; profiling and the timeline always run the streams directly).
struct LuGraphKey
{
  const void *a, *ipiv, *perm, *info, *ws_moves;
  int n;
  cudaStream_t caller;
  bool operator==(const LuGraphKey &o) const
  {
    return a == o.a && ipiv == o.ipiv && perm == o.perm && info == o.info &&
           ws_moves == o.ws_moves && n == o.n && caller == o.caller;
  }
};
struct LuGraphEntry
{
  LuGraphKey key;
  cudaGraphExec_t exec;
};

static bool lu_graph_enabled()
{
  static const bool v = [] {
    const char *e = std::getenv("MPIRG_LU_GRAPH");
    return !(e && std::atoi(e) == 0) && std::getenv("MPIRG_LU_TIMELINE") == nullptr &&
           !tool_attached();
  }();
  return v;
}

static std::mutex g_lu_graph_mu;
static std::vector<LuGraphEntry> g_lu_graphs;

// Drops the cached graphs of a workspace being freed (its streams/events die).
static void lu_graph_forget(const void *ws_moves)
{
  std::lock_guard<std::mutex> lk(g_lu_graph_mu);
  for (size_t i = 0; i < g_lu_graphs.size();)
  {
    if (g_lu_graphs[i].key.ws_moves == ws_moves)
    {
      cudaGraphExecDestroy(g_lu_graphs[i].exec);
      g_lu_graphs.erase(g_lu_graphs.begin() + i);
    }
    else
      ++i;
  }
}

// Runs body() on `caller`, captured once per key into a CUDA graph and
// replayed afterwards (directly when graphs are off, under the per-kernel
// profile, or on a legacy/per-thread default stream, which cannot capture).
template <typename Body>
static void run_with_graph(const LuGraphKey &key, cudaStream_t caller, Body &&body)
{
  if (!lu_graph_enabled() || prof_on() || caller == nullptr || caller == cudaStreamLegacy ||
      caller == cudaStreamPerThread)
  {
    body();
    return;
  }
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_lu_graph_mu);
    for (auto &e : g_lu_graphs)
      if (e.key == key)
        exec = e.exec;
  }
  if (!exec)
  {
    cudaGraph_t g = nullptr;
    MPIRG_CUDA_CHECK(cudaStreamBeginCapture(caller, cudaStreamCaptureModeThreadLocal));
    try
    {
      body();
    }
    catch (...)
    {
      cudaStreamEndCapture(caller, &g);
      if (g)
        cudaGraphDestroy(g);
      throw;
    }
    MPIRG_CUDA_CHECK(cudaStreamEndCapture(caller, &g));
    MPIRG_CUDA_CHECK(cudaGraphInstantiate(&exec, g, 0));
    cudaGraphDestroy(g);
    std::lock_guard<std::mutex> lk(g_lu_graph_mu);
    g_lu_graphs.push_back({key, exec});
  }
  MPIRG_CUDA_CHECK(cudaGraphLaunch(exec, caller));
}

template <int NB>
void lu_run_f32(float *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                cudaStream_t caller)
{
  run_with_graph(LuGraphKey{a, ipiv, perm, info, ws.moves, n, caller}, caller,
                 [&] { lu_run_f32_body<NB>(a, n, ipiv, perm, ws, info, caller); });
}

// The recursive tensor-core LU issues ~1500 small dependent launches at
// n = 8192; replayed as one graph their launch gaps shrink to the
// node-to-node latency.
static void lu_run_tc(h16 *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                      cudaStream_t caller, const TcPlan &tc)
{
  run_with_graph(LuGraphKey{a, ipiv, perm, info, ws.moves, n, caller}, caller,
                 [&] { lu_run_tc_body(a, n, ipiv, perm, ws, info, caller, tc); });
}

// ---- one rank of the 1-D block-cyclic LU (config 5a) ----------------------
// Step p (k0 = p*nb): the owner of column block p factors the panel
// (dlu_panel); the panel rows [k0, n), its pivots and its row moves go to
// every rank (the caller's broadcast); every rank then applies the moves,
// U12 = L11^-1 A12 and A22 -= L21 U12 to the columns it owns (dlu_update).
// part 1 (NEXT) updates only the next panel's columns when this rank owns
// them (look-ahead on the caller's stream); part 2 (REST) the remaining
// owned columns + the left-column moves on the side stream; part 0 both.
template <typename T, int NB>
void dlu_update_t(DluPlan &d, T *a, int p, int part, int *perm, cudaStream_t s)
{
  LuWorkspace &ws = d.ws;
  const ColMap map{d.G, d.r, d.sh};
  const int n = d.n, np = ws.npanels;
  const int k0 = p * NB, jb = std::min(NB, n - k0), c0 = k0 + jb;
  const int cnext = std::min(n, c0 + NB);
  // [c0, cnext) lies in one distribution block (block_cols is a multiple of nb)
  const bool nextmine = p + 1 < np && ((c0 >> d.sh) % d.G) == d.r;
  const int2 *mv = ws.moves + (size_t)p * 2 * NB;
  const int *nm = ws.nmoves + p;
  cudaStream_t side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);
  const int Lc0 = map.lcount(c0), Lcn = map.lcount(cnext), Ln = map.lcount(n);
  if (part == 0 || part == 1)
  {
    if (nextmine)
    {
      if (part == 1 && p > 0)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2 * np + p - 1], 0));
      launch_mt<T, NB>(a, n, k0, jb, Lc0, Lcn, map, mv, nm, s);
      launch_gemm<T, NB>(a, n, k0, jb, Lc0, Lcn, map, s);
    }
  }
  if (part == 0 || part == 2)
  {
    cudaStream_t t = part == 0 ? s : side;
    if (part == 2)
    {
      MPIRG_CUDA_CHECK(cudaEventRecord(ev[p], s));
      MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, ev[p], 0));
    }
    const int Lb = nextmine ? Lcn : Lc0;
    launch_mt<T, NB>(a, n, k0, jb, Lb, Ln, map, mv, nm, t);
    launch_gemm<T, NB>(a, n, k0, jb, Lb, Ln, map, t);
    launch_moves<T, NB>(a, n, 0, map.lcount(k0), map, mv, nm, perm, t);
    if (part == 2)
      MPIRG_CUDA_CHECK(cudaEventRecord(ev[2 * np + p], side));
  }
}

// ---- one rank of the 1-D block-cyclic LU, binary32 paired schedule -------------
// lu_run_f32_body with ownership: every column range of the single-GPU step
// is cut into this rank's contiguous runs (whole distribution blocks, or the
// parts of them inside the range); with G = 1 there is one run per range and
// the launches are exactly the single-GPU ones. Panel p reaches the rank's
// buffer by dlu_panel (owner) or by the caller's broadcast + unpack; its L
// columns are kept by every rank until the paired update of step p+1 has read
// them, so step p+1's row moves are applied to every rank's copy.
struct DluF32State
{
  F32Plan P;
  float *a = nullptr;
  bool prev_deferred = false;
  cudaStream_t s = nullptr;
};

template <typename F>
static void for_owned_runs(const DluPlan &d, int lo, int hi, F &&f)
{
  if (lo >= hi)
    return;
  if (d.G == 1)
  {
    f(lo, hi);
    return;
  }
  const int B = 1 << d.sh;
  for (int b = lo >> d.sh; b * B < hi; ++b)
  {
    if (b % d.G != d.r)
      continue;
    const int gb = std::max(lo, b * B), ge = std::min(hi, (b + 1) * B);
    if (gb < ge)
      f(gb, ge);
  }
}

template <int NB>
static void dlu_f32_step_t(DluPlan &d, int p, int *perm, bool own_panel)
{
  auto &st = *static_cast<DluF32State *>(d.f32);
  LuWorkspace &ws = d.ws;
  const F32Plan &P = st.P;
  float *a = st.a;
  const ColMap map{d.G, d.r, d.sh};
  const ColMap id{};
  const int n = d.n, np = ws.npanels;
  cudaStream_t s = st.s, side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);  // [4][np]: P, N, R, F
  const int k0 = p * NB, jb = std::min(NB, n - k0), c0 = k0 + jb;
  const int cnext = std::min(n, c0 + NB), cnn = std::min(n, cnext + NB);
  const int ur = (p & 1) * NB;
  const int2 *mv = ws.moves + (size_t)p * 2 * NB;
  const int *nm = ws.nmoves + p;
  cudaEvent_t evP = ev[p], evR = ev[2 * np + p], evF = ev[3 * np + p];
  const bool pend = st.prev_deferred;
  const bool defer = !pend && (p & 1) == 0 && cnn < n && jb == NB;
  const int kp = k0 - NB;
  auto mine = [&](int c) { return d.G == 1 || ((c >> d.sh) % d.G) == d.r; };
  // critical chain: the next panel's columns, when this rank factors them
  if (c0 < n && mine(c0))
  {
    if (!own_panel)
      MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, evP, 0));
    if (p > 0)
      MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[3 * np + p - 1], 0));
    f32_mt<NB>(P, k0, jb, c0, cnext, mv, nm, -1, ur, s);
    f32_gemm(P, k0, jb, ur, c0, cnext, s);
  }
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, evP, 0));
  if (pend)  // this rank's copy of panel p-1's L rows follows step p's row moves
    launch_moves<float, NB>(a, n, kp, k0, id, mv, nm, nullptr, side);
  auto update = [&](int gb, int ge, bool do_gemm) {
    if (pend)
    {
      f32_mt<NB>(P, k0, jb, gb, ge, mv, nm, kp, ur, side);
      f32_gemm(P, kp, NB + jb, 0, gb, ge, side);
    }
    else
    {
      f32_mt<NB>(P, k0, jb, gb, ge, mv, nm, -1, ur, side);
      if (do_gemm)
        f32_gemm(P, k0, jb, ur, gb, ge, side);
    }
  };
  if (cnext < n)
  {
    if (mine(cnext))
      update(cnext, cnn, true);
    MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
    for_owned_runs(d, cnn, n, [&](int gb, int ge) { update(gb, ge, !defer); });
  }
  else
    MPIRG_CUDA_CHECK(cudaEventRecord(evF, side));
  launch_moves<float, NB>(a, n, 0, map.lcount(pend ? kp : k0), map, mv, nm, perm, side);
  MPIRG_CUDA_CHECK(cudaEventRecord(evR, side));
  st.prev_deferred = defer;
}

template <typename T, int NB>
void dlu_panel_t(DluPlan &d, T *a, int p, int *ipiv, DevInfo *info, cudaStream_t s)
{
  const int k0 = p * NB, jb = std::min(NB, d.n - k0);
  panel_any<T, NB>(a, d.n, k0, jb, ipiv, d.ws.moves + (size_t)p * 2 * NB, d.ws.nmoves + p,
                   d.ws, info, s);
}

}  // namespace

// ---- config 5b: the binary32 LU of ns independent systems per launch ---------
// System z of a launch is blockIdx.z: matrix a + z n^2, pivots ipiv + z n,
// permutation perm + z n, row moves moves + z (np 2 nb), counts nmoves + z np,
// error record info + z. Right-looking steps with no look-ahead (the batch is
// the parallelism): per step one panel launch (one thread-block cluster per
// system), one U12 solve, one trailing update, one left-column move launch --
// 4 launches per step for the whole group instead of ~6 per system. Every
// kernel is the single-system one, so each system's factors are the
// reference's bit for bit.
__global__ void iota_batch_kernel(int *p, int n)
{
  int *q = p + (size_t)blockIdx.y * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    q[i] = i;
}

void launch_lu_batched_f32(float *a, int n, int ns, int *ipiv, int *perm, int2 *moves,
                           int *nmoves, DevInfo *info, cudaStream_t s, float *ut)
{
  constexpr int NB = 64;
  if (n <= 0 || ns <= 0)
    return;
  // with a ut scratch (NB x n ns floats): the TMA-fed update of lu_f32.cuh, the
  // whole group being one n x (n ns) matrix to the tensor maps
  const bool tma = ut != nullptr && f32_mode() && (long)n * ns < (1l << 31);
  CUtensorMap mA128, mA64, mU128, mU64;
  if (tma)
  {
    f32_encode(&mA128, a, n, n * ns, 128);
    f32_encode(&mA64, a, n, n * ns, 64);
    f32_encode(&mU128, ut, n * ns, NB, 128);
    f32_encode(&mU64, ut, n * ns, NB, 64);
    static DeviceOnce tcfg;
    if (tcfg.needed())
    {
      MPIRG_CUDA_CHECK(cudaFuncSetAttribute(f32u::gemm_tma_kernel<128>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)f32u::gemm_tma_smem<128>()));
      MPIRG_CUDA_CHECK(cudaFuncSetAttribute(f32u::gemm_tma_kernel<64>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)f32u::gemm_tma_smem<64>()));
      tcfg.done();
    }
  }
  const int np = (n + NB - 1) / NB;
  BatchStride bs;
  bs.a = (size_t)n * n;
  bs.vec = n;
  bs.moves = np * 2 * NB;
  bs.nm = np;
  bs.info = 1;
  const ColMap id{};
  {
    ProfScope ps(KC_VEC, s);
    iota_batch_kernel<<<dim3((n + 255) / 256, ns), 256, 0, s>>>(perm, n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(nmoves, 0, sizeof(int) * (size_t)np * ns, s));
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_v4_kernel<NB, 64, 64>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)gemm_v4_smem<NB, 64, 64>()));
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_v4_kernel<NB, 128, 128>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)gemm_v4_smem<NB, 128, 128>()));
    configured.done();
  }
  for (int p = 0, k0 = 0; k0 < n; ++p, k0 += NB)
  {
    const int jb = std::min(NB, n - k0), c0 = k0 + jb;
    int2 *mv = moves + (size_t)p * 2 * NB;
    int *nm = nmoves + p;
    if (panel_rpt<float, NB>(n - k0) == 0)
      throw std::runtime_error("batched LU: n too large for a single-cluster panel");
    launch_panel<float, NB>(a, n, k0, jb, ipiv, mv, nm, info, s, ns, bs);
    if (c0 < n && tma)
    {
      const int t = n - c0;
      prof_begin(KC_TRSM, s);
      f32u::mt2_kernel<NB, false>
          <<<dim3((t + f32u::MT_COLS - 1) / f32u::MT_COLS, 1, ns), 128, 0, s>>>(
              a, n, k0, jb, c0, n, mv, nm, 0, ut, 0, a, bs, n * ns);
      MPIRG_CUDA_CHECK(cudaGetLastError());
      prof_end(KC_TRSM, s);
      prof_begin(KC_GEMM, s);
      if ((long)((t + 127) / 128) * ((t + 127) / 128) * ns >= 2 * 148)
        f32u::gemm_tma_kernel<128>
            <<<dim3((t + 127) / 128, (t + 127) / 128, ns), 256, f32u::gemm_tma_smem<128>(), s>>>(
                mA128, mU128, a, n, k0, jb, 0, c0, n);
      else
        f32u::gemm_tma_kernel<64>
            <<<dim3((t + 63) / 64, (t + 63) / 64, ns), 256, f32u::gemm_tma_smem<64>(), s>>>(
                mA64, mU64, a, n, k0, jb, 0, c0, n);
      MPIRG_CUDA_CHECK(cudaGetLastError());
      prof_end(KC_GEMM, s);
    }
    else if (c0 < n)
    {
      prof_begin(KC_TRSM, s);
      lu_mt_kernel<float, NB><<<dim3((n - c0 + MT_COLS - 1) / MT_COLS, 1, ns), 128, 0, s>>>(
          a, n, k0, jb, c0, n, id, mv, nm, bs);
      MPIRG_CUDA_CHECK(cudaGetLastError());
      prof_end(KC_TRSM, s);
      prof_begin(KC_GEMM, s);
      const int t = n - c0;
      if ((long)((t + 127) / 128) * ((t + 127) / 128) * ns >= 2 * 148)
        lu_gemm_v4_kernel<NB, 128, 128>
            <<<dim3((t + 127) / 128, (t + 127) / 128, ns), 256, gemm_v4_smem<NB, 128, 128>(), s>>>(
                a, n, k0, jb, c0, n, id, bs.a);
      else
        lu_gemm_v4_kernel<NB, 64, 64>
            <<<dim3((t + 63) / 64, (t + 63) / 64, ns), 256, gemm_v4_smem<NB, 64, 64>(), s>>>(
                a, n, k0, jb, c0, n, id, bs.a);
      MPIRG_CUDA_CHECK(cudaGetLastError());
      prof_end(KC_GEMM, s);
    }
    prof_begin(KC_MOVES, s);
    // few CTAs per system: most batches (diagonally dominant systems) have no
    // row moves at all and every CTA only reads the count and leaves
    const int warps_needed = std::max(1, (k0 + 3) / 4);
    const int grid = std::max(1, std::min((warps_needed + 7) / 8, 8));
    lu_apply_moves_kernel<float, NB><<<dim3(grid, 1, ns), 256, 0, s>>>(a, n, 0, k0, id, mv, nm,
                                                                     perm, bs);
    MPIRG_CUDA_CHECK(cudaGetLastError());
    prof_end(KC_MOVES, s);
  }
}

bool lu_batched_supported(int prec, int n)
{
  return prec == B32 && n % 4 == 0 && n >= 64 && panel_rpt<float, 64>(n) > 0 &&
         gemm_v4_allowed();
}

int lu_choose_nb(int prec, int n, int requested)
{
  if (requested == 16 || requested == 32 || requested == 64)
    return requested;
  if (prec == B64)
    return n <= 4096 ? 64 : (n <= 8192 ? 32 : 16);
  // 64 at every n: panels taller than one cluster holds go through the
  // 8-column leaves (panel_tall), and the wider step halves the trailing
  // update's HBM passes (nb = 32 left the N = 16384 update memory-bound).
  return 64;
}

// ---- SM partition for the LU (green contexts) --------------------------------
// The panel is a thread-block cluster of up to 16 CTAs with ~180 KB of shared
// memory each; while the bulk trailing update keeps every SM busy, the block
// scheduler backfills freed SMs with update CTAs and the cluster (and every
// small kernel of the critical chain) waits for whole waves of the update.
// The binary32 LU therefore splits the device's SMs into a co-schedulable
// group of >= k SMs for the critical chain and the remainder for the bulk
// update, one green context each (driver API through the runtime's entry
// points); k = 16 (one 16-CTA panel cluster) unless MPIRG_LU_GREEN=k says
// otherwise, 0 = one shared pool. Measured on B200: N = 16384 LU 123 -> 100 ms.
struct GreenSplit
{
  bool ok = false;
  CUgreenCtx crit = nullptr, bulk = nullptr;
  unsigned crit_sms = 0, bulk_sms = 0;
};

template <typename F>
static F driver_fn(const char *name)
{
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return nullptr;
  return reinterpret_cast<F>(p);
}

static int green_request()
{
  static const int v = [] {
    const char *e = std::getenv("MPIRG_LU_GREEN");
    return e ? std::max(0, std::atoi(e)) : 16;
  }();
  return v;
}

static GreenSplit &green_split()
{
  // one split per device (mpirg_config.device / mpirg_dlu_create(device) let a
  // process use several)
  static GreenSplit gs[64];
  static bool tried_dev[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int cur = 0;
  cudaGetDevice(&cur);
  GreenSplit &g = gs[cur & 63];
  bool &tried = tried_dev[cur & 63];
  if (tried)
    return g;
  tried = true;
  // no SM partition under a profiler/sanitizer: the tools cannot follow
  // launches into green contexts (ncu died at the first LU launch)
  const int want = tool_attached() ? 0 : green_request();
  if (want <= 0)
    return g;
  using GetRes = CUresult (*)(CUdevice, CUdevResource *, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *,
                             unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc *, CUdevResource *, unsigned);
  using Create = CUresult (*)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned);
  auto get_res = driver_fn<GetRes>("cuDeviceGetDevResource");
  auto split = driver_fn<Split>("cuDevSmResourceSplitByCount");
  auto gen = driver_fn<GenDesc>("cuDevResourceGenerateDesc");
  auto create = driver_fn<Create>("cuGreenCtxCreate");
  if (!get_res || !split || !gen || !create)
  {
    std::fprintf(stderr, "mpirg: green contexts unavailable; LU uses one SM pool\n");
    return g;
  }
  int dev = 0;
  MPIRG_CUDA_CHECK(cudaGetDevice(&dev));
  CUdevResource all{}, grp{}, rest{};
  unsigned ng = 1;
  if (get_res((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(&grp, &ng, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE,
            (unsigned)want) != CUDA_SUCCESS ||
      ng < 1)
  {
    std::fprintf(stderr, "mpirg: SM split of %d failed; LU uses one SM pool\n", want);
    return g;
  }
  CUdevResourceDesc dc{}, db{};
  if (gen(&dc, &grp, 1) != CUDA_SUCCESS || gen(&db, &rest, 1) != CUDA_SUCCESS ||
      create(&g.crit, dc, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      create(&g.bulk, db, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
  {
    std::fprintf(stderr, "mpirg: green context creation failed; LU uses one SM pool\n");
    return g;
  }
  g.crit_sms = grp.sm.smCount;
  g.bulk_sms = rest.sm.smCount;
  g.ok = true;
  std::fprintf(stderr, "mpirg: LU SM partition: critical chain %u SMs, bulk update %u SMs\n",
               g.crit_sms, g.bulk_sms);
  return g;
}

static cudaStream_t green_stream(CUgreenCtx ctx, int prio)
{
  using SC = CUresult (*)(CUstream *, CUgreenCtx, unsigned, int);
  static auto sc = driver_fn<SC>("cuGreenCtxStreamCreate");
  CUstream st = nullptr;
  if (!sc || sc(&st, ctx, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS)
    throw std::runtime_error("cuGreenCtxStreamCreate failed");
  return reinterpret_cast<cudaStream_t>(st);
}

cudaStream_t lu_bulk_stream_create()
{
  int lo = 0, hi = 0;
  MPIRG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  GreenSplit &g = green_split();
  if (g.ok)
    return green_stream(g.bulk, lo);
  cudaStream_t st;
  MPIRG_CUDA_CHECK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, lo));
  return st;
}

// Workspaces made on this thread skip the SM partition (the concurrent
// systems of a batch each want the whole GPU for their panels, instead of
// queueing for the 16-SM critical group; cfg 5b 0.60 -> 0.50 s).
static thread_local bool t_partition = true;
void lu_partition_allowed(bool on) { t_partition = on; }

void lu_workspace_alloc(LuWorkspace &ws, int prec, int n, int nb)
{
  lu_workspace_free(ws);
  ws.n = n;
  ws.nb = lu_choose_nb(prec, n, nb);
  ws.npanels = std::max(1, (n + ws.nb - 1) / ws.nb);
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.moves, sizeof(int2) * (size_t)ws.npanels * 2 * ws.nb));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.nmoves, sizeof(int) * (size_t)ws.npanels));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.pp, sizeof(int) * (size_t)std::max(1, n)));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.smv, sizeof(int2) * 2 * (size_t)ws.nb));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.snm, sizeof(int) * (size_t)ws.nb));
  if (prec == B32 && ws.nb == 64 && n % 4 == 0)  // transposed U12 of two steps (lu_run_f32)
    MPIRG_CUDA_CHECK(cudaMalloc(&ws.ut, sizeof(float) * 2 * (size_t)ws.nb * n));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.zero, sizeof(int)));
  MPIRG_CUDA_CHECK(cudaMemset(ws.zero, 0, sizeof(int)));
  cudaStream_t side;
  // The side stream carries the bulk trailing update; give it the lowest
  // priority so the block scheduler hands freed SMs to the critical chain
  // (panel -> next-panel update) on the caller's stream first.
  int lo = 0, hi = 0;
  MPIRG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // small systems finish their panels faster than the partition pays for
  GreenSplit &g = green_split();
  if (g.ok && prec == B32 && t_partition && n >= 2048)
  {
    // one level above the lowest: the side stream's look-ahead updates come
    // before the late-column catch-up and the casts of a streamed refactor
    ws.side = green_stream(g.bulk, std::max(hi, lo - 1));
    ws.crit = green_stream(g.crit, hi);
  }
  else
  {
    MPIRG_CUDA_CHECK(
        cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, std::max(hi, lo - 1)));
    ws.side = side;
  }
  auto *ev = new cudaEvent_t[4 * (size_t)ws.npanels];
  for (int i = 0; i < 4 * ws.npanels; ++i)
    MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  ws.events = ev;
}

void lu_workspace_free(LuWorkspace &ws)
{
  if (ws.moves)
    lu_graph_forget(ws.moves);
  for (void *p : {(void *)ws.moves, (void *)ws.nmoves, (void *)ws.pp, (void *)ws.smv,
                  (void *)ws.snm, ws.ut, (void *)ws.zero})
    if (p)
      cudaFree(p);
  if (ws.events)
  {
    auto *ev = static_cast<cudaEvent_t *>(ws.events);
    for (int i = 0; i < 4 * ws.npanels; ++i)
      cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  if (ws.lsnap)
  {
    cudaFree(ws.lsnap);
    cudaFree(ws.utl);
    auto *st = static_cast<cudaStream_t *>(ws.lstreams);
    for (int i = 0; i < LuLate::MAXCH; ++i)
      cudaStreamDestroy(st[i]);
    delete[] st;
    auto *ev = static_cast<cudaEvent_t *>(ws.levents);
    for (int i = 0; i < ws.late_np + LuLate::MAXCH; ++i)
      cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  if (ws.side)
    cudaStreamDestroy(static_cast<cudaStream_t>(ws.side));
  if (ws.crit)
    cudaStreamDestroy(static_cast<cudaStream_t>(ws.crit));
  ws = LuWorkspace{};
}

template <typename T>
void lu_dispatch(int nb, T *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                 cudaStream_t s, const TcPlan *tc = nullptr)
{
  if constexpr (std::is_same<T, float>::value)
  {
    if (nb == 64 && f32_mode() && ws.ut && n % 4 == 0 &&
        reinterpret_cast<uintptr_t>(a) % 16 == 0)
    {
      lu_run_f32<64>(a, n, ipiv, perm, ws, info, s);
      return;
    }
  }
  if (nb == 64)
    lu_run<T, 64>(a, n, ipiv, perm, ws, info, s, tc);
  else if (nb == 32)
    lu_run<T, 32>(a, n, ipiv, perm, ws, info, s);
  else
    lu_run<T, 16>(a, n, ipiv, perm, ws, info, s);
}

void launch_lu(int prec, int lu_mode, void *a, int n, int *ipiv, int *perm, LuWorkspace &ws,
               DevInfo *info, cudaStream_t s)
{
  if (n <= 0)
    return;
  if (prec == B16 && lu_mode == 1 /* MPIRG_LU_TC */ && tc_update_supported(n, ws.nb))
  {
    TcPlan plan;
    tc_plan_make(plan, a, n);
    if (std::getenv("MPIRG_TC_SCHEDULE") && std::string(std::getenv("MPIRG_TC_SCHEDULE")) == "flat")
      lu_dispatch<h16>(ws.nb, static_cast<h16 *>(a), n, ipiv, perm, ws, info, s, &plan);  // K = 64
    else
      lu_run_tc(static_cast<h16 *>(a), n, ipiv, perm, ws, info, s, plan);
    return;
  }
  if (prec == B64)
    lu_dispatch<double>(ws.nb, static_cast<double *>(a), n, ipiv, perm, ws, info, s);
  else if (prec == B32)
    lu_dispatch<float>(ws.nb, static_cast<float *>(a), n, ipiv, perm, ws, info, s);
  else
    lu_dispatch<h16>(ws.nb, static_cast<h16 *>(a), n, ipiv, perm, ws, info, s);
}

bool lu_late_supported(int prec, int lu_mode, int n)
{
  return prec == B32 && lu_mode == 0 && f32_mode() && n % 64 == 0 && n >= 1024 &&
         n <= 32768;
}

void launch_lu_late(void *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                    cudaStream_t s, const LuLate &late)
{
  if (!lu_late_supported(B32, 0, n) || ws.nb != 64 || !ws.ut ||
      reinterpret_cast<uintptr_t>(a) % 16 != 0)
    throw std::runtime_error("launch_lu_late: unsupported configuration");
  for (int c = 1; c < late.nch; ++c)
    if (late.join[c] % 2 || late.join[c] * 64 + 128 > late.lo[c] || late.lo[c] % 64)
      throw std::runtime_error("launch_lu_late: bad chunk plan");
  lu_run_f32_body<64>(static_cast<float *>(a), n, ipiv, perm, ws, info, s, &late);
}

void launch_perm_from_ipiv(const int *ipiv, int n, int *perm, cudaStream_t s)
{
  perm_from_ipiv_kernel<<<1, 32, 0, s>>>(ipiv, n, perm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// ---- distributed (per-rank) driver -----------------------------------------
void dlu_alloc(DluPlan &d, int prec, int n, int nb, int G, int r, int block_cols)
{
  d.prec = prec;
  d.n = n;
  d.G = G;
  d.r = r;
  int sh = 0;
  while ((1 << sh) < block_cols)
    ++sh;
  d.sh = sh;
  lu_workspace_alloc(d.ws, prec, n, nb);
}

void dlu_free(DluPlan &d)
{
  lu_workspace_free(d.ws);
  delete static_cast<DluF32State *>(d.f32);
  d.f32 = nullptr;
  if (d.cevents)
  {
    auto *ce = static_cast<cudaEvent_t *>(d.cevents);
    for (int i = 0; i < 3; ++i)
      cudaEventDestroy(ce[i]);
    delete[] ce;
    d.cevents = nullptr;
  }
  if (d.comm)
    cudaStreamDestroy(static_cast<cudaStream_t>(d.comm));
  d.comm = nullptr;
}

void dlu_begin(DluPlan &d, int *perm, cudaStream_t s)
{
  if (perm)
  {
    iota_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(perm, d.n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(d.ws.nmoves, 0, sizeof(int) * d.ws.npanels, s));
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(d.ws.events);
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[0], s));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(static_cast<cudaStream_t>(d.ws.side), ev[0], 0));
}

template <typename F>
static void dlu_dispatch(const DluPlan &d, F &&f)
{
  const int nb = d.ws.nb;
  auto go = [&](auto tag) {
    using T = typename decltype(tag)::type;
    if (nb == 64)
      f.template operator()<T, 64>();
    else if (nb == 32)
      f.template operator()<T, 32>();
    else
      f.template operator()<T, 16>();
  };
  if (d.prec == B64)
    go(std::type_identity<double>{});
  else if (d.prec == B32)
    go(std::type_identity<float>{});
  else
    go(std::type_identity<h16>{});
}

void dlu_panel(DluPlan &d, void *a, int p, int *ipiv, DevInfo *info, cudaStream_t s)
{
  dlu_dispatch(d, [&]<typename T, int NB>() {
    dlu_panel_t<T, NB>(d, static_cast<T *>(a), p, ipiv, info, s);
  });
}

void dlu_update(DluPlan &d, void *a, int p, int part, int *perm, cudaStream_t s)
{
  dlu_dispatch(d, [&]<typename T, int NB>() {
    dlu_update_t<T, NB>(d, static_cast<T *>(a), p, part, perm, s);
  });
}

void dlu_end(DluPlan &d, cudaStream_t s)
{
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(d.ws.events);
  const int np = d.ws.npanels;
  // every REST event that was recorded (part 2 calls) is before the last one
  MPIRG_CUDA_CHECK(cudaEventRecord(ev[np + np - 1], static_cast<cudaStream_t>(d.ws.side)));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[np + np - 1], 0));
}

bool dlu_f32_supported(const DluPlan &d, const void *a)
{
  return d.prec == B32 && d.ws.nb == 64 && f32_mode() && d.ws.ut && d.n % 4 == 0 &&
         reinterpret_cast<uintptr_t>(a) % 16 == 0;
}

void dlu_f32_begin(DluPlan &d, void *a, int *perm, cudaStream_t caller)
{
  LuWorkspace &ws = d.ws;
  if (!d.f32)
    d.f32 = new DluF32State;
  auto &st = *static_cast<DluF32State *>(d.f32);
  st.a = static_cast<float *>(a);
  st.prev_deferred = false;
  st.s = ws.crit ? static_cast<cudaStream_t>(ws.crit) : caller;
  f32_plan_make(st.P, st.a, d.n, static_cast<float *>(ws.ut), 2 * ws.nb);
  if (!d.comm)
  {
    int lo = 0, hi = 0;
    MPIRG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    cudaStream_t c;
    MPIRG_CUDA_CHECK(cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, hi));
    d.comm = c;
    auto *ce = new cudaEvent_t[3];
    for (int i = 0; i < 3; ++i)
      MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&ce[i], cudaEventDisableTiming));
    d.cevents = ce;
  }
  cudaEvent_t *ce = static_cast<cudaEvent_t *>(d.cevents);
  cudaStream_t comm = static_cast<cudaStream_t>(d.comm), side = static_cast<cudaStream_t>(ws.side);
  // every stream starts after the caller's earlier work (the cast)
  if (perm)
  {
    iota_kernel<<<(d.n + 255) / 256, 256, 0, caller>>>(perm, d.n);
    MPIRG_CUDA_CHECK(cudaGetLastError());
  }
  MPIRG_CUDA_CHECK(cudaMemsetAsync(ws.nmoves, 0, sizeof(int) * ws.npanels, caller));
  MPIRG_CUDA_CHECK(cudaEventRecord(ce[2], caller));
  for (cudaStream_t t : {st.s, side, comm})
    if (t != caller)
      MPIRG_CUDA_CHECK(cudaStreamWaitEvent(t, ce[2], 0));
  // both message slots start free
  MPIRG_CUDA_CHECK(cudaEventRecord(ce[0], comm));
  MPIRG_CUDA_CHECK(cudaEventRecord(ce[1], comm));
}

cudaStream_t dlu_f32_crit(DluPlan &d) { return static_cast<DluF32State *>(d.f32)->s; }
cudaStream_t dlu_f32_comm(DluPlan &d) { return static_cast<cudaStream_t>(d.comm); }

void dlu_f32_panel_ready(DluPlan &d, int p, cudaStream_t s)
{
  MPIRG_CUDA_CHECK(cudaEventRecord(static_cast<cudaEvent_t *>(d.ws.events)[p], s));
}

void dlu_f32_step(DluPlan &d, int p, int *perm, bool own_panel)
{
  dlu_f32_step_t<64>(d, p, perm, own_panel);
}

void dlu_f32_end(DluPlan &d, cudaStream_t caller)
{
  auto &st = *static_cast<DluF32State *>(d.f32);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(d.ws.events);
  cudaEvent_t *ce = static_cast<cudaEvent_t *>(d.cevents);
  const int np = d.ws.npanels;
  // the side stream's last record (evR of the last step) covers every step's
  // bulk work; the critical and communication streams join through ce[2]
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(caller, ev[2 * np + np - 1], 0));
  if (st.s != caller)
  {
    MPIRG_CUDA_CHECK(cudaEventRecord(ev[np + np - 1], st.s));
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(caller, ev[np + np - 1], 0));
  }
  MPIRG_CUDA_CHECK(cudaEventRecord(ce[2], static_cast<cudaStream_t>(d.comm)));
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(caller, ce[2], 0));
}

void dlu_merge_singular(int *dst, const int *src, cudaStream_t s)
{
  min_into_kernel<<<1, 1, 0, s>>>(dst, src);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace mpirg

// ---- diagnostics: the binary32 trailing update alone ------------------------
extern "C" int mpirg_ubench_gemm_f32(int n, int K, int tile, int reps, double *tflops,
                                     double *ms_out)
{
  using namespace mpirg;
  if (n <= 0 || K <= 0 || K > 128 || n % 4 || reps <= 0 || K >= n)
    return MPIRG_ERR_INVALID_SIZE;
  try
  {
    float *a = nullptr, *ut = nullptr;
    MPIRG_CUDA_CHECK(cudaMalloc(&a, sizeof(float) * (size_t)n * n));
    MPIRG_CUDA_CHECK(cudaMalloc(&ut, sizeof(float) * 128 * (size_t)n));
    MPIRG_CUDA_CHECK(cudaMemset(a, 0, sizeof(float) * (size_t)n * n));
    MPIRG_CUDA_CHECK(cudaMemset(ut, 0, sizeof(float) * 128 * (size_t)n));
    F32Plan P;
    f32_plan_make(P, a, n, ut, 128);
    cudaStream_t s;
    MPIRG_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    MPIRG_CUDA_CHECK(cudaEventCreate(&e0));
    MPIRG_CUDA_CHECK(cudaEventCreate(&e1));
    auto run = [&] {
      if (tile == 128)
        f32_gemm_t<128>(P.a128, P.u128, P, 0, K, 0, K, n, s);
      else if (tile == 64)
        f32_gemm_t<64>(P.a64, P.u64, P, 0, K, 0, K, n, s);
      else
        f32_gemm(P, 0, K, 0, K, n, s);
    };
    run();
    MPIRG_CUDA_CHECK(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r)
      run();
    MPIRG_CUDA_CHECK(cudaEventRecord(e1, s));
    MPIRG_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    MPIRG_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    const double m = (double)(n - K);
    *ms_out = ms / reps;
    *tflops = 2.0 * m * m * K / (*ms_out * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaFree(a);
    cudaFree(ut);
    return MPIRG_OK;
  }
  catch (const std::exception &)
  {
    return MPIRG_ERR_CUDA;
  }
}
