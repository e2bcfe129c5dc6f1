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

#include "common.cuh"
#include "kernels.cuh"
#include "lu_panel.cuh"
#include "lu_panel5.cuh"

namespace cg = cooperative_groups;

namespace mpirg
{

namespace
{

// Gather-apply the panel's row moves (new[dst] = old[src]) to the columns
// [cb, ce) -- one warp per column -- and to perm (block 0, warp 0).
template <typename T, int NB>
__global__ void __launch_bounds__(256) lu_apply_moves_kernel(T *__restrict__ A, int n, int cb,
                                                             int ce,
                                                             const int2 *__restrict__ moves,
                                                             const int *__restrict__ nmoves,
                                                             int *__restrict__ perm)
{
  constexpr int PER = (2 * NB + 31) / 32;
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
        const T *cp = A + (size_t)(cb + c0 + u) * n;
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
        T *cp = A + (size_t)(cb + c0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            cp[mv[q].x] = v[u][q];
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
                                                    int cb, int ce,
                                                    const int2 *__restrict__ moves,
                                                    const int *__restrict__ nmoves)
{
  constexpr int PER = (2 * NB + 31) / 32;
  constexpr int RL = (NB + 31) / 32;  // panel rows per lane
  __shared__ T L[NB][NB + 1];
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
        const T *cp = A + (size_t)(col0 + u) * n;
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
        T *cp = A + (size_t)(col0 + u) * n;
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
      x[u][h] = (col0 + u < ce && i < jb) ? A[(size_t)(col0 + u) * n + k0 + i] : T{};
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
        A[(size_t)(col0 + u) * n + k0 + i] = x[u][h];
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
                                                      int cb, int ce)
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
      tb[u] = (kb < jb && col < ce) ? to_c(A[(size_t)col * n + k0 + kb]) : C(0);
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
      acc[i][j] = (row < n && col < ce) ? to_c(A[(size_t)col * n + row]) : C(0);
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
        from_c(A[(size_t)col * n + row], acc[i][j]);
    }
  }
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
template <typename T, int NB, int RPT>
void configure_panel()
{
  static bool done = false;
  if (done)
    return;
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(panel2::lu_panel2_kernel<T, NB, RPT>,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(panel2::lu_panel2_kernel<T, NB, RPT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)panel2::panel_dyn_smem<T, NB, RPT>()));
  done = true;
}

template <typename T, int NB>
void configure_gemm()
{
  static bool done = false;
  if (done)
    return;
  MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_kernel<T, NB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)gemm_smem_bytes<T, NB>()));
  done = true;
}

template <typename T, int NB, int RPT>
void launch_panel_rpt(int cs, T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm,
                      DevInfo *info, cudaStream_t s)
{
  configure_panel<T, NB, RPT>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(panel2::NT);
  cfg.dynamicSmemBytes = panel2::panel_dyn_smem<T, NB, RPT>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel2::lu_panel2_kernel<T, NB, RPT>, a, n, k0, jb,
                                      ipiv, mv, nm, info));
}

// Largest rows-per-thread the register file allows for (T, NB).
template <typename T, int NB>
constexpr int max_rpt()
{
  return panel2::panel_dyn_smem<T, NB, 4>() <= 180 * 1024
             ? 4
             : (panel2::panel_dyn_smem<T, NB, 2>() <= 180 * 1024 ? 2 : 1);
}

template <typename T, int NB, int RPL, int IB>
void launch_panel5(int cs, T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm,
                   DevInfo *info, cudaStream_t s)
{
  constexpr size_t smem = panel5::panel5_dyn_smem<T, NB, RPL, IB>();
  static bool done = false;
  if (!done)
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(panel5::lu_panel5_kernel<T, NB, RPL, IB>,
                                          cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(panel5::lu_panel5_kernel<T, NB, RPL, IB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(panel5::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MPIRG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel5::lu_panel5_kernel<T, NB, RPL, IB>, a, n, k0,
                                      jb, ipiv, mv, nm, info));
}

// Block width of the critical warp's register tile for (T, rows per lane).
template <typename T, int RPL>
constexpr int ib_of()
{
  // RPL * IB * words(T) <= 128 registers
  constexpr int words = (int)((sizeof(T) + 3) / 4);
  return (128 / (RPL * words)) >= 8 ? 8 : ((128 / (RPL * words)) >= 4 ? 4 : 2);
}

template <typename T, int NB, int RPL>
constexpr bool panel5_ok()
{
  constexpr int IB = ib_of<T, RPL>();
  return NB % IB == 0 && (IB * sizeof(T)) % 16 == 0 &&
         panel5::panel5_dyn_smem<T, NB, RPL, IB>() <= 200 * 1024;
}

// Experimental critical-warp panel (lu_panel5.cuh), opt-in via MPIRG_PANEL=5.
template <typename T, int NB>
bool launch_panel5_dispatch(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm,
                            DevInfo *info, cudaStream_t s, int max_cs)
{
  const int m = n - k0;
  int rpl = 4;
  while (rpl * 32 * max_cs < m && rpl < 32)
    rpl *= 2;
  const int cs = std::max(1, (m + rpl * 32 - 1) / (rpl * 32));
  if (cs > panel5::MAXCS)
    return false;
  bool launched = false;
  if (rpl == 4)
  {
    if constexpr (panel5_ok<T, NB, 4>())
    {
      launch_panel5<T, NB, 4, ib_of<T, 4>()>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
      launched = true;
    }
  }
  else if (rpl == 8)
  {
    if constexpr (panel5_ok<T, NB, 8>())
    {
      launch_panel5<T, NB, 8, ib_of<T, 8>()>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
      launched = true;
    }
  }
  else if (rpl == 16)
  {
    if constexpr (panel5_ok<T, NB, 16>())
    {
      launch_panel5<T, NB, 16, ib_of<T, 16>()>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
      launched = true;
    }
  }
  else
  {
    if constexpr (panel5_ok<T, NB, 32>())
    {
      launch_panel5<T, NB, 32, ib_of<T, 32>()>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
      launched = true;
    }
  }
  return launched;
}

template <typename T, int NB>
void launch_panel(T *a, int n, int k0, int jb, int *ipiv, int2 *mv, int *nm, DevInfo *info,
                  cudaStream_t s)
{
  const int m = n - k0;
  const int per_cta = panel2::NT;
  static const int max_cs = [] {
    const char *e = std::getenv("MPIRG_PANEL_MAXCS");
    const int v = e ? std::atoi(e) : panel2::MAXCS;
    return std::max(1, std::min(panel2::MAXCS, v));
  }();
  int rpt = 1;
  while (rpt * per_cta * max_cs < m)
    rpt *= 2;
  if (rpt > max_rpt<T, NB>())
    throw std::runtime_error("LU panel: n too large for a single-cluster panel at this nb");
  const int cs = std::max(1, (m + rpt * per_cta - 1) / (rpt * per_cta));
  static const bool p5 = [] {
    const char *e = std::getenv("MPIRG_PANEL");
    return e && std::atoi(e) == 5;
  }();
  prof_begin(KC_PANEL, s);
  if (p5 && launch_panel5_dispatch<T, NB>(a, n, k0, jb, ipiv, mv, nm, info, s, max_cs))
    ;
  else if (rpt == 1)
    launch_panel_rpt<T, NB, 1>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
  else if (rpt == 2)
  {
    if constexpr (max_rpt<T, NB>() >= 2)
      launch_panel_rpt<T, NB, 2>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
  }
  else
  {
    if constexpr (max_rpt<T, NB>() >= 4)
      launch_panel_rpt<T, NB, 4>(cs, a, n, k0, jb, ipiv, mv, nm, info, s);
  }
  prof_end(KC_PANEL, s);
}

template <typename T, int NB>
void launch_mt(T *a, int n, int k0, int jb, int cb, int ce, const int2 *mv, const int *nm,
               cudaStream_t s)
{
  if (ce <= cb)
    return;
  prof_begin(KC_TRSM, s);
  lu_mt_kernel<T, NB><<<(ce - cb + MT_COLS - 1) / MT_COLS, 128, 0, s>>>(a, n, k0, jb, cb, ce, mv,
                                                                      nm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_TRSM, s);
}

template <typename T, int NB>
void launch_gemm(T *a, int n, int k0, int jb, int cb, int ce, cudaStream_t s)
{
  const int c0 = k0 + jb;
  if (ce <= cb || c0 >= n)
    return;
  configure_gemm<T, NB>();
  prof_begin(KC_GEMM, s);
  const dim3 grid((n - c0 + GB - 1) / GB, (ce - cb + GB - 1) / GB);
  lu_gemm_kernel<T, NB><<<grid, 256, gemm_smem_bytes<T, NB>(), s>>>(a, n, k0, jb, cb, ce);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_GEMM, s);
}

template <typename T, int NB>
void launch_moves(T *a, int n, int cb, int ce, const int2 *mv, const int *nm, int *perm,
                  cudaStream_t s)
{
  const int ncols = ce - cb;
  if (ncols <= 0 && !perm)
    return;
  prof_begin(KC_MOVES, s);
  const int warps_needed = std::max(1, (ncols + 3) / 4);
  const int grid = std::max(1, std::min((warps_needed + 7) / 8, 148 * 8));
  lu_apply_moves_kernel<T, NB><<<grid, 256, 0, s>>>(a, n, cb, std::max(cb, ce), mv, nm, perm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_MOVES, s);
}

template <typename T, int NB>
void lu_run(T *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info, cudaStream_t s)
{
  cudaStream_t side = static_cast<cudaStream_t>(ws.side);
  cudaEvent_t *ev = static_cast<cudaEvent_t *>(ws.events);  // [3][npanels]: P, N, R
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
    cudaEvent_t evP = ev[p], evN = ev[np + p], evR = ev[2 * np + p];
    // main: the critical chain
    launch_panel<T, NB>(a, n, k0, jb, ipiv, mv, nm, info, s);
    MPIRG_CUDA_CHECK(cudaEventRecord(evP, s));
    const int cnext = std::min(n, c0 + NB);
    if (c0 < n)
    {
      if (p > 0)
        MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2 * np + p - 1], 0));
      launch_mt<T, NB>(a, n, k0, jb, c0, cnext, mv, nm, s);
      launch_gemm<T, NB>(a, n, k0, jb, c0, cnext, s);
    }
    MPIRG_CUDA_CHECK(cudaEventRecord(evN, s));
    // side: the rest of this step's update + the left-column moves
    MPIRG_CUDA_CHECK(cudaStreamWaitEvent(side, evP, 0));
    if (cnext < n)
    {
      launch_mt<T, NB>(a, n, k0, jb, cnext, n, mv, nm, side);
      launch_gemm<T, NB>(a, n, k0, jb, cnext, n, side);
    }
    launch_moves<T, NB>(a, n, 0, k0, mv, nm, perm, side);
    MPIRG_CUDA_CHECK(cudaEventRecord(evR, side));
  }
  MPIRG_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2 * np + np - 1], 0));
}

}  // namespace

int lu_choose_nb(int prec, int n, int requested)
{
  if (requested == 16 || requested == 32 || requested == 64)
    return requested;
  if (prec == B64)
    return n <= 4096 ? 64 : (n <= 8192 ? 32 : 16);
  return n <= 8192 ? 64 : 32;
}

void lu_workspace_alloc(LuWorkspace &ws, int prec, int n, int nb)
{
  lu_workspace_free(ws);
  ws.n = n;
  ws.nb = lu_choose_nb(prec, n, nb);
  ws.npanels = std::max(1, (n + ws.nb - 1) / ws.nb);
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.moves, sizeof(int2) * (size_t)ws.npanels * 2 * ws.nb));
  MPIRG_CUDA_CHECK(cudaMalloc(&ws.nmoves, sizeof(int) * (size_t)ws.npanels));
  cudaStream_t side;
  MPIRG_CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  ws.side = side;
  auto *ev = new cudaEvent_t[3 * (size_t)ws.npanels];
  for (int i = 0; i < 3 * ws.npanels; ++i)
    MPIRG_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  ws.events = ev;
}

void lu_workspace_free(LuWorkspace &ws)
{
  if (ws.moves)
    cudaFree(ws.moves);
  if (ws.nmoves)
    cudaFree(ws.nmoves);
  if (ws.events)
  {
    auto *ev = static_cast<cudaEvent_t *>(ws.events);
    for (int i = 0; i < 3 * ws.npanels; ++i)
      cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  if (ws.side)
    cudaStreamDestroy(static_cast<cudaStream_t>(ws.side));
  ws = LuWorkspace{};
}

template <typename T>
void lu_dispatch(int nb, T *a, int n, int *ipiv, int *perm, LuWorkspace &ws, DevInfo *info,
                 cudaStream_t s)
{
  if (nb == 64)
    lu_run<T, 64>(a, n, ipiv, perm, ws, info, s);
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
  (void)lu_mode;
  if (prec == B64)
    lu_dispatch<double>(ws.nb, static_cast<double *>(a), n, ipiv, perm, ws, info, s);
  else if (prec == B32)
    lu_dispatch<float>(ws.nb, static_cast<float *>(a), n, ipiv, perm, ws, info, s);
  else
    lu_dispatch<h16>(ws.nb, static_cast<h16 *>(a), n, ipiv, perm, ws, info, s);
}

void launch_perm_from_ipiv(const int *ipiv, int n, int *perm, cudaStream_t s)
{
  perm_from_ipiv_kernel<<<1, 32, 0, s>>>(ipiv, n, perm);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace mpirg
