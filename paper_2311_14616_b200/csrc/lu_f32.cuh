// K4/K5 for binary32 factors on one GPU: U12 solve with a transposed copy of
// U12, and a TMA-fed trailing update that can take two panel steps at once.
//
// Why two steps at once keeps the reference's bits (dense_lu.hpp:91-107):
// each element a_ij takes one FMA per elimination step k, in ascending k.
// Deferring step p's update of the far columns to step p+1 and applying
// steps p and p+1 back to back (k = k0(p) .. k0(p+1)+nb-1, ascending) is the
// same per-element sequence. Three things make the deferral exact:
//   * the row moves of step p+1 are applied to the far columns AND to panel
//     p's L columns before the deferred update, so C and L21(p) rows stay
//     paired (a row interchange swaps whole rows, dense_lu.hpp:79-85);
//   * the panel rows [k0(p+1), k0(p+1)+nb) of the far columns receive step
//     p's update (the "pending" update, same FMA order) before the U12 solve
//     of step p+1 reads them;
//   * the update of rows below then runs K = 2nb in ascending k.
// Halving the number of passes over the trailing matrix halves its HBM
// traffic (8 bytes per element per pass against 2K flops), which bounds the
// K = 64 update at large n.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace mpirg
{
namespace f32u
{

constexpr int MT_COLS = 32;  // columns per CTA of the U12 solve (4 warps x 8)

// Row moves + (PEND: step kp's deferred update of the panel rows) + U12 =
// L11^{-1} A12 for the columns [cb, ce); U12 is also written transposed into
// ut[(ut_row + kk) * n + col] (row-major, contiguous along columns) so the
// trailing update can stage it with TMA. The L factors are read from Ls (the
// matrix itself, or the snapshot of the panel taken for late columns).
// CPW columns per warp (4 CPW per CTA): 8 for throughput (the bulk of the
// columns), 2 for the critical chain's next-panel block, whose 2 x NB
// sequential steps (shuffle + FMA each) then cost their latency instead of
// the issue time of eight interleaved columns.
template <int NB, bool PEND, int CPW = 8>
__global__ void __launch_bounds__(128) mt2_kernel(float *__restrict__ A, int n, int k0, int jb,
                                                  int cb, int ce,
                                                  const int2 *__restrict__ moves,
                                                  const int *__restrict__ nmoves, int kp,
                                                  float *__restrict__ ut, int ut_row,
                                                  const float *__restrict__ Ls,
                                                  BatchStride bs = BatchStride{}, int ut_ld = 0)
{
  constexpr int PER = (2 * NB + 31) / 32;
  constexpr int RL = (NB + 31) / 32;  // panel rows per lane
  __shared__ float L[NB][NB + 1];
  if constexpr (CPW < 8)
    pdl_trigger();  // the chain's update may become resident while this solve runs
  pdl_wait();
  // batched launches (config 5b): system blockIdx.z; its U12 copy occupies
  // columns [z n, z n + n) of a ut with row pitch ut_ld = n * (systems)
  A += (size_t)blockIdx.z * bs.a;
  Ls += (size_t)blockIdx.z * bs.a;
  moves += (size_t)blockIdx.z * bs.moves;
  nmoves += (size_t)blockIdx.z * bs.nm;
  ut += (size_t)blockIdx.z * n;
  const size_t utp = ut_ld ? (size_t)ut_ld : (size_t)n;
  __shared__ float Lp[PEND ? NB : 1][NB + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int MTC = 4 * CPW;  // columns per CTA
  const int col0 = cb + blockIdx.x * MTC + warp * CPW;
  // Every load that does not depend on the row moves is issued up front (the
  // L factors, the move count, this warp's panel rows and, for PEND, step
  // kp's U rows): on the LU's critical chain each dependent round trip costs
  // about a microsecond. The panel rows are reloaded if rows moved.
  float x[CPW][RL];
  float uv[CPW][PEND ? RL : 1];
  int nm;
  {
    constexpr int PT = (NB * NB + 127) / 128;
    float tmp[PT], tp[PEND ? PT : 1];
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = threadIdx.x + u * 128;
      const int kk = idx / NB, i = idx % NB;
      tmp[u] = (kk < jb && i < jb) ? Ls[(size_t)(k0 + kk) * n + k0 + i] : 0.f;
      if constexpr (PEND)
        tp[u] = (kk < NB && i < jb) ? Ls[(size_t)(kp + kk) * n + k0 + i] : 0.f;
    }
    nm = *nmoves;
#pragma unroll
    for (int u = 0; u < CPW; ++u)
#pragma unroll
      for (int h = 0; h < RL; ++h)
      {
        const int i = lane + 32 * h;
        x[u][h] = (col0 + u < ce && i < jb) ? A[(size_t)(col0 + u) * n + k0 + i] : 0.f;
        if constexpr (PEND)
          uv[u][h] = (col0 + u < ce) ? A[(size_t)(col0 + u) * n + kp + lane + 32 * h] : 0.f;
      }
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int idx = threadIdx.x + u * 128;
      const int kk = idx / NB, i = idx % NB;
      if (kk < NB)
      {
        L[i][kk] = tmp[u];
        if constexpr (PEND)
          Lp[i][kk] = tp[u];
      }
    }
  }
  if (nm > 0)
  {
    int2 mv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
    {
      const int e = lane + 32 * q;
      mv[q] = e < nm ? moves[e] : make_int2(-1, -1);
    }
    float v[CPW][PER];
#pragma unroll
    for (int u = 0; u < CPW; ++u)
      if (col0 + u < ce)
      {
        const float *cp = A + (size_t)(col0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            v[u][q] = cp[mv[q].y];
      }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < CPW; ++u)
      if (col0 + u < ce)
      {
        float *cp = A + (size_t)(col0 + u) * n;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (mv[q].x >= 0)
            cp[mv[q].x] = v[u][q];
      }
    __syncwarp();
    // the panel rows after the moves (this warp's columns only)
#pragma unroll
    for (int u = 0; u < CPW; ++u)
#pragma unroll
      for (int h = 0; h < RL; ++h)
      {
        const int i = lane + 32 * h;
        x[u][h] = (col0 + u < ce && i < jb) ? A[(size_t)(col0 + u) * n + k0 + i] : 0.f;
      }
  }
  __syncthreads();
  if constexpr (PEND)
  {
    // step kp's update of the panel rows: x_i -= L(kp)[i][kk] * U(kp)[kk], kk ascending
#pragma unroll 4
    for (int kk = 0; kk < NB; ++kk)
    {
      const int hk = kk >> 5, lk = kk & 31;
      float lv[RL];
#pragma unroll
      for (int h = 0; h < RL; ++h)
        lv[h] = Lp[lane + 32 * h][kk];
#pragma unroll
      for (int u = 0; u < CPW; ++u)
      {
        float src = uv[u][0];
#pragma unroll
        for (int h = 1; h < RL; ++h)
          if (hk == h)
            src = uv[u][h];
        const float uk = __shfl_sync(0xffffffffu, src, lk);
#pragma unroll
        for (int h = 0; h < RL; ++h)
          x[u][h] = __fmaf_rn(-lv[h], uk, x[u][h]);
      }
    }
  }
#pragma unroll 4
  for (int kk = 0; kk < jb; ++kk)
  {
    const int hk = kk >> 5, lk = kk & 31;
    float lv[RL];
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      lv[h] = (i > kk && i < jb) ? L[i][kk] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < CPW; ++u)
    {
      float src = x[u][0];
#pragma unroll
      for (int h = 1; h < RL; ++h)
        if (hk == h)
          src = x[u][h];
      const float xk = __shfl_sync(0xffffffffu, src, lk);
#pragma unroll
      for (int h = 0; h < RL; ++h)
      {
        const int i = lane + 32 * h;
        if (i > kk && i < jb)
          x[u][h] = __fmaf_rn(-lv[h], xk, x[u][h]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
    {
      const int i = lane + 32 * h;
      if (col0 + u < ce && i < jb)
        A[(size_t)(col0 + u) * n + k0 + i] = x[u][h];
    }
  // transposed copy through shared memory: 128-byte row segments of ut
  __syncthreads();
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int h = 0; h < RL; ++h)
      L[lane + 32 * h][warp * CPW + u] = x[u][h];
  __syncthreads();
  const int cbase = cb + blockIdx.x * MTC;
  for (int idx = threadIdx.x; idx < jb * MTC; idx += 128)
  {
    const int kk = idx / MTC, c = idx % MTC;
    if (cbase + c < ce)
      ut[(size_t)(ut_row + kk) * utp + cbase + c] = L[kk][c];
  }
}

// Trailing update A[r, c] -= sum_k L[r, k] U[k, c] for rows [k0 + K, n) and
// columns [cb, ce), k = k0 .. k0 + K - 1 ascending (K <= 128: one or two
// panel steps). BM x BM tile per CTA of 256 threads, (BM/16)^2 accumulators
// per thread started from A and taking one FMA per k. L21 chunks (BM rows x
// 32 k) come from A and U12 chunks (32 k x BM columns) from the transposed
// copy ut, both by TMA into a 3-stage ring of shared-memory buffers.
constexpr int GKC = 32;  // k per chunk
constexpr int GST = 3;   // ring stages
template <int BM>
constexpr size_t gemm_tma_smem()
{
  return 128 + (size_t)GST * 2 * BM * GKC * sizeof(float);
}

template <int BM>
__global__ void __launch_bounds__(256, BM == 128 ? 2 : 3)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapU, float *__restrict__ A, int n,
                    int k0, int K, int ut_row, int cb, int ce)
{
  constexpr int TM = BM / 16;
  constexpr uint32_t CHUNK = BM * GKC * sizeof(float);
  extern __shared__ unsigned char gsm_raw[];
  __shared__ __align__(8) uint64_t full[GST];
  pdl_wait();
  if constexpr (BM == 64)
    pdl_trigger();
  float *base = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(gsm_raw) + 127) &
                                          ~uintptr_t(127));
  float *As = base;                   // [GST][GKC][BM]
  float *Bs = base + GST * BM * GKC;  // [GST][GKC][BM]
  const int c0 = k0 + K;
  const int r0 = c0 + blockIdx.x * BM;
  const int cc0 = cb + blockIdx.y * BM;
  // batched launches (config 5b): the systems are stored back to back, so the
  // batch is one n x (n systems) matrix to the tensor maps; system blockIdx.z
  // is a column offset of z n in both maps
  const int zc = blockIdx.z * n;
  A += (size_t)blockIdx.z * n * n;
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int nch = (K + GKC - 1) / GKC;
  if (t == 0)
  {
#pragma unroll
    for (int s = 0; s < GST; ++s)
      tc::mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int s = 0; s < GST && s < nch; ++s)
    {
      tc::mbar_expect_tx(&full[s], 2 * CHUNK);
      tc::tma_load_2d(As + s * BM * GKC, &mapA, &full[s], r0, zc + k0 + s * GKC);
      tc::tma_load_2d(Bs + s * BM * GKC, &mapU, &full[s], zc + cc0, ut_row + s * GKC);
    }

  float acc[TM][TM];
#pragma unroll
  for (int gj = 0; gj < TM / 4; ++gj)
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
          v = *reinterpret_cast<const float4 *>(A + (size_t)col * n + row);
        acc[gi * 4 + 0][gj * 4 + j] = v.x;
        acc[gi * 4 + 1][gj * 4 + j] = v.y;
        acc[gi * 4 + 2][gj * 4 + j] = v.z;
        acc[gi * 4 + 3][gj * 4 + j] = v.w;
      }
    }

  auto step = [&](const float *ar, const float *br) {
    float a[TM], b[TM];
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
    for (int gj = 0; gj < TM / 4; ++gj)
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
      for (int j = 0; j < TM; ++j)
        acc[i][j] = __fmaf_rn(-a[i], b[j], acc[i][j]);
  };

  for (int ch = 0; ch < nch; ++ch)
  {
    const int st = ch % GST;
    tc::mbar_wait(&full[st], (ch / GST) & 1);
    const float *as = As + st * BM * GKC;
    const float *bs = Bs + st * BM * GKC;
    const int kc = min(GKC, K - ch * GKC);
    if (kc == GKC)
    {
#pragma unroll 8
      for (int kk = 0; kk < GKC; ++kk)
        step(as + kk * BM, bs + kk * BM);
    }
    else
    {
#pragma unroll 1
      for (int kk = 0; kk < kc; ++kk)
        step(as + kk * BM, bs + kk * BM);
    }
    if (ch + GST < nch)
    {
      __syncthreads();  // every warp is done with stage st
      if (t == 0)
      {
        const int nx = ch + GST;
        tc::mbar_expect_tx(&full[st], 2 * CHUNK);
        tc::tma_load_2d(As + st * BM * GKC, &mapA, &full[st], r0, zc + k0 + nx * GKC);
        tc::tma_load_2d(Bs + st * BM * GKC, &mapU, &full[st], zc + cc0, ut_row + nx * GKC);
      }
    }
  }

#pragma unroll
  for (int gj = 0; gj < TM / 4; ++gj)
#pragma unroll
    for (int j = 0; j < 4; ++j)
    {
      const int col = cc0 + gj * 64 + ty * 4 + j;
#pragma unroll
      for (int gi = 0; gi < TM / 4; ++gi)
      {
        const int row = r0 + gi * 64 + tx * 4;
        if (row < n && col < ce)
          *reinterpret_cast<float4 *>(A + (size_t)col * n + row) =
              make_float4(acc[gi * 4 + 0][gj * 4 + j], acc[gi * 4 + 1][gj * 4 + j],
                          acc[gi * 4 + 2][gj * 4 + j], acc[gi * 4 + 3][gj * 4 + j]);
      }
    }
}

// Critical-chain step for the next panel's columns, fused into one launch:
// panel p's row moves + U12 = L11^{-1} A12 + the K = jb update of the rows
// below, for the column block [cb, ce) (ce - cb <= NB). Replaces mt2_kernel +
// gemm_tma_kernel on the chain (two launches, ~30 us per step at n = 4096 on
// the 16-SM partition) with one cluster of CS CTAs:
//   * every CTA reads the pre-move values it needs -- the moved rows' sources
//     and the U12 rows (a row's value after the moves is its source's value;
//     moves permute the moved positions among themselves) -- then the cluster
//     barrier separates every read of a pre-move value from every write;
//   * every CTA solves U12 (one thread per column, the column in registers,
//     k ascending, one FMA per term: mt2_kernel's bits);
//   * CTA r updates the 64-row tiles r, r + CS, ... below: accumulators start
//     from A (or the moved source) and take one FMA per k in ascending k, as
//     gemm_tma_kernel does (dense_lu.hpp:91-107);
//   * CTA 0 writes U12 back (and its transposed copy for the TMA update).
constexpr int NX_TM = 64;  // rows per update tile (two CTAs fit an SM)
template <int NB>
struct NextSmem
{
  float Lt[NB][NX_TM];  // L21 tile, k-major
  float Ct[NB][NX_TM + 1];  // C tile (coalesced staging of the global loads/stores)
  float U[NB][NB + 4];  // U12 rows (k) x columns (padded: the solve reads columns)
  float LT[NB][NB];     // L11 transposed: LT[kk][i] = l_(k0+i, k0+kk)
  float Mv[2 * NB][NB]; // the moved rows' source values, next columns
  int2 mv[2 * NB];
  int um[NB];           // U12 row i <- move index, -1: not moved
  int mvi[NX_TM];       // tile row r <- move index, -1: not moved
};
template <int NB>
constexpr size_t next_smem() { return sizeof(NextSmem<NB>); }

template <int NB>
__global__ void __launch_bounds__(256, 2)
    next_kernel(float *__restrict__ A, int n, int k0, int jb, int cb, int ce,
                const int2 *__restrict__ moves, const int *__restrict__ nmoves,
                float *__restrict__ ut, int ut_row)
{
  static_assert(NB == 64 && NX_TM == 64, "thread mapping assumes 64 x 64 blocks");
  constexpr int PT = NB * NX_TM / 256;  // elements per thread of a 64 x 64 block
  extern __shared__ __align__(16) unsigned char nsm[];
  NextSmem<NB> &S = *reinterpret_cast<NextSmem<NB> *>(nsm);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int CS = (int)gridDim.x, rank = (int)blockIdx.x;  // the grid is one cluster
  const int w = ce - cb;
  const int r_lo = k0 + jb;
  const int ntile = (n - r_lo + NX_TM - 1) / NX_TM;
  const int nm = *nmoves;
  // element u of this thread in a 64 x 64 block: column (or k) t / 64 + 4u,
  // row t % 64 (consecutive threads read consecutive rows: coalesced)
  const int er = t & 63, ec = t >> 6;

  // ---- phase 0: pre-move reads (all loads in flight before any store)
  {
    float lv[PT], av[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int c = ec + 4 * u;
      lv[u] = (c < jb && er < jb) ? A[(size_t)(k0 + c) * n + k0 + er] : 0.f;
      av[u] = (c < w && er < jb) ? A[(size_t)(cb + c) * n + k0 + er] : 0.f;
    }
    for (int e = t; e < nm; e += 256)
      S.mv[e] = moves[e];
    if (t < NB)
      S.um[t] = -1;
#pragma unroll
    for (int u = 0; u < PT; ++u)
      S.LT[ec + 4 * u][er] = lv[u];
    __syncthreads();
    for (int idx = t; idx < nm * NB; idx += 256)
    {
      const int c = idx / nm, e = idx - c * nm;
      S.Mv[e][c] = c < w ? A[(size_t)(cb + c) * n + S.mv[e].y] : 0.f;
    }
    for (int e = t; e < nm; e += 256)
    {
      const int d = S.mv[e].x - k0;
      if (d >= 0 && d < jb)
        S.um[d] = e;
    }
    __syncthreads();
    const int e = S.um[er];
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int c = ec + 4 * u;
      S.U[er][c] = (e >= 0 && c < w) ? S.Mv[e][c] : av[u];
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");

  // first tile's L21 and C values in flight during the U12 solve
  float pl[PT], pc[PT];
  auto prefetch = [&](int tt) {
    const int r0 = r_lo + tt * NX_TM;
    const int rows = min(NX_TM, n - r0);
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int c = ec + 4 * u;
      pl[u] = (c < jb && er < rows) ? A[(size_t)(k0 + c) * n + r0 + er] : 0.f;
      pc[u] = (c < w && er < rows) ? A[(size_t)(cb + c) * n + r0 + er] : 0.f;
    }
  };
  if (rank < ntile)
    prefetch(rank);

  // ---- phase 1: U12 = L11^{-1} A12, one thread per column (warps 0-1), the
  // column in registers: x_i = fma(-l_ik, x_k, x_i), k ascending (the terms
  // with k >= jb multiply zeros of LT and only touch rows >= jb, never stored)
  if (t < NB)
  {
    float x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i)
      x[i] = S.U[i][t];
#pragma unroll
    for (int kk = 0; kk < NB - 1; ++kk)
    {
      const float xk = x[kk];
#pragma unroll
      for (int i4 = (kk + 1) / 4; i4 < NB / 4; ++i4)
      {
        const float4 l = *reinterpret_cast<const float4 *>(&S.LT[kk][4 * i4]);
        const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * i4 + e > kk)
            x[4 * i4 + e] = __fmaf_rn(-lv[e], xk, x[4 * i4 + e]);
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i)
      S.U[i][t] = x[i];
  }
  __syncthreads();
  if (rank == 0)
  {
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int c = ec + 4 * u;
      if (c < w && er < jb)
        A[(size_t)(cb + c) * n + k0 + er] = S.U[er][c];
    }
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int i = ec + 4 * u, c = er;  // row-major ut: consecutive threads, consecutive columns
      if (c < w && i < jb)
        ut[(size_t)(ut_row + i) * n + cb + c] = S.U[i][c];
    }
  }

  // ---- phase 2: the rows below, 64-row tiles; thread: 4 rows x 4 columns
  const int tx = t & 15, ty = t >> 4;
  for (int tt = rank; tt < ntile; tt += CS)
  {
    const int r0 = r_lo + tt * NX_TM;
    const int rows = min(NX_TM, n - r0);
    if (t < NX_TM)
      S.mvi[t] = -1;
    __syncthreads();  // previous tile's readers of Lt / Ct / mvi are done
    for (int e = t; e < nm; e += 256)
    {
      const int d = S.mv[e].x - r0;
      if (d >= 0 && d < rows)
        S.mvi[d] = e;
    }
    __syncthreads();
    {
      const int e = S.mvi[er];
#pragma unroll
      for (int u = 0; u < PT; ++u)
      {
        const int c = ec + 4 * u;
        S.Lt[c][er] = pl[u];
        S.Ct[c][er] = (e >= 0 && c < w) ? S.Mv[e][c] : pc[u];
      }
    }
    __syncthreads();
    if (tt + CS < ntile)
      prefetch(tt + CS);  // next tile's loads overlap this tile's FMAs
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        acc[i][j] = S.Ct[tx * 4 + j][ty * 4 + i];
#pragma unroll 8
    for (int kk = 0; kk < jb; ++kk)
    {
      const float4 l0 = *reinterpret_cast<const float4 *>(&S.Lt[kk][ty * 4]);
      const float4 uu = *reinterpret_cast<const float4 *>(&S.U[kk][tx * 4]);
      const float l[4] = {l0.x, l0.y, l0.z, l0.w};
      const float u[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          acc[i][j] = __fmaf_rn(-l[i], u[j], acc[i][j]);
    }
    __syncthreads();  // every thread has read its C values
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        S.Ct[tx * 4 + j][ty * 4 + i] = acc[i][j];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PT; ++u)
    {
      const int c = ec + 4 * u;
      if (c < w && er < rows)
        A[(size_t)(cb + c) * n + r0 + er] = S.Ct[c][er];
    }
  }
}

}  // namespace f32u
}  // namespace mpirg
