// K2 -- LU panel factorization, critical-warp design (one thread-block
// cluster of <= 16 CTAs, 4 warps each).
//
// Reproduces the column loop of detail::lu_inplace (dense_lu.hpp:63-107)
// restricted to the panel columns [k0, k0+jb), bit for bit:
//   pivot: first position maximising |a_ik| (as double), strict '>', NaN
//          never chosen, NaN on the diagonal keeps p = k   (65-78)
//   swap:  rows k and p exchange their whole panel row      (79-85)
//   scale: l = a_ik / piv, a true division                  (87-89)
//   update a_ic = a_ic - l * u_kc, one FMA (fp32/fp64) or r16(c - r16(l*u))
//                                                            (91-107)
//
// Design (B200):
//  * Warp 0 of each CTA is the *critical warp*: lane l owns the RPL rows
//    l + 32q of the CTA and keeps their IB current-block columns in
//    registers (static indices; the IB steps of a block are unrolled, the
//    block loop is not). A pivot step is warp-local: candidate, redux.sync
//    argmax, shuffle of the winner's block values, one small st.async message
//    (key, position, NaN flag, IB values) to every CTA of the cluster, an
//    mbarrier wait, a redux argmax over the CS messages, elimination. No
//    __syncthreads and no CTA-level reduction on the per-column path; with a
//    single CTA (m <= 32*RPL) there is no exchange at all.
//  * Rows never move: each row carries its position; a swap is two position
//    updates; rows are written to their final positions at the end (which
//    yields the panel's row-move list for the other columns).
//  * Columns right of the block live in shared memory. At each block end the
//    owners of the block's IB pivot rows broadcast those rows' right columns
//    (one exchange per block), every CTA completes them with the block's
//    multipliers (triangular, step order), and all 4 warps apply the block's
//    IB rank-1 updates to their rows in step order -- the reference's
//    per-element FMA sequence.
#pragma once

#include <climits>

#include "common.cuh"
#include "lu_panel.cuh"

namespace mpirg
{
namespace panel5
{

using panel2::argmax_redux;
using panel2::cluster_rank;
using panel2::cluster_size;
using panel2::cluster_sync_all;
using panel2::is_nan_t;
using panel2::mag_key;
using panel2::mapa;
using panel2::mbar_expect_tx;
using panel2::mbar_init;
using panel2::mbar_wait;
using panel2::smem_addr;
using panel2::st_async_v4;

constexpr int NT = 128;
constexpr int MAXCS = 16;

// Per-step message: header + the candidate row's current-block values.
template <typename T, int IB>
struct alignas(16) Msg
{
  unsigned long long key;  // mag_key of the CTA candidate, 0 = none
  int pos;                 // its position (INT_MAX = none)
  int nan;                 // the row at position k is NaN in column k
  T blk[IB];
};

__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T, int NB, int RPL, int IB>
__host__ __device__ constexpr size_t panel5_dyn_smem()
{
  // P[NB][R] + Ubr[IB][NB] + posS[R]
  return a16(sizeof(T) * (size_t)NB * 32 * RPL) + a16(sizeof(T) * (size_t)IB * NB) +
         a16(sizeof(int) * 32 * RPL);
}

template <typename T, int NB, int RPL, int IB>
__global__ void __launch_bounds__(NT, 1)
    lu_panel5_kernel(T *__restrict__ A, int n, int k0, int jb, int *__restrict__ ipiv,
                     int2 *__restrict__ moves, int *__restrict__ nmoves, DevInfo *info)
{
  constexpr int R = 32 * RPL;
  constexpr bool WIDE = sizeof(T) > 4;
  using M = Msg<T, IB>;
  constexpr int MCH = sizeof(M) / 16;
  constexpr int EPC = 16 / sizeof(T);  // elements per 16-byte chunk
  static_assert(sizeof(M) % 16 == 0, "message must be whole chunks");
  static_assert(NB % IB == 0, "IB must divide NB");
  static_assert((IB * sizeof(T)) % 16 == 0, "block boundaries must be chunk aligned");

  __shared__ M inbox[2][MAXCS];
  __shared__ __align__(8) uint64_t bars[3];  // [0],[1]: step inboxes, [2]: block exchange
  __shared__ T Ublk[IB][IB];                 // block values of the block's pivot rows
  __shared__ int piv_rank[IB], piv_lrow[IB];
  extern __shared__ __align__(16) unsigned char dsm[];
  T *P = reinterpret_cast<T *>(dsm);                                                // [NB][R]
  T *Ubr = reinterpret_cast<T *>(dsm + a16(sizeof(T) * (size_t)NB * R));            // [IB][NB]
  int *posS = reinterpret_cast<int *>(dsm + a16(sizeof(T) * (size_t)NB * R) +
                                      a16(sizeof(T) * (size_t)IB * NB));           // [R]

  const int t = threadIdx.x, lane = t & 31;
  const int warp = t >> 5;
  const int CS = (int)cluster_size();
  const int rank = (int)cluster_rank();
  const int row0 = k0 + rank * R;
  const int mloc = max(0, min(R, n - row0));
  const bool multi = CS > 1;

  // ---- stage the panel (coalesced columns, 4 columns of loads in flight)
  for (int c0 = 0; c0 < jb; c0 += 4)
  {
    T tmp[4][R / NT > 0 ? R / NT : 1];
    constexpr int PER = R / NT > 0 ? R / NT : 1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int s = 0; s < PER; ++s)
      {
        const int i = t + s * NT;
        tmp[u][s] = (i < mloc && c0 + u < jb) ? A[(size_t)(k0 + c0 + u) * n + row0 + i] : T{};
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int s = 0; s < PER; ++s)
      {
        const int i = t + s * NT;
        if (i < R && c0 + u < NB)
          P[(c0 + u) * R + i] = tmp[u][s];
      }
  }
  for (int i = t; i < R; i += NT)
    posS[i] = i < mloc ? row0 + i : -1;

  constexpr uint32_t kStepBytes = 0;  // placeholder (computed per CS below)
  (void)kStepBytes;
  if (t == 0 && multi)
  {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bars[0], (uint32_t)(CS * sizeof(M)));
    if (jb > 1)
      mbar_expect_tx(&bars[1], (uint32_t)(CS * sizeof(M)));
  }
  if (multi)
    cluster_sync_all();
  else
    __syncthreads();

  // critical-warp state
  int pos[RPL];
#pragma unroll
  for (int q = 0; q < RPL; ++q)
    pos[q] = posS[lane + 32 * q];
  uint32_t dst_inbox[2] = {0u, 0u}, dst_bar[2] = {0u, 0u};
  if (warp == 0 && multi && lane < CS)
  {
#pragma unroll
    for (int par = 0; par < 2; ++par)
    {
      dst_inbox[par] = mapa(smem_addr(&inbox[par][rank]), lane);
      dst_bar[par] = mapa(smem_addr(&bars[par]), lane);
    }
  }

#ifdef MPIRG_DEBUG_PANEL
  long long pacc[16] = {};
  long long plast = clock64();
#define P5_MARK(i)                          \
  do                                        \
  {                                         \
    if (t == 0)                             \
    {                                       \
      const long long now = clock64();      \
      pacc[i] += now - plast;               \
      plast = now;                          \
    }                                       \
  } while (0)
#else
#define P5_MARK(i) \
  do               \
  {                \
  } while (0)
#endif
  int step = 0;
  int blk = 0;
#pragma unroll 1
  for (int jb0 = 0; jb0 < jb; jb0 += IB, ++blk)
  {
    const int bend = min(jb0 + IB, jb);
    const int nb_here = bend - jb0;
    // right-column chunks of one pivot row (from bend to NB, chunk aligned)
    const int rch = (int)(((size_t)(NB - (jb0 + IB)) * sizeof(T) + 15) / 16);
    // Arm the block exchange before any of this block's step messages leave:
    // a peer can only send block data after it got every CTA's last step message.
    if (t == 0 && multi && rch > 0 && jb0 + IB < jb)
      mbar_expect_tx(&bars[2], (uint32_t)(nb_here * rch * 16));

    if (warp == 0)
    {
      T cur[RPL][IB];
#pragma unroll
      for (int q = 0; q < RPL; ++q)
#pragma unroll
        for (int c = 0; c < IB; ++c)
          cur[q][c] = P[(jb0 + c) * R + lane + 32 * q];

#pragma unroll
      for (int jj = 0; jj < IB; ++jj)
      {
        const int j = jb0 + jj;
        if (j >= jb)
          break;
        const int k = k0 + j;
        const int par = step & 1;
        // 1. candidate among my unchosen rows
        unsigned long long bkey = 0ull;
        int bp = INT_MAX, bq = 0, nan = 0;
#pragma unroll
        for (int q = 0; q < RPL; ++q)
        {
          if (pos[q] >= k)
          {
            if (is_nan_t(cur[q][jj]))
              nan |= (pos[q] == k);
            else
            {
              const unsigned long long key = mag_key(cur[q][jj]);
              if (key > bkey || (key == bkey && pos[q] < bp))
              {
                bkey = key;
                bp = pos[q];
                bq = q;
              }
            }
          }
        }
        P5_MARK(0);
        // 2. CTA argmax (= warp argmax)
        unsigned long long ckey;
        int cpos;
        argmax_redux<WIDE>(bkey, bp, ckey, cpos);
        const int cn = __any_sync(0xffffffffu, nan);
        const bool owner = bkey != 0ull && bkey == ckey && bp == cpos;
        const unsigned obal = __ballot_sync(0xffffffffu, owner);
        const int ol = obal ? __ffs(obal) - 1 : 0;
        if (ckey == 0ull)
          cpos = INT_MAX;
        P5_MARK(1);
        // 3. the candidate's block values to every lane
        T wv[IB];
#pragma unroll
        for (int c = 0; c < IB; ++c)
        {
          T mine = cur[0][c];
#pragma unroll
          for (int q = 1; q < RPL; ++q)
            if (bq == q)
              mine = cur[q][c];
          wv[c] = shfl_t(mine, ol);
        }
        P5_MARK(2);
        // 4. exchange across the cluster (or take it directly)
        unsigned long long gkey = ckey;
        int gp = cpos, gn = cn, gr = rank;
        T U[IB];
        if (multi)
        {
          if (lane < CS)
          {
            M m;
            m.key = ckey;
            m.pos = cpos;
            m.nan = cn;
#pragma unroll
            for (int c = 0; c < IB; ++c)
              m.blk[c] = wv[c];
            const uint4 *src = reinterpret_cast<const uint4 *>(&m);
#pragma unroll
            for (int ch = 0; ch < MCH; ++ch)
              st_async_v4(dst_inbox[par] + ch * 16, src[ch], dst_bar[par]);
          }
          mbar_wait(&bars[par], (uint32_t)((step >> 1) & 1));
          if (lane == 0 && step + 2 < jb)
            mbar_expect_tx(&bars[par], (uint32_t)(CS * sizeof(M)));
          const unsigned long long gk0 = lane < CS ? inbox[par][lane].key : 0ull;
          const int gp0 = lane < CS ? inbox[par][lane].pos : INT_MAX;
          argmax_redux<WIDE>(gk0, gp0, gkey, gp);
          gr = __ffs(__ballot_sync(0xffffffffu, lane < CS && gk0 == gkey &&
                                                    (gkey == 0ull || gp0 == gp))) -
               1;
          gn = __any_sync(0xffffffffu, lane < CS ? inbox[par][lane].nan : 0);
#pragma unroll
          for (int c = 0; c < IB; ++c)
            U[c] = inbox[par][gr].blk[c];
        }
        else
        {
#pragma unroll
          for (int c = 0; c < IB; ++c)
            U[c] = wv[c];
        }
        P5_MARK(3);
        const int p = gn ? k : gp;
        if (lane == 0)
        {
          if (rank == 0)
          {
            ipiv[k] = p;
            if (!gn && gkey == 1ull)  // |pivot| == +0
              atomicMin(&info->singular_col, k);
          }
          piv_rank[jj] = gn ? -1 : gr;  // NaN pivot: the row at position k (owner marks it)
        }
        if (lane < IB)
        {
          T u = U[0];
#pragma unroll
          for (int c = 1; c < IB; ++c)
            if (lane == c)
              u = U[c];
          Ublk[jj][lane] = u;
        }
        const T piv = U[jj];
        P5_MARK(4);
        // 5. positions + elimination inside the block
#pragma unroll
        for (int q = 0; q < RPL; ++q)
        {
          if (pos[q] >= k)
          {
            if (pos[q] == p)
            {
              pos[q] = k;  // the pivot row moves to position k
              // record the owner's local row for the block exchange
              piv_rank[jj] = rank;
              piv_lrow[jj] = lane + 32 * q;
            }
            else
            {
              if (pos[q] == k)
                pos[q] = p;  // the displaced row takes the pivot's old position
              const T l = divide(cur[q][jj], piv);
              cur[q][jj] = l;
#pragma unroll
              for (int c = jj + 1; c < IB; ++c)
                cur[q][c] = upd(cur[q][c], l, U[c]);
            }
          }
        }
        ++step;
        P5_MARK(5);
      }
#pragma unroll
      for (int q = 0; q < RPL; ++q)
      {
#pragma unroll
        for (int c = 0; c < IB; ++c)
          P[(jb0 + c) * R + lane + 32 * q] = cur[q][c];
        posS[lane + 32 * q] = pos[q];
      }
    }
    __syncthreads();  // block columns, positions, piv_rank/lrow, Ublk final
    P5_MARK(6);

    if (bend < jb)
    {
      // ---- block end (a): the block's pivot rows, right columns, to every CTA
      const int c_lo = jb0 + IB;  // chunk-aligned start of the right columns
      if (multi)
      {
        // sender side: (jj, dst, ch) triples for the pivot rows I own
        const int per_row = CS * rch;
        for (int idx = t; idx < nb_here * per_row; idx += NT)
        {
          const int jj = idx / per_row, rem = idx % per_row;
          if (piv_rank[jj] != rank)
            continue;
          const int dst = rem / rch, ch = rem % rch;
          const int lrow = piv_lrow[jj];
          T e[EPC];
#pragma unroll
          for (int w = 0; w < EPC; ++w)
          {
            const int c = c_lo + ch * EPC + w;
            e[w] = (c < jb) ? P[c * R + lrow] : T{};
          }
          const uint32_t raddr = mapa(smem_addr(Ubr + jj * NB + c_lo) + ch * 16, dst);
          st_async_v4(raddr, *reinterpret_cast<const uint4 *>(e), mapa(smem_addr(&bars[2]), dst));
        }
        mbar_wait(&bars[2], (uint32_t)(blk & 1));
      }
      else
      {
        for (int idx = t; idx < nb_here * (jb - bend); idx += NT)
        {
          const int jj = idx / (jb - bend), c = bend + idx % (jb - bend);
          Ubr[jj * NB + c] = P[c * R + piv_lrow[jj]];
        }
        __syncthreads();
      }
      P5_MARK(7);
      // (b) complete the pivot rows: U_jj[c] -= l(pivot jj, jp) * U_jp[c], jp < jj
      for (int c = bend + t; c < jb; c += NT)
      {
        T u[IB];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
          u[jj] = Ubr[jj * NB + c];
#pragma unroll
        for (int jj = 1; jj < IB; ++jj)
          if (jj < nb_here)
          {
#pragma unroll
            for (int jp = 0; jp < jj; ++jp)
              u[jj] = upd(u[jj], Ublk[jj][jp], u[jp]);
          }
#pragma unroll
        for (int jj = 1; jj < IB; ++jj)
          Ubr[jj * NB + c] = u[jj];
      }
      __syncthreads();
      P5_MARK(8);
      // (c) every row of this CTA: right columns get the block's updates for
      //     the steps at which it was below the pivot.
      for (int i = t; i < mloc; i += NT)
      {
        const int ps = posS[i];
        if (ps < k0 + jb0)
          continue;  // a pivot of an earlier block
        const int upto = ps < k0 + bend ? ps - (k0 + jb0) : IB;
        T lq[IB];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
          lq[jj] = P[(jb0 + jj) * R + i];
        int c = bend;
        for (; c + 4 <= jb; c += 4)
        {
          T v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[e] = P[(c + e) * R + i];
#pragma unroll
          for (int jj = 0; jj < IB; ++jj)
            if (jj < upto)
            {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                v[e] = upd(v[e], lq[jj], Ubr[jj * NB + c + e]);
            }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            P[(c + e) * R + i] = v[e];
        }
        for (; c < jb; ++c)
        {
          T v = P[c * R + i];
#pragma unroll
          for (int jj = 0; jj < IB; ++jj)
            if (jj < upto)
              v = upd(v, lq[jj], Ubr[jj * NB + c]);
          P[c * R + i] = v;
        }
      }
      __syncthreads();
      P5_MARK(9);
    }
  }
#ifdef MPIRG_DEBUG_PANEL
  if (t == 0 && rank == 0 && (k0 == 0 || k0 + jb >= n || k0 == n / 2))
    printf("p5 k0=%d CS=%d RPL=%d IB=%d per step: cand %lld argmax %lld bcast %lld xchg %lld rec %lld "
           "upd %lld | per panel: wtail %lld bx %lld compl %lld upd %lld\n",
           k0, CS, RPL, IB, pacc[0] / step, pacc[1] / step, pacc[2] / step, pacc[3] / step,
           pacc[4] / step, pacc[5] / step, pacc[6], pacc[7], pacc[8], pacc[9]);
#endif

  // ---- write every row to its final position; record the row moves
  for (int i = t; i < mloc; i += NT)
  {
    const int ps = posS[i];
    const int g = row0 + i;
    for (int c = 0; c < jb; ++c)
      A[(size_t)(k0 + c) * n + ps] = P[c * R + i];
    if (ps != g)
    {
      const int e = atomicAdd(nmoves, 1);
      moves[e] = make_int2(ps, g);
    }
  }
  if (multi)
    cluster_sync_all();  // no CTA may exit while peers can still write its memory
}

}  // namespace panel5
}  // namespace mpirg
