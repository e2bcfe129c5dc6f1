// K2 -- LU panel factorization on one thread-block cluster (<= 16 CTAs).
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
//  * Rows never move. Each row carries its current position; a swap is two
//    position updates, and every row is written to its final position at the
//    end (which also yields the panel's row-move list for the other columns).
//  * One pivot step = one cluster-wide exchange: each CTA reduces its best
//    candidate (|a|, position) with warp shuffles + one __syncthreads, then
//    pushes the candidate's row into every CTA's inbox with st.async, which
//    completes bytes on the receiver's mbarrier. Each CTA waits only on its
//    own mbarrier -- no barrier.cluster on the critical path.
//  * Inner blocking (IB columns): the IB columns of the current block live in
//    registers with static indices (the IB steps are unrolled, the block loop
//    is not -- a fully unrolled panel is ~400 KB of SASS and stalls on
//    instruction fetch). Columns right of the block live in shared memory
//    and receive the block's IB rank-1 updates at the block end, in step
//    order, after the block's pivot rows are completed by a small triangular
//    correction -- the same per-element FMA sequence as the reference.
#pragma once

#include <climits>

#include "common.cuh"

namespace mpirg
{
namespace panel2
{

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int MAXCS = 16;
constexpr int IB = 8;

template <typename T, int NB>
struct alignas(16) Slot
{
  double val;  // |pivot candidate| as double, -1 = none
  int pos;     // its current position (INT_MAX = none)
  int nan;     // the row at position k holds a NaN in column k
  T row[NB];   // the candidate row (panel columns, as of this step)
};

// Warp-level candidate staged for the CTA reduction.
template <typename T>
struct alignas(16) WSlot
{
  double val;
  int pos;
  int nan;
  int lrow;  // local row index (for the columns right of the block, in P)
  int pad[3];
  T blk[IB];  // the block columns (registers of the owner thread)
};

__device__ __forceinline__ bool better(double v1, int p1, double v2, int p2)
{
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// Argmax with the reference's tie rule: the largest |a| (as double bits, all
// candidates are >= +0 so the bit order is the numeric order; 0 = no
// candidate), then the lowest position among equal values.
__device__ __forceinline__ unsigned long long max_u64_xor(unsigned long long v, int width)
{
  for (int o = width >> 1; o > 0; o >>= 1)
  {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  // a partial-width butterfly leaves the result only in lanes [0, width):
  // make it warp-uniform
  return width < 32 ? __shfl_sync(0xffffffffu, v, 0) : v;
}

__device__ __forceinline__ unsigned long long cand_bits(double a)
{
  // +0.0 and positive values map above 0 so "no candidate" can be 0.
  return (unsigned long long)__double_as_longlong(a) + 1ull;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank)
{
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar)
{
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
      "[%5];" ::"r"(raddr),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
      : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all()
{
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank()
{
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_size()
{
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// Dynamic shared memory: P[NB][R] (this CTA's rows, column-major) + Ub[IB][NB].
template <typename T, int NB, int RPT>
__host__ __device__ constexpr size_t panel_dyn_smem()
{
  return a16(sizeof(T) * (size_t)NB * RPT * NT) + a16(sizeof(T) * (size_t)IB * NB);
}

// rows of this CTA: row0 + t + q*NT, q < RPT (R = RPT*NT rows per CTA)
template <typename T, int NB, int RPT>
__global__ void __launch_bounds__(NT, 1)
    lu_panel2_kernel(T *__restrict__ A, int n, int k0, int jb, int *__restrict__ ipiv,
                     int2 *__restrict__ moves, int *__restrict__ nmoves, DevInfo *info)
{
  using S = Slot<T, NB>;
  constexpr int NCH = sizeof(S) / 16;
  constexpr int R = RPT * NT;
  static_assert(sizeof(S) % 16 == 0, "slot must be a multiple of 16 bytes");
  static_assert(NB % IB == 0, "NB must be a multiple of IB");
  __shared__ WSlot<T> wslot[2][NW];  // double-buffered: a slow pusher of step j never sees step j+1
  __shared__ S inbox[2][MAXCS];
  __shared__ __align__(8) uint64_t bars[2];
  extern __shared__ __align__(16) unsigned char dsm[];
  T *P = reinterpret_cast<T *>(dsm);                                   // [NB][R]
  T *Ub = reinterpret_cast<T *>(dsm + a16(sizeof(T) * (size_t)NB * R));  // [IB][NB]

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int CS = (int)cluster_size();
  const int rank = (int)cluster_rank();
  const int row0 = k0 + rank * R;

  int pos[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q)
  {
    const int g = row0 + t + q * NT;
    pos[q] = g < n ? g : -1;  // -1: no row
  }
  // Stage the panel rows in shared memory (coalesced columns, 8 columns of
  // loads in flight per batch).
  for (int c0 = 0; c0 < jb; c0 += 8)
  {
    T tmp[8][RPT];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        tmp[u][q] = (pos[q] >= 0 && c0 + u < jb) ? A[(size_t)(k0 + c0 + u) * n + pos[q]] : T{};
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (c0 + u < NB)
          P[(c0 + u) * R + t + q * NT] = tmp[u][q];
  }
  // Bytes my inbox receives at step s (all CS candidates; chunks left of the
  // step's block are not sent).
  auto step_bytes = [&](int s) -> uint32_t {
    const int blk0 = (s / IB) * IB;
    return (uint32_t)(CS * (NCH - (int)((blk0 * sizeof(T)) / 16)) * 16);
  };
  if (t == 0)
  {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // Arm the first two phases before any peer can send (the expect_tx must
    // precede every complete_tx of its phase).
    mbar_expect_tx(&bars[0], step_bytes(0));
    if (jb > 1)
      mbar_expect_tx(&bars[1], step_bytes(1));
  }
  cluster_sync_all();

  // Push assignment (fixed for the whole panel): chunk idx = t + u*NT of the
  // CS*NCH chunks goes to CTA idx / NCH, chunk idx % NCH of my inbox slot there.
  constexpr int PUSH_PER = (MAXCS * NCH + NT - 1) / NT;
  int my_ch[PUSH_PER];
  uint32_t my_raddr[PUSH_PER], my_rbar[PUSH_PER];
  {
    const uint32_t slot0 = smem_addr(&inbox[0][rank]);
    const uint32_t bar0 = smem_addr(&bars[0]);
#pragma unroll
    for (int u = 0; u < PUSH_PER; ++u)
    {
      const int idx = t + u * NT;
      if (idx < CS * NCH)
      {
        const int dst = idx / NCH, ch = idx % NCH;
        my_ch[u] = ch;
        my_raddr[u] = mapa(slot0 + ch * 16, dst);
        my_rbar[u] = mapa(bar0, dst);
      }
      else
      {
        my_ch[u] = -1;
        my_raddr[u] = my_rbar[u] = 0;
      }
    }
  }

  T cur[RPT][IB];  // current block columns (registers, static indices)
  int step = 0;    // global step index j (parity / phase bookkeeping)
#pragma unroll 1
  for (int jb0 = 0; jb0 < jb; jb0 += IB)
  {
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int jj = 0; jj < IB; ++jj)
        cur[q][jj] = P[(jb0 + jj) * R + t + q * NT];
    int chosen[RPT];  // step within this block at which the row became a pivot, IB = never
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      chosen[q] = IB;
    const int bend = min(jb0 + IB, jb);  // first column right of the block

#pragma unroll
    for (int jj = 0; jj < IB; ++jj)
    {
      const int j = jb0 + jj;
      if (j >= jb)
        break;
      const int k = k0 + j;
      const int par = step & 1;

      // 1. thread-local candidate among unchosen rows (positions >= k).
      unsigned long long bkey = 0ull;
      int bp = INT_MAX, bq = 0, nan = 0;
#pragma unroll
      for (int q = 0; q < RPT; ++q)
      {
        if (pos[q] >= k)
        {
          const double a = fabs(to_d(cur[q][jj]));
          if (isnan(a))
            nan |= (pos[q] == k);
          else
          {
            const unsigned long long key = cand_bits(a);
            if (key > bkey || (key == bkey && pos[q] < bp))
            {
              bkey = key;
              bp = pos[q];
              bq = q;
            }
          }
        }
      }
      // 2. warp argmax: max |a|, then min position among ties.
      const unsigned long long wkey = max_u64_xor(bkey, 32);
      const int wpos = (int)__reduce_min_sync(0xffffffffu,
                                              (bkey == wkey && bkey != 0ull) ? (unsigned)bp
                                                                             : 0x7fffffffu);
      nan = __any_sync(0xffffffffu, nan);
      // 3. the warp winner stages header + its block columns + its local row id.
      const bool owner = bkey != 0ull && bkey == wkey && bp == wpos;
      if (owner || (lane == 0 && wkey == 0ull))
      {
        WSlot<T> &ws = wslot[par][warp];
        ws.val = wkey == 0ull ? -1.0 : __longlong_as_double((long long)(wkey - 1ull));
        ws.pos = wkey == 0ull ? INT_MAX : wpos;
        ws.nan = nan;
        ws.lrow = t + bq * NT;
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          if (q == bq)
          {
#pragma unroll
            for (int c = 0; c < IB; ++c)
              ws.blk[c] = cur[q][c];
          }
      }
      __syncthreads();
      // 4. CTA winner over the warp slots (every warp computes it redundantly).
      const double wv = lane < NW ? wslot[par][lane].val : -1.0;
      const int wp = lane < NW ? wslot[par][lane].pos : INT_MAX;
      const unsigned long long ckey0 = (lane < NW && wv >= 0.0) ? cand_bits(wv) : 0ull;
      const unsigned long long ckey = max_u64_xor(ckey0, 8);
      const int cp = (int)__reduce_min_sync(0xffffffffu, (ckey0 == ckey && ckey0 != 0ull)
                                                             ? (unsigned)wp
                                                             : 0x7fffffffu);
      const unsigned cmatch = __ballot_sync(0xffffffffu, lane < NW && ckey0 == ckey &&
                                                             (ckey == 0ull || wp == cp));
      const int cw = __ffs(cmatch) - 1;
      const double cv = ckey == 0ull ? -1.0 : __longlong_as_double((long long)(ckey - 1ull));
      const int cpos = ckey == 0ull ? INT_MAX : cp;
      const int cn = __any_sync(0xffffffffu, lane < NW ? wslot[par][lane].nan : 0);
      // 5. push [header | block cols from wslot | right cols from P] to every inbox.
      {
        const WSlot<T> &ws = wslot[par][cw];
        const int lrow = ws.lrow;
        const int ch_lo = 1 + (int)((jb0 * sizeof(T)) / 16);  // first chunk holding col >= jb0
        constexpr int EPC = 16 / sizeof(T);                    // elements per chunk
#pragma unroll
        for (int u = 0; u < PUSH_PER; ++u)
        {
          const int ch = my_ch[u];
          if (ch < 0 || (ch != 0 && ch < ch_lo))
            continue;  // columns left of the block are never read by receivers
          uint4 val;
          if (ch == 0)
          {
            const unsigned long long vb = (unsigned long long)__double_as_longlong(cv);
            val = make_uint4((uint32_t)vb, (uint32_t)(vb >> 32), (uint32_t)cpos, (uint32_t)cn);
          }
          else
          {
            T e[EPC];
#pragma unroll
            for (int w = 0; w < EPC; ++w)
            {
              const int c = (ch - 1) * EPC + w;
              e[w] = (c < bend) ? ws.blk[c - jb0]
                                : (c < jb && cpos != INT_MAX ? P[c * R + lrow] : T{});
            }
            val = *reinterpret_cast<const uint4 *>(e);
          }
          st_async_v4(my_raddr[u] + (uint32_t)(par * MAXCS * sizeof(S)), val,
                      my_rbar[u] + (uint32_t)(par * sizeof(uint64_t)));
        }
      }
      // 6. wait until all CS candidates are in my inbox.
      mbar_wait(&bars[par], (uint32_t)((step >> 1) & 1));
      // Re-arm this barrier for step+2 now: no peer can send step+2 data before
      // every CTA (this one included) has pushed step+1, which this thread
      // precedes in program order.
      if (t == 0 && step + 2 < jb)
        mbar_expect_tx(&bars[par], step_bytes(step + 2));
      // 7. global winner (identical in every thread of every CTA).
      const double iv = lane < CS ? inbox[par][lane].val : -1.0;
      const int ip = lane < CS ? inbox[par][lane].pos : INT_MAX;
      const unsigned long long gkey0 = (lane < CS && iv >= 0.0) ? cand_bits(iv) : 0ull;
      const unsigned long long gkey = max_u64_xor(gkey0, 16);
      const int gp = (int)__reduce_min_sync(0xffffffffu, (gkey0 == gkey && gkey0 != 0ull)
                                                             ? (unsigned)ip
                                                             : 0x7fffffffu);
      const unsigned gmatch = __ballot_sync(0xffffffffu, lane < CS && gkey0 == gkey &&
                                                             (gkey == 0ull || ip == gp));
      const int gr = __ffs(gmatch) - 1;
      const int gn = __any_sync(0xffffffffu, lane < CS ? inbox[par][lane].nan : 0);
      const double gv = gkey == 0ull ? -1.0 : __longlong_as_double((long long)(gkey - 1ull));
      const int p = gn ? k : gp;
      const T *U = inbox[par][gr].row;
      if (rank == 0 && t == 0)
      {
        ipiv[k] = p;
        if (!gn && gv == 0.0)
          atomicMin(&info->singular_col, k);
      }
      // keep the pivot row (stale right columns) for the block-end update
      for (int c = bend + t; c < jb; c += NT)
        Ub[jj * NB + c] = U[c];
      if (t < IB)
        Ub[jj * NB + jb0 + t] = U[jb0 + t];
      const T piv = U[j];
      T ub[IB];
#pragma unroll
      for (int c = jj + 1; c < IB; ++c)
        ub[c] = U[jb0 + c];
      // 8. positions + elimination inside the block (a NaN pivot makes U
      //    irrelevant: l = NaN).
#pragma unroll
      for (int q = 0; q < RPT; ++q)
      {
        if (pos[q] >= k)
        {
          if (pos[q] == p)
          {
            pos[q] = k;  // the pivot row moves to position k
            chosen[q] = jj;
          }
          else
          {
            if (pos[q] == k)
              pos[q] = p;  // the displaced row takes the pivot's old position
            const T l = divide(cur[q][jj], piv);
            cur[q][jj] = l;
#pragma unroll
            for (int c = jj + 1; c < IB; ++c)
              cur[q][c] = upd(cur[q][c], l, ub[c]);
          }
        }
      }
      ++step;
    }

    // ---- block end: apply the block's rank-1 updates to the columns right
    // of the block, in step order.
    __syncthreads();  // Ub complete
    const int nb_here = bend - jb0;
    // (a) complete the pivot rows: U_jj[c] -= l(pivot jj, jj') * U_jj'[c], jj' < jj
    for (int c = bend + t; c < jb; c += NT)
    {
      T u[IB];
#pragma unroll
      for (int jj = 0; jj < IB; ++jj)
        u[jj] = Ub[jj * NB + c];
#pragma unroll
      for (int jj = 1; jj < IB; ++jj)
        if (jj < nb_here)
        {
#pragma unroll
          for (int jp = 0; jp < jj; ++jp)
            u[jj] = upd(u[jj], Ub[jj * NB + jb0 + jp], u[jp]);
        }
#pragma unroll
      for (int jj = 1; jj < IB; ++jj)
        Ub[jj * NB + c] = u[jj];
    }
    __syncthreads();
    // (b) every row: its right columns get the updates of the steps at which it
    //     was still below the pivot (all IB for non-pivot rows).
#pragma unroll
    for (int q = 0; q < RPT; ++q)
    {
      const int r = t + q * NT;
#pragma unroll
      for (int jj = 0; jj < IB; ++jj)
        P[(jb0 + jj) * R + r] = cur[q][jj];
      if (pos[q] < 0 || (pos[q] < k0 + jb0 && chosen[q] == IB))
        continue;  // no row, or a pivot of an earlier block
      const int upto = min(chosen[q], nb_here);
#pragma unroll 4
      for (int c = bend; c < jb; ++c)
      {
        T v = P[c * R + r];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
          if (jj < upto)
            v = upd(v, cur[q][jj], Ub[jj * NB + c]);
        P[c * R + r] = v;
      }
    }
    __syncthreads();
  }

  // Write every row to its final position; record the row moves.
#pragma unroll
  for (int q = 0; q < RPT; ++q)
  {
    if (pos[q] >= 0)
    {
      const int g = row0 + t + q * NT;
      for (int c = 0; c < jb; ++c)
        A[(size_t)(k0 + c) * n + pos[q]] = P[c * R + t + q * NT];
      if (pos[q] != g)
      {
        const int e = atomicAdd(nmoves, 1);
        moves[e] = make_int2(pos[q], g);
      }
    }
  }
  cluster_sync_all();  // no CTA may exit while peers can still write its inbox
}

}  // namespace panel2
}  // namespace mpirg
