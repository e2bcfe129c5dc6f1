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
#include "lu_spec.cuh"

namespace mpirg
{
namespace panel2
{

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int IB = 8;

// Per-step message of one CTA: its candidate and the candidate's current
// block columns (the columns right of the block travel once per block).
template <typename T>
struct alignas(16) Slot
{
  unsigned long long key;  // mag_key of the candidate, 0 = none
  int pos;                 // its current position (INT_MAX = none)
  int nan;                 // the row at position k holds a NaN in column k
  T blk[IB];               // the candidate's block columns, as of this step
};

// Speculative block message: the block's IB finished pivot rows (block
// columns) and whether the block's natural rows were in place.
template <typename T>
struct alignas(16) BMsg
{
  T blk[IB][IB];
  uint32_t flag;
  uint32_t pad[3];
};

// Warp-level candidate staged for the CTA reduction.
template <typename T>
struct alignas(16) WSlot
{
  unsigned long long key;
  int pos;
  int nan;
  int lrow;  // local row index (for the columns right of the block, in P)
  int pad[3];
  T blk[IB];  // the block columns (registers of the owner thread)
};

__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, uint32_t src_cta,
                                               uint32_t bytes, uint32_t bar_cluster)
{
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(bar_cluster)
      : "memory");
}

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

// Warp-uniform argmax over (key, pos): the largest key, ties to the lowest
// position. redux.sync does each reduction in one instruction; 64-bit keys
// (binary64 magnitudes) take a hi/lo pass.
template <bool WIDE>
__device__ __forceinline__ void argmax_redux(unsigned long long key, int pos,
                                             unsigned long long &mkey, int &mpos)
{
  if constexpr (!WIDE)
  {
    const unsigned k32 = (unsigned)key;
    const unsigned m = __reduce_max_sync(0xffffffffu, k32);
    mkey = m;
    mpos = (int)__reduce_min_sync(0xffffffffu, (k32 == m && m != 0u) ? (unsigned)pos
                                                                      : 0x7fffffffu);
  }
  else
  {
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    mkey = ((unsigned long long)mh << 32) | ml;
    mpos = (int)__reduce_min_sync(0xffffffffu, (key == mkey && mkey != 0ull) ? (unsigned)pos
                                                                           : 0x7fffffffu);
  }
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
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


// Dynamic shared memory: P[NB][R] (this CTA's rows, column-major) + Ub[IB][NB]
// (the block's pivot rows: block columns from the step messages, right
// columns from the block-end exchange).
template <typename T, int NB, int RPT, int NTX = NT>
__host__ __device__ constexpr size_t panel_exact_smem()
{
  return a16(sizeof(T) * (size_t)NB * RPT * NTX) + a16(sizeof(T) * (size_t)IB * NB);
}
// With the whole-panel speculation (which keeps its own layout in the same
// buffer: lu_spec.cuh) enabled for the launch.
template <typename T, int NB, int RPT, int NTX = NT>
__host__ __device__ constexpr size_t panel_dyn_smem()
{
  const size_t exact = panel_exact_smem<T, NB, RPT, NTX>();
  const size_t spec = (sizeof(T) == 4 && NB == 64 && RPT == 1 && NTX == 256)
                          ? a16(2 * sizeof(float) * (size_t)NB * NB + 256) + sizeof(float) * (size_t)2 * NB * NTX
                          : 0;
  return exact > spec ? exact : spec;
}

#ifdef MPIRG_DEBUG_PANEL
#define PT_MARK(i)                                                         \
  do                                                                       \
  {                                                                        \
    if (t == 0)                                                            \
    {                                                                      \
      const long long now = clock64();                                     \
      ptacc[i] += now - ptlast;                                            \
      ptlast = now;                                                        \
    }                                                                      \
  } while (0)
#else
#define PT_MARK(i) \
  do                \
  {                 \
  } while (0)
#endif

// rows of this CTA: row0 + t + q*NT, q < RPT (R = RPT*NT rows per CTA)
// NTX threads per CTA (256 for the panel of the blocked LU; 512 for the
// 8-column leaf of a tall panel, lu.cu panel_tall).
// TG: the matrix's storage type when it differs from the arithmetic type T
// (the tensor-core mode factors binary16 panels in binary32: widened on load,
// rounded once on store).
template <typename T, typename TG>
__device__ __forceinline__ T panel_in(TG v)
{
  if constexpr (std::is_same<T, TG>::value)
    return v;
  else
    return promote<T, TG>(v);
}
template <typename TG, typename T>
__device__ __forceinline__ TG panel_out(T v)
{
  if constexpr (std::is_same<T, TG>::value)
    return v;
  else
    return demote<TG, T>(v);
}

// Returns true when the panel was completed here (A, ipiv, info updated).
// Row mapping of this pass (its own, not the exchange algorithm's): warp 0 of
// every CTA has the diagonal block only; the m - NB rows below it are dealt to
// the other NTX - 32 threads of the CS CTAs, consecutive rows to consecutive
// threads, in up to NR slots per thread.
template <int NB, int NR, int NTX, typename TG>
__device__ __forceinline__ bool whole_panel_spec(TG *__restrict__ A, int n, int k0, unsigned char *dsm,
                                                 int *__restrict__ ipiv, DevInfo *info, int CS,
                                                 int rank)
{
  constexpr int NBLK = NB / 8;
  constexpr int RT = NTX - 32;  // row threads per CTA
  auto &sh = *reinterpret_cast<SpecShared<NB> *>(dsm);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float *stash = reinterpret_cast<float *>(dsm + a16(sizeof(SpecShared<NB>))) + t;
#ifdef MPIRG_DEBUG_PANEL
  const long long w0 = clock64();
  long long w1 = w0, w2 = w0, w3 = w0;
#endif
  if (t == 0)
  {
    sh.prog = 0;
    sh.abort = 0;
    sh.zj = NB;
  }
  __syncthreads();
  bool beaten = false, stop = false;
  // an equal share of the rows below the block per CTA (contiguous), slot q of
  // thread t - 32 = the share's row q RT + t - 32: only the first warps of a
  // CTA have second-slot rows
  const int below = n - k0 - NB;
  const int per = (below + CS - 1) / CS;
  const int base = k0 + NB + rank * per;
  int row[NR];
  bool act[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q)
  {
    const int i = q * RT + (t - 32);
    row[q] = base + i;
    act[q] = warp != 0 && i < per && row[q] < n;
  }
  if (warp == 0)
  {
    float D[2][NBLK][8];
#pragma unroll
    for (int c = 0; c < NB; ++c)
    {
      D[0][c / 8][c % 8] = panel_in<float, TG>(A[(size_t)(k0 + c) * n + k0 + lane]);
      D[1][c / 8][c % 8] = panel_in<float, TG>(A[(size_t)(k0 + c) * n + k0 + lane + 32]);
    }
    int zj = NB;
#ifdef MPIRG_DEBUG_PANEL
    w1 = clock64();
#endif
    spec_diag_phase<NB, 0>(D, sh, lane, rank == 0, beaten, zj, stop);
    spec_diag_phase<NB, 1>(D, sh, lane, rank == 0, beaten, zj, stop);
#ifdef MPIRG_DEBUG_PANEL
    w2 = clock64();
#endif
    if (rank == 0 && lane == 0)
      sh.zj = zj;
    beaten = false;  // (recorded in sh.abort)
  }
  else if (__any_sync(0xffffffffu, act[0]))
  {
    const bool two = NR > 1 && __any_sync(0xffffffffu, act[NR - 1]);  // this warp has second-slot rows
    // the rows go to the stash, eight columns of loads in flight at a time
#pragma unroll 1
    for (int c0 = 0; c0 < NB; c0 += 8)
    {
      float tmp[NR][8];
#pragma unroll
      for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          tmp[q][e] = act[q] ? panel_in<float, TG>(A[(size_t)(k0 + c0 + e) * n + row[q]]) : 0.0f;
#pragma unroll
      for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          stash[(size_t)(q * NB + c0 + e) * NTX] = tmp[q][e];
    }
#pragma unroll 1
    for (int b = 0; b < NBLK; ++b)
    {
      if (b > 0 && __any_sync(0xffffffffu, beaten))
      {
        // tell every CTA of the cluster, not only this one: the others would
        // run their whole share before the verdict (plain remote stores; the
        // verdict's cluster barrier completes them before any shared memory is reused)
        sh.abort = 1;
        if (CS > 1 && lane < CS)
          asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(
                           mapa(smem_addr(const_cast<const int *>(&sh.abort)), (uint32_t)lane)),
                       "r"(1u)
                       : "memory");
      }
      while (sh.prog < 8 * (b + 1) && !sh.abort)
        __nanosleep(40);
      if (sh.abort)
        stop = true;
      if (stop)
        break;
      __threadfence_block();
      if (two)
        spec_rows_block<NB, NR, NTX>(stash, act, sh.U, b, beaten);
      else
      {
        const bool act1[1] = {act[0]};
        spec_rows_block<NB, 1, NTX>(stash, act1, sh.U, b, beaten);
      }
    }
  }
  if (__any_sync(0xffffffffu, beaten))
    sh.abort = 1;
#ifdef MPIRG_DEBUG_PANEL
  w3 = clock64();
#endif
  __syncthreads();
#ifdef MPIRG_DEBUG_PANEL
  if (t == 0 && rank == 0)
    printf("spec k0=%d rank=%d t=%d abort=%d load=%lld diag=%lld rows=%lld sync=%lld\n", k0, rank, t, sh.abort, w1 - w0,
           w2 - w1, w3 - w2, clock64() - w3);
#endif
  // verdict
  bool bad = sh.abort != 0;
  if (CS > 1)
  {
    if (warp == 0 && lane < CS)
    {
      const uint32_t v = bad ? 1u : 0u;
      asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(
                       mapa(smem_addr(&sh.verdict[rank]), (uint32_t)lane)),
                   "r"(v)
                   : "memory");
    }
    cluster_sync_all();
    bad = false;
    for (int i = 0; i < CS; ++i)
      bad |= sh.verdict[i] != 0u;
  }
  if (bad)
  {
    __syncthreads();  // every thread has read the verdicts before the panel is staged over them
    return false;
  }
  // clean: write the panel back; ipiv = identity, no row moves
#pragma unroll
  for (int q = 0; q < NR; ++q)
    if (act[q])
    {
#pragma unroll 8
      for (int c = 0; c < NB; ++c)
        A[(size_t)(k0 + c) * n + row[q]] = panel_out<TG, float>(stash[(size_t)(q * NB + c) * NTX]);
    }
  if (rank == 0)
  {
    for (int idx = t; idx < NB * NB; idx += NTX)
    {
      const int c = idx / NB, r = idx - c * NB;
      A[(size_t)(k0 + c) * n + k0 + r] = panel_out<TG, float>(c >= r ? sh.U[r][c] : sh.Dg[r][c]);
    }
    if (t < NB)
      ipiv[k0 + t] = k0 + t;
    if (t == 0 && sh.zj < NB)
      atomicMin(&info->singular_col, k0 + sh.zj);
  }
  return true;
}

template <typename T, int NB, int RPT, int NTX = NT, typename TG = T>
__global__ void __launch_bounds__(NTX, 1)
    lu_panel2_kernel(TG *__restrict__ A, int n, int k0, int jb, int *__restrict__ ipiv,
                     int2 *__restrict__ moves, int *__restrict__ nmoves, DevInfo *info,
                     int spec_ok, BatchStride bs)
{
  constexpr int NT = NTX;  // hides the namespace default inside this kernel
  pdl_trigger();
  pdl_wait();
  A += (size_t)blockIdx.z * bs.a;
  ipiv += (size_t)blockIdx.z * bs.vec;
  moves += (size_t)blockIdx.z * bs.moves;
  nmoves += (size_t)blockIdx.z * bs.nm;
  info += (size_t)blockIdx.z * bs.info;
  constexpr int NW = NTX / 32;
  static_assert(NW <= 32 && NW * 2 >= MAXCS, "push mapping needs 2*NW >= MAXCS");
  using S = Slot<T>;
  constexpr int R = RPT * NT;
  constexpr bool WIDE = sizeof(T) > 4;
  constexpr unsigned long long FORCED = WIDE ? ~0ull : 0xFFFFFFFFull;
  static_assert(sizeof(S) % 16 == 0, "slot must be a multiple of 16 bytes");
  static_assert(NB % IB == 0, "NB must be a multiple of IB");
  __shared__ WSlot<T> wslot[2][NW];  // double-buffered: a slow reader of step j never sees j+1
  __shared__ S inbox[2][MAXCS];      // every CTA's candidate (st.async from the peers)
  // [0],[1]: exchange-step inboxes, [2]: block exchange, [3],[4]: block
  // verification flags, [5 + jj]: speculative step jj of a block
  // [6]: a clean speculative block's pivot rows, right columns (raw)
  __shared__ __align__(8) uint64_t bars[7];
  __shared__ BMsg<T> binbox;               // speculative block: its IB pivot rows
  __shared__ BMsg<T> bstage;               // the owner warp's staged message
  __shared__ __align__(16) T Ubs[IB][NB];  // clean speculative block: pivot rows as of block start
  __shared__ int spec_clean_s;
  __shared__ uint32_t vflag[2][MAXCS];     // every CTA's "speculation beaten" flag
  __shared__ int cta_beaten;
  __shared__ int piv_rank[IB], piv_lrow[IB];  // owner CTA / local row of the block's pivots
  extern __shared__ __align__(16) unsigned char dsm[];
  T *P = reinterpret_cast<T *>(dsm);                                     // [NB][R]
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
  // Whole-panel speculation first (see above); a clean panel ends here.
  int spec_skip = 0;
  if constexpr (whole_spec_eligible<T, NB, RPT, NTX>())
  {
    // DevInfo::pad: panels still to skip (low byte) | back-off level (next
    // byte): consecutive beaten panels make the next 0, 1, 3, 7 panels not try
    // (level 1, 2, 4, 8), a clean one resets the level -- an isolated
    // interchange (cfg 2a has one every ~7 panels) costs no skipped panel, a
    // pivot-heavy matrix (cfg 4) tries one panel in eight. Every CTA reads it
    // before anyone writes it (kernel end).
    spec_skip = info->pad;
    if ((spec_ok & 2) && (spec_skip & 0xff) == 0 && jb == NB)
    {
      if (whole_panel_spec<NB, 2, NTX, TG>(A, n, k0, dsm, ipiv, info, CS, rank))
      {
        if (rank == 0 && t == 0 && spec_skip != 0)
          info->pad = 0;
        return;
      }
      const int level = min(max(2 * (spec_skip >> 8), 1), kSpecSkip);
      spec_skip = -((level << 8) | (level - 1));  // beaten: negative = store at kernel end
    }
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
        tmp[u][q] = (pos[q] >= 0 && c0 + u < jb)
                        ? panel_in<T, TG>(A[(size_t)(k0 + c0 + u) * n + pos[q]])
                        : T{};
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (c0 + u < NB)
          P[(c0 + u) * R + t + q * NT] = tmp[u][q];
  }
  const bool multi = CS > 1;
  // Bytes my inbox receives per step: one message from each of the CS CTAs.
  const uint32_t step_bytes = (uint32_t)(CS * sizeof(S));
  if (t == 0 && multi)
  {
    for (int i = 0; i < 7; ++i)
      mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // Arm every first phase before any peer can send: the exchange steps'
    // two parities, both verdict parities, the speculative block message.
    mbar_expect_tx(&bars[0], step_bytes);
    mbar_expect_tx(&bars[1], step_bytes);
    mbar_expect_tx(&bars[3], (uint32_t)(CS * 4));
    mbar_expect_tx(&bars[4], (uint32_t)(CS * 4));
    mbar_expect_tx(&bars[5], (uint32_t)sizeof(BMsg<T>));
  }
  if (t == 0)
    cta_beaten = 0;
  if (t < IB)
    piv_rank[t] = -1;
  if (multi)
    cluster_sync_all();
  else
    __syncthreads();

  // Warp w pushes this CTA's candidate to CTAs w and w + NW (slot rank there).
  uint32_t push_dst[2][2] = {{0u, 0u}, {0u, 0u}}, push_bar[2][2] = {{0u, 0u}, {0u, 0u}};
  if (multi)
  {
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int e = 0; e < 2; ++e)
      {
        const int d = warp + e * NW;
        if (d < CS)
        {
          push_dst[par][e] = mapa(smem_addr(&inbox[par][rank]), d);
          push_bar[par][e] = mapa(smem_addr(&bars[par]), d);
        }
      }
  }

#ifdef MPIRG_DEBUG_PANEL
  long long ptacc[16] = {};
  long long ptlast = clock64();
#endif
  T cur[RPT][IB];  // current block columns (registers, static indices)
  int step = 0;    // exchange steps so far (inbox parity / phase bookkeeping)
  int vblk = 0;    // speculative block messages so far (bars[5] phase)
  int nverd = 0;   // verdict exchanges so far (bars[3 + parity] phases)
  int nbx = 0;     // block-end exchanges so far (bars[2] phases)
  int nrc = 0;     // speculative right-column messages so far (bars[6] phases)
  int skip = 0, backoff = 0;  // speculation back-off after a beaten block
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
    // right-column chunks of one pivot row, from the chunk-aligned jb0 + IB on
    const int rch = (int)(((size_t)(NB - (jb0 + IB)) * sizeof(T) + 15) / 16);
    // (piv_rank is reset at the previous block's end / kernel start)
    // Arm the block exchange before this CTA sends any step message of the
    // block: a peer sends block data only after every CTA's last step message.
    const bool try_spec = multi && (spec_ok & 1) && skip == 0 && jb0 + IB <= jb;
    // (a speculative block arms it at block end, only if it is beaten)
    if (t == 0 && multi && bend < jb && !try_spec)
      mbar_expect_tx(&bars[2], (uint32_t)((bend - jb0) * rch * 16));

    // ---- speculative block: assume every pivot of the block is the row
    // already at position k (no row interchange). The CTA that naturally
    // holds positions [k, k+IB) factors those IB rows among themselves (a
    // small LU on IB lanes of one warp) and pushes the IB finished pivot rows
    // to every CTA in ONE message; every CTA then runs the block's IB steps
    // locally, checking that no row below a pivot beats it (|a| strictly
    // larger; NaN never), and the verdicts are exchanged once per block. A
    // beaten block is restored and redone with the exchange steps below --
    // the result is the reference's either way. If the natural rows are not
    // in place (an earlier interchange moved them) the message says so and
    // the block takes the exchange steps directly.
    bool spec_done = false;
    bool rc_pushed = false;  // this block's right columns came with the block message
    if (!try_spec && skip > 0)
      --skip;
    if (try_spec)
    {
      const int kb = k0 + jb0;                   // first position of the block
      const int orank = (kb - k0) / R;           // CTA naturally holding [kb, kb+IB)
      const int oidx = kb - k0 - orank * R;      // = t0 + q0 * NT
      const int t0 = oidx % NT, q0 = oidx / NT;
      if (rank == orank)
      {
        // the owner warp decides whether the natural rows are in place; the
        // other warps of the owner CTA then push the pivot rows' right
        // columns (raw, as of block start) to every CTA while it factors the
        // block part -- the block-end exchange is then not needed
        if (warp == t0 / 32)
        {
          const int li = lane - (t0 & 31);
          bool inplace = false;
#pragma unroll
          for (int q = 0; q < RPT; ++q)
            if (q == q0)
              inplace = li >= 0 && li < IB && pos[q] == kb + li;
          const bool cl = __popc(__ballot_sync(0xffffffffu, inplace)) == IB;
          if (lane == 0)
            spec_clean_s = cl ? 1 : 0;
        }
        __syncthreads();
      }
      if (rank == orank && warp != t0 / 32 && spec_clean_s && bend < jb)
      {
        constexpr int EPC = 16 / sizeof(T);
        const int c_lo = jb0 + IB;
        const int wi = warp < t0 / 32 ? warp : warp - 1;
        const int per_row = CS * rch;
        for (int idx = wi * 32 + lane; idx < IB * per_row; idx += (NW - 1) * 32)
        {
          const int jj = idx / per_row, rem = idx - jj * per_row;
          const int dst = rem / rch, ch = rem - dst * rch;
          T e[EPC];
#pragma unroll
          for (int w = 0; w < EPC; ++w)
          {
            const int c = c_lo + ch * EPC + w;
            e[w] = c < jb ? P[c * R + oidx + jj] : T{};
          }
          st_async_v4(mapa(smem_addr(&Ubs[jj][c_lo]) + ch * 16, (uint32_t)dst),
                      *reinterpret_cast<const uint4 *>(e),
                      mapa(smem_addr(&bars[6]), (uint32_t)dst));
        }
      }
      if (rank == orank && warp == t0 / 32)
      {
        const int li = lane - (t0 & 31);  // 0..IB-1 on the block's lanes
        const bool mine = li >= 0 && li < IB;
        T rv[IB];
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          if (q == q0)
          {
#pragma unroll
            for (int c = 0; c < IB; ++c)
              rv[c] = cur[q][c];
          }
        const bool clean = spec_clean_s != 0;
        if (clean)
        {
          // IB-step LU of the block's pivot rows (reference order per element)
#pragma unroll
          for (int jj = 0; jj < IB; ++jj)
          {
            T u[IB];
#pragma unroll
            for (int c = jj; c < IB; ++c)
              u[c] = shfl_t(rv[c], (t0 & 31) + jj);
            if (mine && li > jj)
            {
              const T l = divide(rv[jj], u[jj]);
              rv[jj] = l;
#pragma unroll
              for (int c = jj + 1; c < IB; ++c)
                rv[c] = upd(rv[c], l, u[c]);
            }
          }
          if (mine)
          {
#pragma unroll
            for (int c = 0; c < IB; ++c)
              bstage.blk[li][c] = rv[c];
          }
        }
        if (lane == 0)
          bstage.flag = clean ? 1u : 0u;
        __syncwarp();
        constexpr int NCH = sizeof(BMsg<T>) / 16;
        const uint4 *src = reinterpret_cast<const uint4 *>(&bstage);
        const uint32_t dst0 = smem_addr(&binbox), bar0 = smem_addr(&bars[5]);
        for (int idx = lane; idx < NCH * CS; idx += 32)
        {
          const int d = idx / NCH, ch = idx - d * NCH;
          st_async_v4(mapa(dst0, (uint32_t)d) + ch * 16, src[ch], mapa(bar0, (uint32_t)d));
        }
      }
      PT_MARK(12);
      mbar_wait(&bars[5], (uint32_t)(vblk & 1));
      PT_MARK(13);
      // re-arm for the next block message: its sender must first pass this
      // block's verdict exchange or exchange steps, which need this CTA
      if (t == 0)
        mbar_expect_tx(&bars[5], (uint32_t)sizeof(BMsg<T>));
      const bool clean = binbox.flag != 0u;
      ++vblk;
      if (clean && bend < jb)
      {
        rc_pushed = true;
        if (t == 0)
          mbar_expect_tx(&bars[6], (uint32_t)(IB * rch * 16));
      }
      if (clean)
      {
        bool beaten = false;
        int zj = IB;  // first step whose pivot is exactly zero
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
        {
          const int k = kb + jj;
          const T piv = binbox.blk[jj][jj];
          const bool pnan = is_nan_t(piv);
          const unsigned long long skey = pnan ? FORCED : mag_key(piv);
          if (!pnan && skey == 1ull)
            zj = min(zj, jj);
          if (t < IB)
            Ub[jj * NB + jb0 + t] = binbox.blk[jj][t];
          T ub[IB];
#pragma unroll
          for (int c = jj + 1; c < IB; ++c)
            ub[c] = binbox.blk[jj][c];
#pragma unroll
          for (int q = 0; q < RPT; ++q)
          {
            if (pos[q] == k)
            {
#pragma unroll
              for (int c = 0; c < IB; ++c)
                cur[q][c] = binbox.blk[jj][c];
              chosen[q] = jj;
              piv_rank[jj] = rank;
              piv_lrow[jj] = t + q * NT;
            }
            else if (pos[q] > k)
            {
              const T v = cur[q][jj];
              if (!is_nan_t(v) && mag_key(v) > skey)
                beaten = true;
              const T l = divide(v, piv);
              cur[q][jj] = l;
#pragma unroll
              for (int c = jj + 1; c < IB; ++c)
                cur[q][c] = upd(cur[q][c], l, ub[c]);
            }
          }
        }
        if (rc_pushed)
        {
          // take the pivot rows' right columns out of Ubs before the verdict
          // goes out: the owner of the next block writes Ubs only after it
          // has every CTA's verdict
          mbar_wait(&bars[6], (uint32_t)(nrc & 1));
          ++nrc;
          for (int idx = t; idx < IB * (jb - bend); idx += NT)
          {
            const int jj = idx / (jb - bend), c = bend + idx % (jb - bend);
            Ub[jj * NB + c] = Ubs[jj][c];
          }
        }
        PT_MARK(14);
        // verdict exchange (one word per CTA)
        if (__any_sync(0xffffffffu, beaten) && lane == 0)
          cta_beaten = 1;
        __syncthreads();
        const int vp = nverd & 1;
        if (warp == 0 && lane < CS)
        {
          const uint32_t v = (uint32_t)cta_beaten;
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                  mapa(smem_addr(&vflag[vp][rank]), (uint32_t)lane)),
              "r"(v), "r"(mapa(smem_addr(&bars[3 + vp]), (uint32_t)lane))
              : "memory");
        }
        mbar_wait(&bars[3 + vp], (uint32_t)((nverd >> 1) & 1));
        ++nverd;
        const bool any_beaten =
            __any_sync(0xffffffffu, lane < CS ? vflag[vp][lane] != 0u : false);
        __syncthreads();  // everyone has read vflag[vp] and cta_beaten
        if (t == 0)
        {
          mbar_expect_tx(&bars[3 + vp], (uint32_t)(CS * 4));  // for the verdict two blocks on
          cta_beaten = 0;
        }
        PT_MARK(15);
        if (!any_beaten)
        {
          spec_done = true;
          backoff = 0;
          if (rank == 0 && t < IB)
            ipiv[kb + t] = kb + t;
          if (rank == 0 && t == 0 && zj < IB)
            atomicMin(&info->singular_col, kb + zj);
        }
        else
        {
          // P still holds the block columns as of the block start
#pragma unroll
          for (int q = 0; q < RPT; ++q)
          {
            chosen[q] = IB;
#pragma unroll
            for (int jj = 0; jj < IB; ++jj)
              cur[q][jj] = P[(jb0 + jj) * R + t + q * NT];
          }
          if (t < IB)
            piv_rank[t] = -1;
          backoff = backoff ? min(2 * backoff, 8) : 1;
          skip = backoff;
          __syncthreads();  // piv_rank reset before the exchange steps set it
        }
      }
    }

#pragma unroll
    for (int jj = 0; jj < IB; ++jj)
    {
      const int j = jb0 + jj;
      if (j >= jb || spec_done)
        break;
      const int k = k0 + j;
      const int par = step & 1;

      // 1. thread-local candidate among unchosen rows (positions >= k). A NaN
      //    is never chosen, except that a NaN at position k keeps p = k
      //    (dense_lu.hpp:65-78): that row takes the FORCED key, above any |a|.
      unsigned long long bkey = 0ull;
      int bp = INT_MAX, bq = 0, nan = 0;
#pragma unroll
      for (int q = 0; q < RPT; ++q)
      {
        if (pos[q] >= k)
        {
          if (is_nan_t(cur[q][jj]))
          {
            if (pos[q] == k)
            {
              nan = 1;
              bkey = FORCED;
              bp = k;
              bq = q;
            }
          }
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
      PT_MARK(0);
      // 2. warp argmax: max |a|, then min position among ties.
      unsigned long long wkey;
      int wpos;
      argmax_redux<WIDE>(bkey, bp, wkey, wpos);
      nan = __any_sync(0xffffffffu, nan);
      // 3. the warp winner stages key, position, block columns, local row id.
      const bool owner = bkey != 0ull && bkey == wkey && bp == wpos;
      if (owner || (lane == 0 && wkey == 0ull))
      {
        WSlot<T> &ws = wslot[par][warp];
        ws.key = wkey;
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
      PT_MARK(1);
      __syncthreads();
      PT_MARK(2);
      // 4. CTA winner over the warp slots (every warp computes it redundantly).
      const unsigned long long ck0 = lane < NW ? wslot[par][lane].key : 0ull;
      const int cp0 = lane < NW ? wslot[par][lane].pos : INT_MAX;
      unsigned long long ckey;
      int cpos;
      argmax_redux<WIDE>(ck0, cp0, ckey, cpos);
      const int cw = __ffs(__ballot_sync(0xffffffffu, lane < NW && ck0 == ckey &&
                                                          (ckey == 0ull || cp0 == cpos))) -
                     1;
      const int cn = __any_sync(0xffffffffu, lane < NW ? wslot[par][lane].nan : 0);
      if (ckey == 0ull)
        cpos = INT_MAX;
      PT_MARK(3);
      // 5. push the CTA candidate [key|pos|nan|block columns] to every CTA:
      //    warp w sends to CTAs w, w+NW; lane l sends 16-byte chunk l (st.async
      //    completes bytes on the receiver's mbarrier).
      const S *U = nullptr;
      const T *Ublk;
      int gr = rank;
      unsigned long long gkey = ckey;
      int gp = cpos, gn = cn;
      constexpr int NCH = sizeof(S) / 16;
      if (multi && lane < NCH)
      {
        const WSlot<T> &ws = wslot[par][cw];
        uint4 val;
        if (lane == 0)
          val = make_uint4((uint32_t)ckey, (uint32_t)(ckey >> 32), (uint32_t)cpos, (uint32_t)cn);
        else
          val = reinterpret_cast<const uint4 *>(ws.blk)[lane - 1];
        for (int d = warp; d < CS; d += NW)
          st_async_v4(push_dst[par][d >= NW] + lane * 16, val, push_bar[par][d >= NW]);
      }
      PT_MARK(4);
      if (multi)
      {
        // 6. wait until all CS candidates are in my inbox, then re-arm the
        //    barrier for step+2 (no peer can send step+2 data before every CTA,
        //    this one included, has pushed step+1).
        mbar_wait(&bars[par], (uint32_t)((step >> 1) & 1));
        if (t == 0)
          mbar_expect_tx(&bars[par], step_bytes);  // for exchange step + 2
        PT_MARK(5);
        // 7. global winner (identical in every thread of every CTA).
        const unsigned long long gk0 = lane < CS ? inbox[par][lane].key : 0ull;
        const int gp0 = lane < CS ? inbox[par][lane].pos : INT_MAX;
        argmax_redux<WIDE>(gk0, gp0, gkey, gp);
        gr = __ffs(__ballot_sync(0xffffffffu, lane < CS && gk0 == gkey &&
                                                  (gkey == 0ull || gp0 == gp))) -
             1;
        gn = __any_sync(0xffffffffu, lane < CS ? inbox[par][lane].nan : 0);
        U = &inbox[par][gr];
        Ublk = U->blk;
      }
      else
        Ublk = wslot[par][cw].blk;  // one CTA: its winner is the pivot
      const int p = gn ? k : gp;
      if (rank == 0 && t == 0)
      {
        ipiv[k] = p;
        if (!gn && gkey == 1ull)  // |pivot| == +0 (key of +0.0)
          atomicMin(&info->singular_col, k);
      }
      (void)U;
      // the pivot row's block columns (its right columns come at block end)
      if (t < IB)
        Ub[jj * NB + jb0 + t] = Ublk[t];
      const T piv = Ublk[jj];
      T ub[IB];
#pragma unroll
      for (int c = jj + 1; c < IB; ++c)
        ub[c] = Ublk[c];
      PT_MARK(6);
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
            piv_rank[jj] = rank;
            piv_lrow[jj] = t + q * NT;
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
      PT_MARK(7);
    }

    // ---- block end: apply the block's rank-1 updates to the columns right
    // of the block, in step order.
    PT_MARK(9);
    __syncthreads();  // block columns of Ub, piv_rank / piv_lrow final
    const int nb_here = bend - jb0;
    if (bend < jb)
    {
      // the block's pivot rows, right columns as of the block start (P is
      // only updated at block end), from their owners to every CTA
      const int c_lo = jb0 + IB;
      constexpr int EPC = 16 / sizeof(T);
      if (multi && spec_done)
      {
        // the pivot rows' right columns came with the block message
      }
      else if (multi)
      {
        if (try_spec && t == 0)  // a beaten speculative block: arm the exchange now
          mbar_expect_tx(&bars[2], (uint32_t)((bend - jb0) * rch * 16));
        const int per_row = CS * rch;
        for (int idx = t; idx < nb_here * per_row; idx += NT)
        {
          const int jj = idx / per_row, rem = idx - jj * per_row;
          if (piv_rank[jj] != rank)
            continue;
          const int dst = rem / rch, ch = rem - dst * rch;
          const int lrow = piv_lrow[jj];
          T e[EPC];
#pragma unroll
          for (int w = 0; w < EPC; ++w)
          {
            const int c = c_lo + ch * EPC + w;
            e[w] = c < jb ? P[c * R + lrow] : T{};
          }
          st_async_v4(mapa(smem_addr(Ub + jj * NB + c_lo) + ch * 16, dst),
                      *reinterpret_cast<const uint4 *>(e), mapa(smem_addr(&bars[2]), dst));
        }
        mbar_wait(&bars[2], (uint32_t)(nbx & 1));
        ++nbx;
      }
      else
      {
        for (int idx = t; idx < nb_here * (jb - bend); idx += NT)
        {
          const int jj = idx / (jb - bend), c = bend + idx % (jb - bend);
          Ub[jj * NB + c] = P[c * R + piv_lrow[jj]];
        }
        __syncthreads();
      }
    }
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
    // piv_rank's last readers are behind this barrier; the next block's first
    // writers are behind the block's final one
    if (t < IB)
      piv_rank[t] = -1;
    PT_MARK(10);
    // (b) every row: its right columns get the updates of the steps at which it
    //     was still below the pivot (all IB for non-pivot rows). Four columns
    //     at a time: independent FMA chains, vector loads of Ub.
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
      T lq[IB];
#pragma unroll
      for (int jj = 0; jj < IB; ++jj)
        lq[jj] = jj < upto ? cur[q][jj] : T{};
      int c = bend;
      for (; c + 4 <= jb; c += 4)
      {
        T v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = P[(c + e) * R + r];
        T ubv[IB][4];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            ubv[jj][e] = Ub[jj * NB + c + e];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
          if (jj < upto)
          {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              v[e] = upd(v[e], lq[jj], ubv[jj][e]);
          }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          P[(c + e) * R + r] = v[e];
      }
      for (; c < jb; ++c)
      {
        T v = P[c * R + r];
#pragma unroll
        for (int jj = 0; jj < IB; ++jj)
          if (jj < upto)
            v = upd(v, lq[jj], Ub[jj * NB + c]);
        P[c * R + r] = v;
      }
    }
    __syncthreads();
    PT_MARK(11);
  }

  PT_MARK(8);
#ifdef MPIRG_DEBUG_PANEL
  if (t == 0 && rank == 0 && (k0 == 0 || k0 + jb >= n))
    printf("panel k0=%d CS=%d spec_blocks=%d steps=%d cycles/step: cand %lld warp %lld sync %lld cta %lld push %lld "
           "wait %lld glob %lld upd %lld | per panel: (a) %lld (b) %lld | spec per blk: owner+push %lld wait %lld local %lld verdict %lld\n",
           k0, CS, vblk, step, ptacc[0] / max(step, 1), ptacc[1] / max(step, 1), ptacc[2] / max(step, 1), ptacc[3] / max(step, 1),
           ptacc[4] / max(step, 1), ptacc[5] / max(step, 1), ptacc[6] / max(step, 1), ptacc[7] / max(step, 1), ptacc[10],
           ptacc[11], ptacc[12] / max(vblk, 1), ptacc[13] / max(vblk, 1), ptacc[14] / max(vblk, 1), ptacc[15] / max(vblk, 1));
#endif
  // Write every row to its final position; record the row moves.
#pragma unroll
  for (int q = 0; q < RPT; ++q)
  {
    if (pos[q] >= 0)
    {
      const int g = row0 + t + q * NT;
      for (int c = 0; c < jb; ++c)
        A[(size_t)(k0 + c) * n + pos[q]] = panel_out<TG, T>(P[c * R + t + q * NT]);
      if (pos[q] != g)
      {
        const int e = atomicAdd(nmoves, 1);
        moves[e] = make_int2(pos[q], g);
      }
    }
  }
  if (multi)
  {
    cluster_sync_all();  // no CTA may exit while peers can still write its inbox
  }
  if constexpr (whole_spec_eligible<T, NB, RPT, NTX>())
  {
    if (rank == 0 && t == 0)
    {
      if (spec_skip < 0)
        info->pad = -spec_skip;
      else if ((spec_skip & 0xff) != 0)
        info->pad = spec_skip - 1;
    }
  }
}

}  // namespace panel2
}  // namespace mpirg
