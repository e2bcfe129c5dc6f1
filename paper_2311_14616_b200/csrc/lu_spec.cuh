// Whole-panel speculation of the LU panel kernel (lu_panel.cuh): the pure
// compute parts (no cluster / global-memory protocol), also built stand-alone
// by tools/ubench/panel_spec.cu.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace mpirg
{
namespace panel2
{

constexpr int MAXCS = 16;
__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// Candidate key of |a| (a non-NaN): its IEEE bits + 1, so 0 means "none" and
// the unsigned order is the numeric order of the (non-negative) magnitudes.
__device__ __forceinline__ unsigned long long mag_key(float a)
{
  return (unsigned long long)__float_as_uint(fabsf(a)) + 1ull;
}
__device__ __forceinline__ unsigned long long mag_key(double a)
{
  return (unsigned long long)__double_as_longlong(fabs(a)) + 1ull;
}
__device__ __forceinline__ unsigned long long mag_key(h16 a) { return mag_key(h2f(a)); }
__device__ __forceinline__ bool is_nan_t(float a) { return isnan(a); }
__device__ __forceinline__ bool is_nan_t(double a) { return isnan(a); }
__device__ __forceinline__ bool is_nan_t(h16 a) { return (a.bits & 0x7c00u) == 0x7c00u && (a.bits & 0x3ffu); }

// ---------------------------------------------------------------------------
// Whole-panel speculation (binary32 arithmetic, NB = 64, one or two rows per
// thread). If every pivot of the panel is the row already at its position --
// no interchange in NB columns, the rule for the diagonally dominant operators
// of configs 1-3 and 5 -- then the panel decouples: the NB x NB diagonal block
// is an LU without pivoting that needs nothing from the rows below it, and
// every row below is its own recurrence against that block's U rows,
//   l_ik = a_ik / u_kk,  a_ic = fma(-l_ik, u_kc, a_ic) (c > k),  k = 0 .. NB-1,
// the reference's per-element order (dense_lu.hpp:87-107). So nothing has to
// cross CTAs until the verdict:
//  * warp 0 of EVERY CTA factors the diagonal block itself (redundantly; lane l
//    holds rows l and l + 32 in registers, all NB steps unrolled) and leaves
//    each finished U row and a progress count in shared memory;
//  * every thread runs its row(s) through the NB steps in registers, eight
//    steps at a time as the U rows appear, checking at each step that its
//    entry does not beat the pivot (|a| strictly larger, NaN never:
//    dense_lu.hpp:65-78);
//  * one cluster-wide verdict; a clean panel is written back with ipiv =
//    identity and no row moves, a beaten one leaves A untouched and the kernel
//    goes on to the exchange algorithm below (after a beaten panel the next
//    kSpecSkip panels do not try: DevInfo::pad counts them down).
// The divisions are l = RN(a/u) by the verified double-word reciprocal of
// trsv.cu (q = fma(a, yh, a*yl), kept only if one Markstein step leaves it
// unchanged and a, u are in range; anything else takes div.rn on the spot), so
// a kept result is the reference's bit for bit.
// ---------------------------------------------------------------------------
constexpr int kSpecSkip = 8;

template <typename T, int NB, int RPT, int NTX>
constexpr bool whole_spec_eligible()
{
  return std::is_same<T, float>::value && NB == 64 && RPT == 1 && NTX == 256;
}

struct SpecDiv
{
  float piv, yh, yl;
  bool ok;  // divisor inside the verified range
};
__device__ __forceinline__ SpecDiv spec_div_make(float piv)
{
  SpecDiv d;
  d.piv = piv;
  d.yh = __frcp_rn(piv);
  d.yl = __fmul_rn(__fmaf_rn(-piv, d.yh, 1.0f), d.yh);
  d.ok = exp_mid_f(piv);
  return d;
}
// l = a / piv by the double-word reciprocal; `bad` is raised when the quotient
// cannot be certified as RN(a / piv) (it failed the Markstein fixed-point test,
// or an operand is zero / outside the range where no intermediate underflows):
// the panel is then treated as beaten and redone by the exchange algorithm,
// which divides with div.rn. Certified quotients are the reference's bit for
// bit (trsv.cu diag_bwd4 has the argument); on random operands 2e-8 of the
// divisions fail, i.e. about one 4096 x 64 panel in 200.
__device__ __forceinline__ float spec_div(float a, const SpecDiv &d, bool act, bool &bad)
{
  const float q = __fmaf_rn(a, d.yh, __fmul_rn(a, d.yl));
  const float v = __fmaf_rn(__fmaf_rn(-d.piv, q, a), d.yh, q);
  // an exactly zero numerator (structural zeros are common: the first and last
  // rows of G are zero) divides to a zero whose sign is the product's
  const bool zero = a == 0.0f;
  bad |= act && !(d.ok && (zero || (v == q && exp_mid_f(a))));
  return zero ? __fmul_rn(a, d.piv) : q;
}

template <int NB>
struct SpecShared
{
  __align__(16) float U[NB][NB];   // U[k][c], c >= 8 (k / 8): pivot row k
  __align__(16) float Dg[NB][NB];  // the finished diagonal block (rank 0 writes it back)
  volatile int prog;               // pivot rows published so far (multiples of 8)
  volatile int abort;              // some thread of this CTA saw a pivot beaten
  int zj;                          // first exactly-zero pivot
  uint32_t verdict[MAXCS];         // every CTA's flag (remote stores, then the cluster barrier)
};

// Dynamic shared memory of the speculative pass: SpecShared + every thread's
// finished row(s), stash[(q NB + c) NTX + t].
template <int NB, int RPT, int NTX>
__host__ __device__ constexpr size_t spec_dyn_smem()
{
  return a16(sizeof(SpecShared<NB>)) + sizeof(float) * (size_t)RPT * NB * NTX;
}

__device__ __forceinline__ void ld8(float (&d)[8], const float *p)
{
  const float4 a = *reinterpret_cast<const float4 *>(p), b = *reinterpret_cast<const float4 *>(p + 4);
  d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = a.w, d[4] = b.x, d[5] = b.y, d[6] = b.z, d[7] = b.w;
}
// st8 under a predicate, without a branch (the owner lane's row publication)
__device__ __forceinline__ void st8_if(bool pred, float *p, const float (&d)[8])
{
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %0, 0;\n\t"
      "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n\t"
      "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};\n\t}\n" ::"r"((int)pred),
      "r"(a), "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7]));
  // (no memory clobber: the step's __syncwarp orders these stores against the
  // loads that read them; a clobber here would also pin every other load and
  // store of the step in place)
}
__device__ __forceinline__ void st8(float *p, const float (&d)[8])
{
  *reinterpret_cast<float4 *>(p) = make_float4(d[0], d[1], d[2], d[3]);
  *reinterpret_cast<float4 *>(p + 4) = make_float4(d[4], d[5], d[6], d[7]);
}

// The code is a rolled loop over the eight-column blocks of the panel with the
// row's blocks ROTATED through the registers (block 0 is always the current
// one), because a fully unrolled 64-step recurrence is ~100 KB of straight-line
// SASS that every warp runs once: it was measured instruction-fetch bound at
// ~2500 cycles per step.
//
// A thread's rows against one block of eight pivot rows, as soon as that block
// is published (eager: when the last pivot block appears only its own eight
// steps are left). The row lives in the thread's stash (shared memory,
// stash[(q NB + c) NTX]); block b is taken into registers for its eight steps
// (check, scale, update), then every later block b' takes the eight rank-1
// updates in step order -- per element the reference's FMA sequence.
template <int NB, int NR, int NTX>
__device__ __forceinline__ void spec_rows_block(float *stash, const bool (&act)[NR], const float (*U)[NB], int b,
                                                bool &beaten)
{
  constexpr int NBLK = NB / 8;
  float R[NR][8];
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      R[q][e] = stash[(size_t)(q * NB + 8 * b + e) * NTX];
  // the block's own steps (rows that are not `act` run on dummy values: no branch)
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
  {
    float ub[8];
    ld8(ub, &U[8 * b + kk][8 * b]);
    const float piv = ub[kk];
    const SpecDiv dv = spec_div_make(piv);
    const float pabs = fabsf(piv);
#pragma unroll
    for (int q = 0; q < NR; ++q)
    {
      const float v = act[q] ? R[q][kk] : 1.0f;
      // beaten: |v| > |piv| (false when either is NaN: a NaN is never chosen, a
      // NaN on the diagonal keeps its place -- dense_lu.hpp:65-78)
      beaten |= act[q] && fabsf(v) > pabs;
      const float l = spec_div(v, dv, act[q], beaten);
      R[q][kk] = l;
#pragma unroll
      for (int e = kk + 1; e < 8; ++e)
        R[q][e] = upd(R[q][e], l, ub[e]);
    }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      stash[(size_t)(q * NB + 8 * b + e) * NTX] = R[q][e];
  // the later blocks
#pragma unroll 1
  for (int bp = b + 1; bp < NBLK; ++bp)
  {
    float V[NR][8];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        V[q][e] = stash[(size_t)(q * NB + 8 * bp + e) * NTX];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
    {
      float uj[8];
      ld8(uj, &U[8 * b + kk][8 * bp]);
#pragma unroll
      for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          V[q][e] = upd(V[q][e], R[q][kk], uj[e]);
    }
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        stash[(size_t)(q * NB + 8 * bp + e) * NTX] = V[q][e];
  }
}

template <int NB, int NR>
__device__ __forceinline__ void spec_rotate(float (&R)[NR][NB / 8][8])
{
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int j = 0; j + 1 < NB / 8; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        R[q][j][e] = R[q][j + 1][e];
}

// The diagonal block by one warp: D[0] = row lane, D[1] = row lane + 32.
// Phase PH: the pivot rows are rows 32 PH .. 32 PH + 31 (slot PH); in phase 1
// the rows of slot 0 are finished and take no part. No lane ever branches on
// whether its row is still active: a finished row's registers just go stale --
// its U part (columns >= the row index) was published in U[row][.] when it
// became the pivot row, and its L part is kept in Dg at the end of the block
// that produced it, so the result is U (on and right of the diagonal) + Dg
// (left of it). The current block of the pivot row travels by shuffles (the
// step's critical path), its later blocks through shared memory.
template <int NB, int PH>
__device__ __forceinline__ void spec_diag_phase(float (&D)[2][NB / 8][8], SpecShared<NB> &sh, int lane,
                                                bool stash, bool &beaten, int &zj, bool &stop)
{
  constexpr int NBLK = NB / 8;
#pragma unroll 1
  for (int bb = 0; bb < 4; ++bb)
  {
    if (stop)
      break;
    const int b = 4 * PH + bb;
    const int nlive = NBLK - 1 - b;
    float *Uk0 = &sh.U[8 * b][8 * b];
    // The later-block updates of step kk run one step late, between the
    // shuffles of step kk+1 and its division: they are the bulk of the
    // instructions and are not on the step-to-step dependency (current block
    // of the next pivot row -> shuffle -> division -> in-block update), so
    // they fill that chain's latency instead of adding to it. The owner of
    // row kk+1 stores its later blocks right after they took update kk.
    // (the pivot row's later blocks are loaded in one batch at the top of the
    // step, before the shuffles: issued back to back they cost one
    // shared-memory latency, loaded block by block in front of their FMAs they
    // cost seven)
    float lprev[2] = {0.0f, 0.0f};
    float ujs[NBLK - 1][8];
    auto later_load = [&](const float *Ukp) {
#pragma unroll
      for (int j = 1; j < NBLK; ++j)
        if (j <= nlive)
          ld8(ujs[j - 1], Ukp + 8 * j);
    };
    auto later_apply = [&]() {
#pragma unroll
      for (int j = 1; j < NBLK; ++j)
        if (j <= nlive)
        {
#pragma unroll
          for (int sl = PH; sl < 2; ++sl)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              D[sl][j][e] = upd(D[sl][j][e], lprev[sl], ujs[j - 1][e]);
        }
    };
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
    {
      const int ol = 8 * bb + kk;  // owner lane of pivot row 8b + kk
      float *Uk = Uk0 + kk * NB;
      const bool own = lane == ol;
      if (kk > 0)
        later_load(Uk - NB);  // step kk-1 (its row was stored one step ago)
      float ub[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        ub[e] = e >= kk ? __shfl_sync(0xffffffffu, D[PH][0][e], ol) : 0.0f;
      if (kk > 0)
        later_apply();
      st8_if(own, Uk, D[PH][0]);
#pragma unroll
      for (int j = 1; j < NBLK; ++j)
        if (j <= nlive)
          st8_if(own, Uk + 8 * j, D[PH][j]);
      const float piv = ub[kk];
      const SpecDiv dv = spec_div_make(piv);
      const float pabs = fabsf(piv);
      if (piv == 0.0f)
        zj = min(zj, 8 * b + kk);
#pragma unroll
      for (int sl = PH; sl < 2; ++sl)
      {
        const bool act = (sl == 1 && PH == 0) || lane > ol;
        const float v = act ? D[sl][0][kk] : 1.0f;
        beaten |= act && fabsf(v) > pabs;
        const float l = spec_div(v, dv, act, beaten);
        lprev[sl] = l;
        D[sl][0][kk] = l;
#pragma unroll
        for (int e = kk + 1; e < 8; ++e)
          D[sl][0][e] = upd(D[sl][0][e], l, ub[e]);
      }
      __syncwarp();  // the owner's row is in shared memory
    }
    later_load(Uk0 + 7 * NB);  // the block's last step
    later_apply();
    // block b is final in every row still active: keep it (rank 0), rotate, publish progress
    if (stash)
    {
      if (PH == 0)
        st8(&sh.Dg[lane][8 * b], D[0][0]);
      st8(&sh.Dg[lane + 32][8 * b], D[1][0]);
    }
    spec_rotate<NB, 2>(D);
    __syncwarp();
    if (lane == 0)
    {
      __threadfence_block();
      sh.prog = 8 * (b + 1);
    }
    if (__any_sync(0xffffffffu, beaten))
    {
      if (lane == 0)
        sh.abort = 1;
      stop = true;
    }
    else if (sh.abort)
      stop = true;
  }
}

}  // namespace panel2
}  // namespace mpirg
