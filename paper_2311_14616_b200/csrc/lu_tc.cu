// K5b -- tensor-core updates for binary16 factors (lu_mode TC).
//
//   C[r0:r1, cb:ce] <- fp16( fp32(C) - L[r0:r1, k0:k0+K] * U[k0:k0+K, cb:ce] )
//
// with L, U and C all inside the one n x n column-major binary16 matrix, the
// K-term products accumulated in fp32 by the 5th-generation tensor cores and
// one rounding to binary16 per call, instead of the reference's two roundings
// per term (dense_lu.hpp:96-107 with half.hpp:285-288). This is NOT
// bit-compatible with the reference; it is the fast mode whose deviation
// SURVEY.md 8(d) discusses. The exact mode (lu.cu lu_gemm_kernel) remains the
// default. K is a multiple of 64; the recursive LU schedule (lu.cu lu_run_tc)
// calls this with K = 64 ... n/2, so most of the 2n^3/3 flops run at K >= 1024
// where the kernel is bound by the tensor pipe and its operand feed, not by
// the HBM traffic of C.
//
// Persistent, warp-specialised kernel, one CTA per SM, 12 warps:
//   warp 0      TMA producer: per 64-k stage the L tile (MT x 128 rows x 64 k,
//               MN-major, 64-row boxes) and the U tile (64 k x TN columns,
//               K-major), SWIZZLE_128B, into a ring of S stages (full/empty
//               mbarriers);
//   warp 1      MMA issuer: one thread issues 4 x MT tcgen05.mma.kind::f16
//               (M = 128, N = TN, K = 16) per stage with A negated, into TMEM
//               accumulators; tcgen05.commit frees the stage and, after the
//               last stage, publishes the accumulator;
//   warp 2      allocates / frees the 512 TMEM columns;
//   warps 4-11  epilogue (two warpgroups, warp w reads TMEM lanes 32 (w % 4) ..):
//               tcgen05.ld of 16 columns at a time, C read from and written to
//               global memory directly (a warp touches 32 consecutive rows of a
//               column, i.e. whole 32-byte sectors), fp16(C + D).
// MT = 1: 128 x TN tiles, two accumulator units, so the epilogue of one tile
// (warpgroup u) overlaps the MMAs of the next. MT = 2: 256 x 256 tiles on both
// units: per 64-k stage 64 KB of operands feed 1024 tensor cycles (64 B/clk/SM
// against 96 for MT = 1; the L2 delivers about 42 B/clk/SM chip-wide,
// B300_MICROARCH.md), used when K is large enough to amortise the exposed
// epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace mpirg
{
namespace
{
constexpr int BK = 64;             // k per pipeline stage
constexpr int TC_THREADS = 384;    // 4 control warps + 8 epilogue warps
constexpr uint32_t RING_BYTES = 192 * 1024;

template <int MT, int TN>
struct TcCfg
{
  static constexpr int TM = 128 * MT;
  static constexpr uint32_t A_BYTES = TM * BK * 2;
  static constexpr uint32_t B_BYTES = TN * BK * 2;
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (int)(RING_BYTES / STAGE) < 6 ? (int)(RING_BYTES / STAGE) : 6;
  static constexpr int NUNITS = 2 / MT;  // accumulator units (MT x TN columns each)
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE;
  static constexpr uint32_t IDESC = tc::idesc_f16_f32(128, TN, /*a_mn=*/true, /*b_mn=*/false,
                                                      /*neg_a=*/true);
  static_assert(STAGES >= 3, "pipeline depth");
  static_assert(2 * 256 >= NUNITS * MT * TN, "TMEM columns");
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

template <int MT, int TN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, h16 *__restrict__ Cmat, int n, int r0,
                   int r1, int cb, int ce, int k0, int K, int mtiles, int ntiles)
{
  using Cfg = TcCfg<MT, TN>;
  constexpr int S = Cfg::STAGES, NU = Cfg::NUNITS;
  extern __shared__ unsigned char tsm_raw[];
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  unsigned char *base = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = mtiles * ntiles, ks = K / BK;

  if (warp == 2)
    tc::tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 0)
  {
#pragma unroll
    for (int s = 0; s < S; ++s)
    {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
    {
      tc::mbar_init(&tfull[u], 1);
      tc::mbar_init(&tempty[u], 4 * MT);  // one arrival per epilogue warp of the unit
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0)
  {
    // ---- TMA producer ------------------------------------------------------
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x)
    {
      const int rt = r0 + (t % mtiles) * Cfg::TM, ct = cb + (t / mtiles) * TN;
      for (int s = 0; s < ks; ++s, ++it)
      {
        if (lane == 0)
        {
          const int st = it % S;
          tc::mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
          unsigned char *As = base + (size_t)st * Cfg::STAGE, *Bs = As + Cfg::A_BYTES;
          tc::mbar_expect_tx(&full[st], Cfg::STAGE);
#pragma unroll
          for (int c = 0; c < 2 * MT; ++c)
            tc::tma_load_2d(As + c * 8192, &mapA, &full[st], rt + 64 * c, k0 + s * BK);
          tc::tma_load_2d(Bs, &mapB, &full[st], k0 + s * BK, ct);
        }
        __syncwarp();
      }
    }
  }
  else if (warp == 1)
  {
    // ---- MMA issuer ----------------------------------------------------------
    uint32_t it = 0;
    int j = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x, ++j)
    {
      const int u = j % NU;
      if (lane == 0)
      {
        tc::mbar_wait(&tempty[u], ((j / NU) & 1) ^ 1);
        tc::fence_after();
      }
      __syncwarp();
      for (int s = 0; s < ks; ++s, ++it)
      {
        if (lane == 0)
        {
          const int st = it % S;
          tc::mbar_wait(&full[st], (it / S) & 1);
          tc::fence_after();
          const uint32_t sa = tc::smem_u32(base + (size_t)st * Cfg::STAGE);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
          {
            // B, K-major: 8-column groups 1 KB apart (SBO); K = 16 is 32 bytes into the row
            const uint64_t bd = tc::desc_sw128(sb + kk * 32, 16, 1024);
#pragma unroll
            for (int m = 0; m < MT; ++m)
            {
              // A, MN-major: 64-row atoms 8 KB apart (LBO), 8-k groups 1 KB apart (SBO);
              // K = 16 per MMA is two 8-k groups
              const uint64_t ad = tc::desc_sw128(sa + m * 16384 + kk * 2048, 8192, 1024);
              tc::mma_f16(tmem + (uint32_t)((u * MT + m) * TN), ad, bd, Cfg::IDESC,
                          (s | kk) ? 1u : 0u);
            }
          }
          tc::mma_commit(&empty[st]);  // frees the stage when these MMAs have read it
          if (s == ks - 1)
            tc::mma_commit(&tfull[u]);  // accumulator complete
        }
        __syncwarp();
      }
    }
  }
  else if (warp >= 4)
  {
    // ---- epilogue --------------------------------------------------------------
    const int g = (warp - 4) >> 2;  // warpgroup
    const int q = warp & 3;         // TMEM lane quarter this warp may read
    int j = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x, ++j)
    {
      const int u = j % NU;
      if (MT == 1 && u != g)
        continue;  // the other warpgroup's tile
      const int m = MT == 2 ? g : 0;
      const int rt = r0 + (t % mtiles) * Cfg::TM, ct = cb + (t / mtiles) * TN;
      {
        // while the tile's MMAs run, pull its C values towards L2: this warp's
        // 32 rows of a column are 64 contiguous bytes (rows are 32-aligned)
        const int prow = rt + m * 128 + q * 32;
        if (prow < r1)
          for (int c = lane; c < TN; c += 32)
            if (ct + c < ce)
            {
              const h16 *pc = Cmat + (size_t)(ct + c) * n + prow;
              asm volatile("prefetch.global.L2 [%0];" ::"l"(pc));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + 16));
            }
      }
      tc::mbar_wait(&tfull[u], (j / NU) & 1);
      tc::fence_after();
      const int row = rt + m * 128 + q * 32 + lane;
      const bool rok = row < r1;
      const uint32_t taddr = tmem + (uint32_t)((u * MT + m) * TN) + ((uint32_t)(q * 32) << 16);
      h16 *crow = Cmat + row;
#pragma unroll 1
      for (int c16 = 0; c16 < TN; c16 += 16)
      {
        h16 cv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
        {
          const int col = ct + c16 + e;
          cv[e] = (rok && col < ce) ? crow[(size_t)col * n] : h16{0};
        }
        float v[16];
        tc::tmem_ld16(taddr + c16, v);
#pragma unroll
        for (int e = 0; e < 16; ++e)
        {
          const int col = ct + c16 + e;
          if (rok && col < ce)
            crow[(size_t)col * n] = f2h(__fadd_rn(h2f(cv[e]), v[e]));
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0)
        mbar_arrive(&tempty[u]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2)
    tc::tmem_dealloc(tmem, 512);
}

void encode(CUtensorMap *map, void *a, int n, int box0, int box1)
{
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = tma_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a, dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed for the TC trailing update");
}

int sm_count()
{
  static int v[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  int &c = v[d & 63];
  if (c == 0)
    MPIRG_CUDA_CHECK(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d));
  return c;
}

template <int MT, int TN>
void launch_cfg(const TcPlan &p, const CUtensorMap &mapB, int r0, int r1, int cb, int ce, int k0,
                int K, cudaStream_t s)
{
  using Cfg = TcCfg<MT, TN>;
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(tc_gemm_kernel<MT, TN>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)Cfg::SMEM));
    configured.done();
  }
  const int mtiles = (r1 - r0 + Cfg::TM - 1) / Cfg::TM, ntiles = (ce - cb + TN - 1) / TN;
  const int grid = std::min(mtiles * ntiles, sm_count());
  tc_gemm_kernel<MT, TN><<<grid, TC_THREADS, Cfg::SMEM, s>>>(
      *reinterpret_cast<const CUtensorMap *>(p.mapA), mapB, static_cast<h16 *>(p.a), p.n, r0, r1,
      cb, ce, k0, K, mtiles, ntiles);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}
}  // namespace

bool tc_update_supported(int n, int nb) { return nb == BK && n % 8 == 0 && n >= BK; }

void tc_plan_make(TcPlan &p, void *a, int n)
{
  static_assert(sizeof(CUtensorMap) <= sizeof(p.mapA), "tensor map storage");
  encode(reinterpret_cast<CUtensorMap *>(p.mapA), a, n, 64, 64);
  encode(reinterpret_cast<CUtensorMap *>(p.mapB), a, n, 64, 256);
  encode(reinterpret_cast<CUtensorMap *>(p.mapB128), a, n, 64, 128);
  encode(reinterpret_cast<CUtensorMap *>(p.mapB64), a, n, 64, 64);
  p.a = a;
  p.n = n;
}

// rows [r0, r1) x columns [cb, ce) -= L[:, k0 .. k0+K) U[k0 .. k0+K, :), K % 64 == 0.
// kclass: the profile class the launch is booked under (the updates inside
// the U12 solve belong to K4, the trailing updates to K5).
void tc_gemm(const TcPlan &p, int r0, int r1, int cb, int ce, int k0, int K, cudaStream_t s,
             int kclass)
{
  if (r1 <= r0 || ce <= cb || K <= 0)
    return;
  if (K % BK)
    throw std::runtime_error("tc_gemm: K must be a multiple of 64");
  prof_begin(kclass, s);
  const int M = r1 - r0, N = ce - cb;
  const long mt128 = (M + 127) / 128;
  const auto &b256 = *reinterpret_cast<const CUtensorMap *>(p.mapB);
  const auto &b128 = *reinterpret_cast<const CUtensorMap *>(p.mapB128);
  const auto &b64 = *reinterpret_cast<const CUtensorMap *>(p.mapB64);
  // narrower column tiles while the launch would leave most SMs idle
  if (N <= 64 || mt128 * ((N + 127) / 128) < 96)
    launch_cfg<1, 64>(p, b64, r0, r1, cb, ce, k0, K, s);
  else if (N <= 128 || mt128 * ((N + 255) / 256) < 96)
    launch_cfg<1, 128>(p, b128, r0, r1, cb, ce, k0, K, s);
  else if (K >= 1024 && M > 128 && (long)((M + 255) / 256) * ((N + 255) / 256) >= 96)
    launch_cfg<2, 256>(p, b256, r0, r1, cb, ce, k0, K, s);
  else
    launch_cfg<1, 256>(p, b256, r0, r1, cb, ce, k0, K, s);
  prof_end(kclass, s);
}

// A22 columns [cb, ce), rows [k0 + 64, n) -= L21 * U12 of the panel at k0 (jb = 64).
void launch_gemm_tc(const TcPlan &p, int k0, int cb, int ce, cudaStream_t s)
{
  tc_gemm(p, k0 + BK, p.n, cb, ce, k0, BK, s, KC_GEMM);
}

}  // namespace mpirg
