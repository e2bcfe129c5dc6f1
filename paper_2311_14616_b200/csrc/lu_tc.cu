// K5b -- tensor-core trailing update for binary16 factors (lu_mode TC).
//
// A22 <- fp16( fp32(A22) - L21 * U12 ), with L21 (rows, nb=64) and U12
// (64, cols) binary16 and the 64-term product accumulated in fp32 by the 5th
// generation tensor cores: one rounding to binary16 per panel step instead of
// the reference's two per term (dense_lu.hpp:96-107 with half.hpp:285-288).
// This is NOT bit-compatible with the reference; it is the fast mode whose
// deviation SURVEY.md 8(d) bounds by the refinement's stopping rule. The exact
// mode (lu.cu lu_gemm_kernel) remains the default.
//
// One CTA = one 128 x 256 tile of A22, 4 warps:
//   * TMA (SWIZZLE_128B) brings L21 (128 x 64, MN-major, two 64-row boxes)
//     and U12 (256 x 64, K-major) into shared memory on one mbarrier;
//   * one thread issues 4 tcgen05.mma.kind::f16 (M=128, N=256, K=16) with A
//     negated into a 256-column TMEM accumulator, then tcgen05.commit;
//   * the C tile (128 x 256 of A22) arrives by TMA with the operands; each
//     warp reads its 32 TMEM lanes (tcgen05.ld 32x32b), forms fp16(C + D) in
//     shared memory, and one TMA store writes the tile back (clipped to the
//     update's column range [cb, ce) by the store map's extent).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdexcept>

#include "common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace mpirg
{
namespace
{
constexpr int TM = 128, TN = 256, TK = 64;
constexpr uint32_t A_BYTES = TM * TK * 2;  // 16 KB
constexpr uint32_t B_BYTES = TN * TK * 2;  // 32 KB
constexpr uint32_t C_BYTES = TM * TN * 2;  // 64 KB
// 112 KB of tiles + 1 KB alignment slack: two CTAs per SM, whose two
// 256-column accumulators fill the 512-column TMEM.
constexpr size_t TC_SMEM = 1024 + A_BYTES + B_BYTES + C_BYTES;
constexpr uint32_t IDESC = tc::idesc_f16_f32(TM, TN, /*a_mn=*/true, /*b_mn=*/false,
                                             /*neg_a=*/true);

__global__ void __launch_bounds__(128, 1)
    lu_gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB,
                      const __grid_constant__ CUtensorMap mapC, int k0, int c0, int cb)
{
  extern __shared__ unsigned char tsm_raw[];
  __shared__ __align__(8) uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  unsigned char *base = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *As = base;            // [2 row chunks][64 k][64 rows] fp16, swizzled
  unsigned char *Bs = base + A_BYTES;  // [256 cols][64 k] fp16, swizzled
  h16 *Cs = reinterpret_cast<h16 *>(base + A_BYTES + B_BYTES);  // [256 cols][128 rows]
  const int warp = threadIdx.x >> 5;
  const int r0 = c0 + blockIdx.x * TM;
  const int j0 = cb + blockIdx.y * TN;

  if (warp == 0)
    tc::tmem_alloc(&tmem_base, TN);
  if (threadIdx.x == 32)
  {
    tc::mbar_init(&bar_tma, 1);
    tc::mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (threadIdx.x == 32)
  {
    tc::mbar_expect_tx(&bar_tma, A_BYTES + B_BYTES + C_BYTES);
    tc::tma_load_2d(Cs, &mapC, &bar_tma, r0, j0);
    tc::tma_load_2d(As, &mapA, &bar_tma, r0, k0);
    tc::tma_load_2d(As + A_BYTES / 2, &mapA, &bar_tma, r0 + 64, k0);
    tc::tma_load_2d(Bs, &mapB, &bar_tma, k0, j0);
    tc::mbar_wait(&bar_tma, 0);
    tc::fence_after();
    const uint32_t sa = tc::smem_u32(As), sb = tc::smem_u32(Bs);
#pragma unroll
    for (int kk = 0; kk < TK / 16; ++kk)
    {
      // A, MN-major: 64-row atoms 8 KB apart (LBO), 8-k groups 1 KB apart (SBO);
      // K=16 per MMA = two 8-k groups.
      const uint64_t ad = tc::desc_sw128(sa + kk * 2048, 8192, 1024);
      // B, K-major: 8-column groups 1 KB apart (SBO); K=16 = 32 bytes into the row.
      const uint64_t bd = tc::desc_sw128(sb + kk * 32, 16, 1024);
      tc::mma_f16(tmem, ad, bd, IDESC, kk > 0 ? 1u : 0u);
    }
    tc::mma_commit(&bar_mma);
  }
  tc::mbar_wait(&bar_mma, 0);
  tc::fence_after();

  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  h16 *crow = Cs + threadIdx.x;  // this thread's row of the tile
#pragma unroll 1
  for (int c16 = 0; c16 < TN; c16 += 16)
  {
    float v[16];
    tc::tmem_ld16(lane_addr + c16, v);
#pragma unroll
    for (int e = 0; e < 16; ++e)
    {
      h16 &dst = crow[(c16 + e) * TM];
      dst = f2h(__fadd_rn(h2f(dst), v[e]));
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0)
  {
    tc::tma_store_2d(&mapC, Cs, r0, j0);
    tc::tma_store_wait();
  }
  if (warp == 0)
    tc::tmem_dealloc(tmem, TN);
}

void encode(CUtensorMap *map, void *a, int n, int box0, int box1, int cols = -1,
            CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B)
{
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)(cols < 0 ? n : cols)};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = tma_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a, dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed for the TC trailing update");
}
}  // namespace

bool tc_update_supported(int n, int nb) { return nb == TK && n % 8 == 0 && n >= TK; }

void tc_plan_make(TcPlan &p, void *a, int n)
{
  static_assert(sizeof(CUtensorMap) <= sizeof(p.mapA), "tensor map storage");
  encode(reinterpret_cast<CUtensorMap *>(p.mapA), a, n, 64, 64);
  encode(reinterpret_cast<CUtensorMap *>(p.mapB), a, n, 64, TN);
  p.a = a;
  p.n = n;
}

// A22 columns [cb, ce), rows [k0 + 64, n) -= L21 * U12 of the panel at k0 (jb = 64).
void launch_gemm_tc(const TcPlan &p, int k0, int cb, int ce, cudaStream_t s)
{
  const int n = p.n, c0 = k0 + TK;
  if (ce <= cb || c0 >= n)
    return;
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(lu_gemm_tc_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)TC_SMEM));
    configured.done();
  }
  // C tiles: the matrix viewed with ce columns, so the store never touches
  // columns outside this update's range (another stream may own them).
  CUtensorMap mapC;
  encode(&mapC, p.a, n, TM, TN, ce, CU_TENSOR_MAP_SWIZZLE_NONE);
  prof_begin(KC_GEMM, s);
  const dim3 grid((n - c0 + TM - 1) / TM, (ce - cb + TN - 1) / TN);
  lu_gemm_tc_kernel<<<grid, 128, TC_SMEM, s>>>(
      *reinterpret_cast<const CUtensorMap *>(p.mapA),
      *reinterpret_cast<const CUtensorMap *>(p.mapB), mapC, k0, c0, cb);
  MPIRG_CUDA_CHECK(cudaGetLastError());
  prof_end(KC_GEMM, s);
}

}  // namespace mpirg
