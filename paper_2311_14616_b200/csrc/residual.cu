// K7 -- compensated residual r = b - A x evaluated in TR, bitwise equal to
// detail::residual_into<TW,TR> (proj/include/mpir/ir_engine.hpp:115-139) with
// two_sum (proj/include/mpir/matrix.hpp:158-164) as the reference build
// contracts it:
//   t = fma(-a_ij, x_j, s_i); z = t - s_i;
//   e = (s_i - (t - z)) + fma(-a_ij, x_j, -z); c_i += e; s_i = t
// with j ascending per row, then r_i = s_i + c_i.
//
// One lane per row (the chain is sequential in j by contract), one warp per
// 32-row stripe. The stripe streams through shared memory in 32 x BC tiles
// brought in by TMA (cp.async.bulk.tensor.2d) into a STAGES-deep mbarrier
// ring, so each SM keeps ~STAGES*16 KB of A in flight -- the bytes-in-flight
// the HBM roofline needs with only n/32 warps in the whole grid. When the
// row pitch is not 16-byte aligned (TMA's requirement) a plain-load path with
// the identical arithmetic is used instead. ||r||_inf (NaN-propagating, as
// norm_inf) is reduced in the same pass.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace mpirg
{

namespace
{

constexpr int RES_BC = 64;  // columns per tile

__device__ __forceinline__ double res_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float res_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double res_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float res_sub(float a, float b) { return __fsub_rn(a, b); }

template <typename TR>
__device__ __forceinline__ void two_sum_step(TR a, TR xj, TR &s, TR &c)
{
  const TR t = res_fma(-a, xj, s);
  const TR z = res_sub(t, s);
  const TR e = add(res_sub(s, res_sub(t, z)), res_fma(-a, xj, -z));
  c = add(c, e);
  s = t;
}

__device__ __forceinline__ double widen(double v) { return v; }
__device__ __forceinline__ double widen_to_d(float v) { return (double)v; }
template <typename TR, typename TW>
__device__ __forceinline__ TR prom(TW v) { return (TR)v; }

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1)
{
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load_1d(void *dst, const void *src, uint32_t bytes,
                                             uint64_t *bar)
{
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename TW, typename TR, int STAGES, int RPW>
__global__ void __launch_bounds__(32) residual_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          int n, const TR *__restrict__ x,
                                                          const TW *__restrict__ b,
                                                          TR *__restrict__ r,
                                                          unsigned long long *rnorm_bits)
{
  // RPW rows per warp (lanes >= RPW idle): at small n there are fewer rows
  // than lanes x SMSPs, so narrower warps spread the n independent chains
  // over more SM sub-partitions.
  // Each stage holds the RPW x RES_BC tile of A and the matching RES_BC-slice
  // of x (one bulk copy on the same mbarrier), so the per-column x values
  // come from shared memory instead of a global load per group of columns.
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TILE_E = RES_BC * RPW;
  constexpr uint32_t kBytes = TILE_E * sizeof(TW);
  constexpr uint32_t xBytes = RES_BC * sizeof(TR);
  constexpr size_t STAGE_B = kBytes + xBytes;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)STAGES * STAGE_B);
  const int lane = threadIdx.x;
  const int r0 = blockIdx.x * RPW;
  const int row = r0 + lane;
  const bool valid = lane < RPW && row < n;
  const int ntiles = (n + RES_BC - 1) / RES_BC;
  const int nfull = n / RES_BC;  // tiles whose x slice is a whole bulk copy
  auto stage_tile = [&](int st) { return reinterpret_cast<TW *>(sm + (size_t)st * STAGE_B); };
  auto stage_x = [&](int st) {
    return reinterpret_cast<TR *>(sm + (size_t)st * STAGE_B + kBytes);
  };
  auto issue = [&](int st, int t) {
    const bool fullx = t < nfull;
    mbar_expect_tx(bars + st, kBytes + (fullx ? xBytes : 0u));
    tma_load_2d(stage_tile(st), &tmap, bars + st, r0, t * RES_BC);
    if (fullx)
      bulk_load_1d(stage_x(st), x + (size_t)t * RES_BC, xBytes, bars + st);
  };

  if (lane == 0)
  {
    for (int s = 0; s < STAGES; ++s)
      mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    for (int s = 0; s < STAGES && s < ntiles; ++s)
      issue(s, s);
  }
  __syncwarp();

  const int lr = lane < RPW ? lane : 0;
  TR s = valid ? prom<TR, TW>(b[row]) : TR(0);
  TR c = TR(0);
  for (int t = 0; t < ntiles; ++t)
  {
    const int st = t % STAGES;
    mbar_wait(bars + st, (uint32_t)((t / STAGES) & 1));
    const TW *tile = stage_tile(st);
    const int j0 = t * RES_BC;
    if (lane < RPW)
    {
      if (t < nfull)
      {
        const TR *xs = stage_x(st);
#pragma unroll 16
        for (int jj = 0; jj < RES_BC; ++jj)
          two_sum_step<TR>(prom<TR, TW>(tile[jj * RPW + lr]), xs[jj], s, c);
      }
      else
      {
        for (int jj = 0; jj < n - j0; ++jj)
          two_sum_step<TR>(prom<TR, TW>(tile[jj * RPW + lr]), __ldg(x + j0 + jj), s, c);
      }
    }
    __syncwarp();
    if (lane == 0 && t + STAGES < ntiles)
      issue(st, t + STAGES);
  }
  TR rv = add(s, c);
  unsigned long long bits = 0;
  if (valid)
  {
    r[row] = rv;
    bits = abs_bits((double)rv);
  }
  bits = warp_max_u64(bits);
  if (lane == 0)
    atomicMax(rnorm_bits, bits);
}

// Plain-load path (row pitch not 16-byte aligned): same arithmetic.
template <typename TW, typename TR>
__global__ void __launch_bounds__(32) residual_plain_kernel(const TW *__restrict__ a, int n,
                                                            const TR *__restrict__ x,
                                                            const TW *__restrict__ b,
                                                            TR *__restrict__ r,
                                                            unsigned long long *rnorm_bits)
{
  const int lane = threadIdx.x;
  const int row = blockIdx.x * 32 + lane;
  const bool valid = row < n;
  TR s = valid ? prom<TR, TW>(b[row]) : TR(0);
  TR c = TR(0);
  const int rr = valid ? row : 0;
  int j = 0;
  for (; j + 16 <= n; j += 16)
  {
    TW v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      v[q] = __ldcs(a + (size_t)(j + q) * n + rr);
#pragma unroll
    for (int q = 0; q < 16; ++q)
      two_sum_step<TR>(prom<TR, TW>(v[q]), __ldg(x + j + q), s, c);
  }
  for (; j < n; ++j)
    two_sum_step<TR>(prom<TR, TW>(__ldcs(a + (size_t)j * n + rr)), __ldg(x + j), s, c);
  TR rv = add(s, c);
  unsigned long long bits = 0;
  if (valid)
  {
    r[row] = rv;
    bits = abs_bits((double)rv);
  }
  bits = warp_max_u64(bits);
  if (lane == 0)
    atomicMax(rnorm_bits, bits);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn)
  {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    MPIRG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int STAGES, int RPW>
int res_stages_smem(int esz)
{
  return STAGES * (RES_BC * RPW * esz + RES_BC * 8) + STAGES * 8;
}

// Rows per warp for the TMA path: the widest warp that still gives every SM
// sub-partition (148 x 4) at least one row chain. MPIRG_RES_RPW overrides.
int residual_rpw(int n)
{
  static const int forced = [] {
    const char *e = std::getenv("MPIRG_RES_RPW");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 8 || forced == 16 || forced == 32)
    return forced;
  if (n / 32 >= 148 * 4)
    return 32;
  if (n / 16 >= 148 * 4)
    return 16;
  return 8;
}

template <typename TW, typename TR, int RPW>
void residual_tma_launch(const ResidualPlan &p, const void *x, const void *b, void *r,
                         unsigned long long *rb, cudaStream_t s)
{
  constexpr int ST = 4;
  const int n = p.n;
  const int smem = res_stages_smem<ST, RPW>(sizeof(TW));
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(residual_tma_kernel<TW, TR, ST, RPW>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.done();
  }
  CUtensorMap map;
  std::memcpy(&map, static_cast<const CUtensorMap *>(p.tmap) + (RPW == 32 ? 0 : RPW == 16 ? 1 : 2),
              sizeof(CUtensorMap));
  residual_tma_kernel<TW, TR, ST, RPW><<<(n + RPW - 1) / RPW, 32, smem, s>>>(
      map, n, static_cast<const TR *>(x), static_cast<const TW *>(b), static_cast<TR *>(r), rb);
}

template <typename TW, typename TR>
void residual_t(const ResidualPlan &p, const void *x, const void *b, void *r,
                unsigned long long *rb, cudaStream_t s)
{
  const int n = p.n;
  const int grid = (n + 31) / 32;
  ProfScope ps(KC_RESID, s);
  // the TMA path bulk-copies x slices: x must be 16-byte aligned too
  if (p.tmap && reinterpret_cast<uintptr_t>(x) % 16 == 0)
  {
    const int rpw = residual_rpw(n);
    if (rpw == 32)
      residual_tma_launch<TW, TR, 32>(p, x, b, r, rb, s);
    else if (rpw == 16)
      residual_tma_launch<TW, TR, 16>(p, x, b, r, rb, s);
    else
      residual_tma_launch<TW, TR, 8>(p, x, b, r, rb, s);
  }
  else
  {
    residual_plain_kernel<TW, TR><<<grid, 32, 0, s>>>(static_cast<const TW *>(p.a), n,
                                                     static_cast<const TR *>(x),
                                                     static_cast<const TW *>(b),
                                                     static_cast<TR *>(r), rb);
  }
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

// ---- IR bookends -----------------------------------------------------------
template <typename TW, typename TR>
__global__ void ir_init_kernel(int n, const TW *__restrict__ b, TR *__restrict__ r,
                               TR *__restrict__ x, unsigned long long *bnorm_bits)
{
  unsigned long long bits = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    const TR v = prom<TR, TW>(b[i]);
    r[i] = v;
    x[i] = TR(0);
    const unsigned long long bb = abs_bits((double)v);
    bits = bb > bits ? bb : bits;
  }
  bits = warp_max_u64(bits);
  if ((threadIdx.x & 31) == 0)
    atomicMax(bnorm_bits, bits);
}

template <typename TW, typename TR>
__global__ void ir_finish_kernel(int n, const TR *__restrict__ x, TW *__restrict__ sol)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    sol[i] = (TW)x[i];
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() { return get_encode(); }

void residual_plan_make(ResidualPlan &p, int tw, int n, const void *a)
{
  residual_plan_free(p);
  p.n = n;
  p.tw = tw;
  p.a = a;
  const size_t esz = elem_size(tw);
  const bool aligned = ((size_t)n * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(a) % 16) == 0;
  if (!aligned || n < 32)
    return;
  // one map per rows-per-warp box height (32, 16, 8)
  CUtensorMap *map = new CUtensorMap[3];
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)n * esz};
  cuuint32_t estr[2] = {1, 1};
  for (int v = 0; v < 3; ++v)
  {
    cuuint32_t box[2] = {(cuuint32_t)(32 >> v), (cuuint32_t)RES_BC};
    const CUresult rc = get_encode()(
        map + v, tw == B64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
        const_cast<void *>(a), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS)
    {
      delete[] map;
      return;  // fall back to the plain-load path
    }
  }
  p.tmap = map;
}

void residual_plan_free(ResidualPlan &p)
{
  delete[] static_cast<CUtensorMap *>(p.tmap);
  p = ResidualPlan{};
}

void launch_residual(const ResidualPlan &p, int tr, const void *x, const void *b, void *r,
                     unsigned long long *rb, cudaStream_t s)
{
  if (p.n <= 0)
    return;
  if (p.tw == B64 && tr == B64)
    residual_t<double, double>(p, x, b, r, rb, s);
  else if (p.tw == B32 && tr == B64)
    residual_t<float, double>(p, x, b, r, rb, s);
  else if (p.tw == B32 && tr == B32)
    residual_t<float, float>(p, x, b, r, rb, s);
  else
    throw std::invalid_argument("residual precision must be at least the working precision");
}

void launch_ir_init(int tw, int tr, int n, const void *b, void *r, void *x,
                    unsigned long long *bnorm_bits, cudaStream_t s)
{
  const int grid = std::min(148 * 4, (n + 255) / 256);
  ProfScope ps(KC_VEC, s);
  if (tw == B64 && tr == B64)
    ir_init_kernel<double, double><<<grid, 256, 0, s>>>(n, (const double *)b, (double *)r,
                                                       (double *)x, bnorm_bits);
  else if (tw == B32 && tr == B64)
    ir_init_kernel<float, double><<<grid, 256, 0, s>>>(n, (const float *)b, (double *)r,
                                                      (double *)x, bnorm_bits);
  else
    ir_init_kernel<float, float><<<grid, 256, 0, s>>>(n, (const float *)b, (float *)r,
                                                     (float *)x, bnorm_bits);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

void launch_ir_finish(int tw, int tr, int n, const void *x, void *sol, cudaStream_t s)
{
  const int grid = std::min(148 * 4, (n + 255) / 256);
  ProfScope ps(KC_VEC, s);
  if (tw == B64 && tr == B64)
    ir_finish_kernel<double, double><<<grid, 256, 0, s>>>(n, (const double *)x, (double *)sol);
  else if (tw == B32 && tr == B64)
    ir_finish_kernel<float, double><<<grid, 256, 0, s>>>(n, (const double *)x, (float *)sol);
  else
    ir_finish_kernel<float, float><<<grid, 256, 0, s>>>(n, (const float *)x, (float *)sol);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace mpirg
