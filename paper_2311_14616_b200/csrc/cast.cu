// K1 -- interprecision copy A_F = I_W^F(A) and the refactor one-norm.
//
// Replaces, bit for bit:
//   demote_matrix_into<To,From>   proj/include/mpir/matrix.hpp:74-85
//   demote_checked<To>            proj/include/mpir/precision.hpp:172-185
//   matrix_one_norm<T>            proj/include/mpir/mp_structures.hpp:22-36
// Demotion is RNE (static_cast / F16C / single-rounding double->half). An
// element whose |x| exceeds the target's largest finite value raises
// OverflowDetected in the reference at the first such element in storage
// order; here every offender does an atomicMin on its storage index so the
// host reports the same one. Underflow (x != 0 rounds to 0) is sticky.
// The one-norm is a sequential per-column sum in the matrix's own precision
// (one lane per column, rows in order), max over columns ignoring NaN like
// std::max(best, s).
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace mpirg
{

namespace
{

__device__ __forceinline__ double max_finite_of(int p)
{
  return p == B64 ? DBL_MAX : (p == B32 ? (double)FLT_MAX : 65504.0);
}

template <typename From, typename To>
__device__ __forceinline__ To demote_one(From x, size_t idx, double maxf, bool &uf,
                                         unsigned long long &ovf)
{
  const double xd = to_d(x);
  if (isfinite(xd) && fabs(xd) > maxf && idx < ovf)
    ovf = idx;
  const To y = demote<To, From>(x);
  if (to_d(y) == 0.0 && xd != 0.0)
    uf = true;
  return y;
}

__device__ __forceinline__ void flush_flags(bool uf, unsigned long long ovf, DevInfo *info)
{
  const unsigned m = __activemask();
  if (__any_sync(m, uf) && (threadIdx.x & 31) == (__ffs(m) - 1))
    info->underflow = 1;
  if (ovf != ~0ull)
    atomicMin(&info->overflow_index, ovf);
}

// Elementwise demotion, 8 elements per thread per iteration.
template <typename From, typename To>
__global__ void demote_kernel(const From *__restrict__ src, To *__restrict__ dst, size_t count,
                              DevInfo *info)
{
  const double maxf = max_finite_of(std::is_same<To, double>::value
                                        ? B64
                                        : (std::is_same<To, float>::value ? B32 : B16));
  bool uf = false;
  unsigned long long ovf = ~0ull;
  const size_t nvec = count / 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < nvec; v += stride)
  {
    From in[8];
    To out[8];
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + v * 8);
#pragma unroll
    for (int q = 0; q < (int)(8 * sizeof(From) / 16); ++q)
      reinterpret_cast<uint4 *>(in)[q] = __ldcs(s4 + q);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      out[e] = demote_one<From, To>(in[e], v * 8 + e, maxf, uf, ovf);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + v * 8);
#pragma unroll
    for (int q = 0; q < (int)(8 * sizeof(To) / 16); ++q)
      d4[q] = reinterpret_cast<const uint4 *>(out)[q];
  }
  for (size_t i = nvec * 8 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += stride)
    dst[i] = demote_one<From, To>(src[i], i, maxf, uf, ovf);
  flush_flags(uf, ovf, info);
}

template <typename T> __device__ __forceinline__ T ldcs_t(const T *p) { return __ldcs(p); }
template <> __device__ __forceinline__ h16 ldcs_t<h16>(const h16 *p)
{
  return h16{__ldcs(reinterpret_cast<const unsigned short *>(p))};
}

// Plain |x| in T arithmetic and the T-typed running sum.
__device__ __forceinline__ double absv(double v) { return fabs(v); }
__device__ __forceinline__ float absv(float v) { return fabsf(v); }
__device__ __forceinline__ h16 absv(h16 v) { return h16{(uint16_t)(v.bits & 0x7fffu)}; }
__device__ __forceinline__ double acc_add(double s, double v) { return __dadd_rn(s, v); }
__device__ __forceinline__ float acc_add(float s, float v) { return __fadd_rn(s, v); }
__device__ __forceinline__ h16 acc_add(h16 s, h16 v) { return hadd(s, v); }

// Fused cast + one-norm. A CTA owns a stripe of CN = 16 columns and walks
// down the rows in chunks of 256. Eight loader warps (lane = row) do the
// coalesced load / demote / store of the chunk -- every element independent --
// and deposit |x| into a double-buffered, padded smem tile; a ninth warp
// (lane = column) performs the reference's strictly sequential per-column sum
// over the previous chunk while the loaders already stream the next one. The
// sum chain (n dependent adds per column) is therefore the only serial part,
// and it overlaps the HBM stream instead of gating it.
// To == From (TF == TW) is a plain copy. NORM_ONLY skips the store.
constexpr int CN = 16;            // columns per CTA
constexpr int CLW = 8;            // loader warps
constexpr int CCH = CLW * 32;     // rows per chunk
constexpr int CAST_NT = CLW * 32 + 32;

template <typename From, typename To, bool NORM_ONLY>
__global__ void __launch_bounds__(CAST_NT) cast_norm_kernel(const From *__restrict__ src,
                                                            To *__restrict__ dst, int rows,
                                                            int cols,
                                                            unsigned long long *norm_bits,
                                                            DevInfo *info, int col_off,
                                                            size_t sys_stride)
{
  extern __shared__ __align__(16) unsigned char cast_sm[];
  // batched launches (config 5b): system blockIdx.y has its own matrix,
  // norm slot and error record; storage-order indices are per system
  src += (size_t)blockIdx.y * sys_stride;
  if constexpr (!NORM_ONLY)
    dst += (size_t)blockIdx.y * sys_stride;
  norm_bits += blockIdx.y;
  if (sys_stride)
    info += blockIdx.y;
  auto tile = reinterpret_cast<From(*)[CN][CCH + 1]>(cast_sm);  // [2][CN][CCH+1]
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  // columns [col_off, col_off + cols) of the rows x * matrix (a column chunk
  // of a matrix that arrives in pieces keeps its storage-order indices)
  const int c0 = col_off + blockIdx.x * CN;
  const int ncol = min(CN, col_off + cols - c0);
  const double maxf =
      NORM_ONLY ? 0.0
                : max_finite_of(std::is_same<To, double>::value
                                    ? B64
                                    : (std::is_same<To, float>::value ? B32 : B16));
  bool uf = false;
  unsigned long long ovf = ~0ull;
  From sum;
  if constexpr (std::is_same<From, h16>::value)
    sum = h16{0};
  else
    sum = From(0);
  const int nchunks = (rows + CCH - 1) / CCH;

  From cur[CN];
  auto load = [&](int ch) {
    const int r = ch * CCH + w * 32 + lane;
#pragma unroll
    for (int c = 0; c < CN; ++c)
      cur[c] = (c < ncol && r < rows) ? ldcs_t(src + (size_t)(c0 + c) * rows + r) : From{};
  };
  if (w < CLW && nchunks > 0)
    load(0);
  for (int ch = 0; ch <= nchunks; ++ch)
  {
    if (w < CLW)
    {
      if (ch < nchunks)
      {
        const int rr = w * 32 + lane;
        const int r = ch * CCH + rr;
        From (*tb)[CCH + 1] = tile[ch & 1];
#pragma unroll
        for (int c = 0; c < CN; ++c)
        {
          if (c < ncol && r < rows)
          {
            if constexpr (!NORM_ONLY)
            {
              const size_t idx = (size_t)(c0 + c) * rows + r;
              dst[idx] = demote_one<From, To>(cur[c], idx, maxf, uf, ovf);
            }
          }
          tb[c][rr] = absv(cur[c]);
        }
        if (ch + 1 < nchunks)
          load(ch + 1);
      }
    }
    else if (ch > 0 && lane < ncol)
    {
      // the sequential column sum over chunk ch-1, rows in order
      const From *tr = tile[(ch - 1) & 1][lane];
      const int nr = min(CCH, rows - (ch - 1) * CCH);
      if (nr == CCH)
      {
#pragma unroll 16
        for (int i = 0; i < CCH; ++i)
          sum = acc_add(sum, tr[i]);
      }
      else
      {
        for (int i = 0; i < nr; ++i)
          sum = acc_add(sum, tr[i]);
      }
    }
    __syncthreads();
  }
  if (w == CLW)
  {
    // best = std::max(best, double(s)): NaN sums never win; sums are >= 0.
    const double sd = lane < ncol ? to_d(sum) : 0.0;
    unsigned long long bits = isnan(sd) ? 0ull : abs_bits(sd);
    bits = warp_max_u64(bits);
    if (lane == 0)
      atomicMax(norm_bits, bits);
  }
  else if constexpr (!NORM_ONLY)
    flush_flags(uf, ovf, info);
}

template <typename From, typename To>
void demote_t(const void *src, void *dst, size_t count, DevInfo *info, cudaStream_t s)
{
  if (count == 0)
    return;
  const size_t nvec = (count + 7) / 8;
  int grid = (int)std::min<size_t>((nvec + 255) / 256, 148 * 8);
  if (grid < 1)
    grid = 1;
  ProfScope ps(KC_CAST, s);
  demote_kernel<From, To><<<grid, 256, 0, s>>>(static_cast<const From *>(src),
                                              static_cast<To *>(dst), count, info);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

template <typename From, typename To, bool NORM_ONLY>
void cast_norm_t(int rows, int cols, const void *src, void *dst, unsigned long long *nb,
                 DevInfo *info, cudaStream_t s, int col_off = 0, int ns = 1)
{
  if (rows <= 0 || cols <= 0 || ns <= 0)
    return;
  const dim3 grid((cols + CN - 1) / CN, ns);
  constexpr int smem = (int)(sizeof(From) * 2 * CN * (CCH + 1));
  static DeviceOnce configured;
  if (configured.needed())
  {
    MPIRG_CUDA_CHECK(cudaFuncSetAttribute(cast_norm_kernel<From, To, NORM_ONLY>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.done();
  }
  ProfScope ps(KC_CAST, s);
  cast_norm_kernel<From, To, NORM_ONLY><<<grid, CAST_NT, smem, s>>>(
      static_cast<const From *>(src), static_cast<To *>(dst), rows, cols, nb, info, col_off,
      ns > 1 ? (size_t)rows * cols : (size_t)0);
  MPIRG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

void launch_demote(int from, int to, const void *src, void *dst, size_t count, DevInfo *info,
                   cudaStream_t s)
{
  if (from == B64 && to == B64)
    demote_t<double, double>(src, dst, count, info, s);
  else if (from == B64 && to == B32)
    demote_t<double, float>(src, dst, count, info, s);
  else if (from == B64 && to == B16)
    demote_t<double, h16>(src, dst, count, info, s);
  else if (from == B32 && to == B32)
    demote_t<float, float>(src, dst, count, info, s);
  else if (from == B32 && to == B16)
    demote_t<float, h16>(src, dst, count, info, s);
  else if (from == B16 && to == B16)
    demote_t<h16, h16>(src, dst, count, info, s);
  else
    throw std::invalid_argument("demotion must not gain precision");
}

void launch_cast_norm(int from, int to, int rows, int cols, const void *src, void *dst,
                      unsigned long long *nb, DevInfo *info, cudaStream_t s, int col_off, int ns)
{
  if (ns > 1 && !(from == B64 && to == B32 && col_off == 0))
    throw std::invalid_argument("batched cast: binary64 -> binary32 only");
  if (from == B64 && to == B64)
    cast_norm_t<double, double, false>(rows, cols, src, dst, nb, info, s, col_off);
  else if (from == B64 && to == B32)
    cast_norm_t<double, float, false>(rows, cols, src, dst, nb, info, s, col_off, ns);
  else if (from == B64 && to == B16)
    cast_norm_t<double, h16, false>(rows, cols, src, dst, nb, info, s, col_off);
  else if (from == B32 && to == B32)
    cast_norm_t<float, float, false>(rows, cols, src, dst, nb, info, s, col_off);
  else if (from == B32 && to == B16)
    cast_norm_t<float, h16, false>(rows, cols, src, dst, nb, info, s, col_off);
  else
    throw std::invalid_argument("unsupported cast");
}

void launch_one_norm(int prec, int rows, int cols, const void *src, unsigned long long *nb,
                     cudaStream_t s)
{
  if (prec == B64)
    cast_norm_t<double, double, true>(rows, cols, src, nullptr, nb, nullptr, s);
  else if (prec == B32)
    cast_norm_t<float, float, true>(rows, cols, src, nullptr, nb, nullptr, s);
  else
    cast_norm_t<h16, h16, true>(rows, cols, src, nullptr, nb, nullptr, s);
}

}  // namespace mpirg
