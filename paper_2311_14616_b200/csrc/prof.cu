// Per-kernel-class CUDA-event timing for bench.py's roofline numbers.
//
// When enabled, every hot-path launch site brackets its kernel with a pair of
// events recorded on the launching stream; collect() synchronises and sums
// the elapsed device time and the launch count per class. Disabled (the
// default) it costs one branch per launch.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/mpir_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace mpirg
{

namespace
{
struct Rec
{
  int kind;
  cudaStream_t s;  // pairs begin/end per stream (batch workers launch concurrently)
  cudaEvent_t a, b;
};
std::mutex g_pmu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::vector<int> g_open;  // stack of open record indices per kind (flat)

cudaEvent_t take()
{
  if (!g_pool.empty())
  {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  MPIRG_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}
}  // namespace

bool prof_on() { return g_on; }

extern "C" char **environ;
bool tool_attached()
{
  static const bool v = [] {
    if (const char *e = std::getenv("MPIRG_TOOL_ATTACHED"))  // explicit override (tests)
      return std::atoi(e) != 0;
    for (char **e = environ; e && *e; ++e)
      for (const char *k : {"CUDA_INJECTION64_PATH=", "CUDA_INJECTION32_PATH=",
                            "NV_COMPUTE_PROFILER_", "NV_SANITIZER_", "NSYS_PROFILING_SESSION_ID=",
                            "NV_NSIGHT_INJECTION_"})
        if (std::strncmp(*e, k, std::strlen(k)) == 0)
          return true;
    return false;
  }();
  return v;
}

void prof_begin(int kind, cudaStream_t s)
{
  if (!g_on)
    return;
  std::lock_guard<std::mutex> lk(g_pmu);
  Rec r{kind, s, take(), take()};
  MPIRG_CUDA_CHECK(cudaEventRecord(r.a, s));
  g_recs.push_back(r);
  g_open.push_back((int)g_recs.size() - 1);
}

void prof_end(int kind, cudaStream_t s)
{
  if (!g_on)
    return;
  std::lock_guard<std::mutex> lk(g_pmu);
  for (int i = (int)g_open.size() - 1; i >= 0; --i)
  {
    Rec &r = g_recs[g_open[i]];
    if (r.kind == kind && r.s == s)
    {
      MPIRG_CUDA_CHECK(cudaEventRecord(r.b, s));
      g_open.erase(g_open.begin() + i);
      return;
    }
  }
}

}  // namespace mpirg

extern "C" {

void mpirg_profile_enable(int on)
{
  std::lock_guard<std::mutex> lk(mpirg::g_pmu);
  mpirg::g_on = on != 0;
}

// Synchronises the device, then returns per-class totals (ms, launches) and
// clears the record list. Classes: enum mpirg_kernel_class.
int mpirg_profile_collect(double *ms, int *count, int nclass)
{
  std::lock_guard<std::mutex> lk(mpirg::g_pmu);
  if (cudaDeviceSynchronize() != cudaSuccess)
    return MPIRG_ERR_CUDA;
  for (int k = 0; k < nclass; ++k)
  {
    ms[k] = 0.0;
    count[k] = 0;
  }
  for (auto &r : mpirg::g_recs)
  {
    float t = 0.0f;
    if (r.kind >= 0 && r.kind < nclass && cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess)
    {
      ms[r.kind] += t;
      count[r.kind] += 1;
    }
    mpirg::g_pool.push_back(r.a);
    mpirg::g_pool.push_back(r.b);
  }
  mpirg::g_recs.clear();
  mpirg::g_open.clear();
  cudaGetLastError();
  return MPIRG_OK;
}

}  // extern "C"

// ---- FP32 FFMA / FP64 DFMA peak microbenchmarks ------------------------------
namespace
{
__device__ __forceinline__ float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T, bool IMM>
__global__ void __launch_bounds__(256) fma_peak_kernel(T *out, int iters, T b, T c)
{
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    a[j] = (T)(threadIdx.x + j) * (T)1e-3;
  for (int i = 0; i < iters; ++i)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      a[j] = IMM ? fma_t(a[j], (T)1.0001, (T)0.9999) : fma_t(a[j], b, c);
  }
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += a[j];
  if (s == (T)12345.678)
    out[blockIdx.x] = s;
}

template <typename T>
int fma_peak(double *tflops, double *ms_out, int iters)
{
  try
  {
    int dev = 0, sms = 0;
    MPIRG_CUDA_CHECK(cudaGetDevice(&dev));
    MPIRG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    T *out = nullptr;
    MPIRG_CUDA_CHECK(cudaMalloc(&out, sizeof(T) * sms * 8));
    cudaEvent_t e0, e1;
    MPIRG_CUDA_CHECK(cudaEventCreate(&e0));
    MPIRG_CUDA_CHECK(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256;
    double best = 0.0, best_ms = 0.0;
    for (int variant = 0; variant < 2; ++variant)
      for (int rep = 0; rep < 4; ++rep)
      {
        MPIRG_CUDA_CHECK(cudaEventRecord(e0));
        if (variant == 0)
          fma_peak_kernel<T, false><<<blocks, threads>>>(out, iters, (T)1.0001, (T)0.9999);
        else
          fma_peak_kernel<T, true><<<blocks, threads>>>(out, iters, (T)1.0001, (T)0.9999);
        MPIRG_CUDA_CHECK(cudaEventRecord(e1));
        MPIRG_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        MPIRG_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (rep > 0 && tf > best)
        {
          best = tf;
          best_ms = ms;
        }
      }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    *tflops = best;
    *ms_out = best_ms;
    return MPIRG_OK;
  }
  catch (const std::exception &)
  {
    return MPIRG_ERR_CUDA;
  }
}
}  // namespace

extern "C" int mpirg_ffma_peak(double *tflops, double *ms_out)
{
  return fma_peak<float>(tflops, ms_out, 8192);
}

extern "C" int mpirg_dfma_peak(double *tflops, double *ms_out)
{
  return fma_peak<double>(tflops, ms_out, 1024);
}

// Dependent-chain latency of one FMA (cycles): the floor per column of the
// residual's and the substitutions' row chains, which the reference's order
// makes sequential.
namespace
{
template <typename T>
__global__ void fma_latency_kernel(T a, T b, T *out, long long *cycles)
{
  T s = a;
  const long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i)
  {
    if constexpr (sizeof(T) == 8)
      s = __fma_rn(s, b, a);
    else
      s = __fmaf_rn(s, b, a);
  }
  const long long t1 = clock64();
  *out = s;
  *cycles = t1 - t0;
}
}  // namespace

extern "C" int mpirg_fma_latency(int prec, double *cycles)
{
  long long *dc = nullptr;
  void *out = nullptr;
  if (cudaMalloc(&dc, 8) != cudaSuccess || cudaMalloc(&out, 8) != cudaSuccess)
    return MPIRG_ERR_CUDA;
  for (int rep = 0; rep < 2; ++rep)
  {
    if (prec == MPIRG_B64)
      fma_latency_kernel<double><<<1, 1>>>(1.0, 0.999, static_cast<double *>(out), dc);
    else
      fma_latency_kernel<float><<<1, 1>>>(1.0f, 0.999f, static_cast<float *>(out), dc);
  }
  long long h = 0;
  const bool ok = cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(dc);
  cudaFree(out);
  if (!ok)
    return MPIRG_ERR_CUDA;
  *cycles = (double)h / 4096.0;
  return MPIRG_OK;
}

// ---- self-check of div_rcp (common.cuh) against the IEEE division ------------
namespace
{
__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Operand classes: 0 random bit patterns (every exponent, specials), 1 random
// mid-range a / b, 2 b with a near-all-ones or near-power-of-two significand.
template <typename T>
__device__ T draw(unsigned long long h, int cls, bool divisor)
{
  if constexpr (sizeof(T) == 4)
  {
    unsigned bits = (unsigned)h;
    if (cls >= 1)
      bits = (bits & 0x807fffffu) | ((unsigned)(127 - 70 + (h >> 40) % 141) << 23);
    if (cls == 2 && divisor)
    {
      const unsigned low = (unsigned)(h >> 48) & 0xfffu;
      bits = (bits & 0xff800000u) | ((h >> 33) & 1 ? (0x7fffffu - low) : low);
    }
    return __uint_as_float(bits);
  }
  else
  {
    unsigned long long bits = h;
    if (cls >= 1)
      bits = (bits & 0x800fffffffffffffull) |
             ((unsigned long long)(1023 - 520 + (mix64(h) % 1041)) << 52);
    if (cls == 2 && divisor)
    {
      const unsigned long long low = mix64(h ^ 0x5555ull) & 0xffffull;
      bits = (bits & 0xfff0000000000000ull) |
             ((mix64(h) & 1) ? (0xfffffffffffffull - low) : low);
    }
    return __longlong_as_double((long long)bits);
  }
}

template <typename T>
__global__ void check_div_kernel(unsigned long long seed, long long count,
                                 unsigned long long *bad, T *ex)
{
  unsigned long long nbad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
  {
    const unsigned long long h1 = mix64(seed * 0x100000001b3ull + 2 * i);
    const unsigned long long h2 = mix64(seed * 0x100000001b3ull + 2 * i + 1);
    const int cls = (int)(i % 3);
    const T a = draw<T>(h1, cls, false), b = draw<T>(h2, cls, true);
    const T want = mpirg::divide(a, b);
    const T got = mpirg::div_rcp(a, b, mpirg::make_rcp(b));
    const bool same = (want == got && signbit(want) == signbit(got)) || (isnan(want) && isnan(got));
    if (!same)
    {
      ++nbad;
      ex[0] = a;
      ex[1] = b;
    }
  }
  if (nbad)
    atomicAdd(bad, nbad);
}
}  // namespace

extern "C" int mpirg_check_fast_div(int prec, unsigned long long seed, long long count,
                                    long long *mismatches, double *example)
{
  try
  {
    unsigned long long *bad = nullptr;
    double *ex = nullptr;
    MPIRG_CUDA_CHECK(cudaMalloc(&bad, sizeof(unsigned long long)));
    MPIRG_CUDA_CHECK(cudaMalloc(&ex, 2 * sizeof(double)));
    MPIRG_CUDA_CHECK(cudaMemset(bad, 0, sizeof(unsigned long long)));
    MPIRG_CUDA_CHECK(cudaMemset(ex, 0, 2 * sizeof(double)));
    if (prec == mpirg::B64)
      check_div_kernel<double><<<148 * 8, 256>>>(seed, count, bad, ex);
    else
      check_div_kernel<float><<<148 * 8, 256>>>(seed, count, bad, reinterpret_cast<float *>(ex));
    MPIRG_CUDA_CHECK(cudaGetLastError());
    unsigned long long h = 0;
    double hex[2] = {0, 0};
    MPIRG_CUDA_CHECK(cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost));
    MPIRG_CUDA_CHECK(cudaMemcpy(hex, ex, sizeof(hex), cudaMemcpyDeviceToHost));
    if (prec != mpirg::B64)
    {
      float f[2];
      std::memcpy(f, hex, sizeof(f));
      hex[0] = f[0];
      hex[1] = f[1];
    }
    cudaFree(bad);
    cudaFree(ex);
    *mismatches = (long long)h;
    if (example)
    {
      example[0] = hex[0];
      example[1] = hex[1];
    }
    return MPIRG_OK;
  }
  catch (const std::exception &)
  {
    return MPIRG_ERR_CUDA;
  }
}
