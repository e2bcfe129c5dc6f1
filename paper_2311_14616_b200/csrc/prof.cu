// Per-kernel-class CUDA-event timing for bench.py's roofline numbers.
//
// When enabled, every hot-path launch site brackets its kernel with a pair of
// events recorded on the launching stream; collect() synchronises and sums
// the elapsed device time and the launch count per class. Disabled (the
// default) it costs one branch per launch.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "../../include/mpir_gpu.h"
#include "kernels.cuh"

namespace mpirg
{

namespace
{
struct Rec
{
  int kind;
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

void prof_begin(int kind, cudaStream_t s)
{
  if (!g_on)
    return;
  std::lock_guard<std::mutex> lk(g_pmu);
  Rec r{kind, take(), take()};
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
    if (r.kind == kind)
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

// ---- FP32 FFMA peak microbenchmark -------------------------------------------
namespace
{
template <bool IMM>
__global__ void __launch_bounds__(256) ffma_peak_kernel(float *out, int iters, float b, float c)
{
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    a[j] = (float)(threadIdx.x + j) * 1e-3f;
  for (int i = 0; i < iters; ++i)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      a[j] = IMM ? __fmaf_rn(a[j], 1.0001f, 0.9999f) : __fmaf_rn(a[j], b, c);
  }
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += a[j];
  if (s == 12345.678f)
    out[blockIdx.x] = s;
}
}  // namespace

extern "C" int mpirg_ffma_peak(double *tflops, double *ms_out)
{
  try
  {
    int dev = 0, sms = 0;
    MPIRG_CUDA_CHECK(cudaGetDevice(&dev));
    MPIRG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float *out = nullptr;
    MPIRG_CUDA_CHECK(cudaMalloc(&out, sizeof(float) * sms * 8));
    cudaEvent_t e0, e1;
    MPIRG_CUDA_CHECK(cudaEventCreate(&e0));
    MPIRG_CUDA_CHECK(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 8192;
    double best = 0.0, best_ms = 0.0;
    for (int variant = 0; variant < 2; ++variant)
      for (int rep = 0; rep < 4; ++rep)
      {
        MPIRG_CUDA_CHECK(cudaEventRecord(e0));
        if (variant == 0)
          ffma_peak_kernel<false><<<blocks, threads>>>(out, iters, 1.0001f, 0.9999f);
        else
          ffma_peak_kernel<true><<<blocks, threads>>>(out, iters, 1.0001f, 0.9999f);
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
