// Microbenchmark (dev tool, not product): latency of the warp-level
// diagonal-tile solve of trsv.cu for LPL rows per lane, and of a SHFL.IDX /
// FFMA dependency chain. Build: nvcc -arch=sm_100a -O3 diag.cu -o diag
#include <cstdio>
#include <cuda_runtime.h>

__global__ void shfl_chain(float *out, int iters, long long *cyc)
{
  float v = threadIdx.x;
  int src = (threadIdx.x * 7) & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
  {
    v = __shfl_sync(0xffffffffu, v, (src + i) & 31);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0)
    cyc[0] = (t1 - t0) / iters;
  out[threadIdx.x] = v;
}

__global__ void ffma_chain(float *out, int iters, long long *cyc)
{
  float v = threadIdx.x, a = 1.0001f, b = 0.9999f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    v = __fmaf_rn(v, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0)
    cyc[1] = (t1 - t0) / iters;
  out[threadIdx.x] = v;
}

template <int TB, int LPL>
__global__ void diag_solve(const float *L, float *out, int reps, long long *cyc)
{
  extern __shared__ float dsm[];
  float (*diag)[TB] = reinterpret_cast<float (*)[TB]>(dsm);
  for (int i = threadIdx.x; i < TB * TB; i += blockDim.x)
    diag[i / TB][i % TB] = L[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  constexpr int NL = TB / LPL;
  const int ln = lane < NL ? lane : 0;
  float a[LPL];
  for (int e = 0; e < LPL; ++e)
    a[e] = 1.0f + 0.001f * (LPL * ln + e);
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
  {
#pragma unroll 2
    for (int m = 0; m < NL; ++m)
    {
      const int k0r = LPL * m;
      float lt[LPL][LPL];
#pragma unroll
      for (int f = 0; f < LPL; ++f)
#pragma unroll
        for (int e = 0; e < LPL; ++e)
          lt[f][e] = diag[k0r + f][LPL * ln + e];
      float s[LPL], xv[LPL];
#pragma unroll
      for (int e = 0; e < LPL; ++e)
        s[e] = a[e];
#pragma unroll
      for (int e = 0; e < LPL; ++e)
      {
#pragma unroll
        for (int f = 0; f < e; ++f)
          s[e] = __fmaf_rn(-lt[f][e], s[f], s[e]);
        xv[e] = __shfl_sync(0xffffffffu, s[e], m);
      }
      const bool later = lane > m;
#pragma unroll
      for (int e = 0; e < LPL; ++e)
      {
        float v = a[e];
#pragma unroll
        for (int f = 0; f < LPL; ++f)
          v = __fmaf_rn(-lt[f][e], xv[f], v);
        a[e] = later ? v : (lane == m ? s[e] : a[e]);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0)
    cyc[2 + (LPL == 8 ? 1 : LPL == 2 ? 2 : 0)] = (t1 - t0) / reps;
  float acc = 0;
  for (int e = 0; e < LPL; ++e)
    acc += a[e];
  out[threadIdx.x] = acc;
}

int main()
{
  float *L, *out;
  long long *cyc;
  cudaMalloc(&L, 128 * 128 * 4);
  cudaMemset(L, 0, 128 * 128 * 4);
  cudaMalloc(&out, 1024 * 4);
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  cudaFuncSetAttribute(diag_solve<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(diag_solve<128, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int r = 0; r < 2; ++r)
  {
    shfl_chain<<<1, 32>>>(out, 10000, cyc);
    ffma_chain<<<1, 32>>>(out, 10000, cyc);
    diag_solve<128, 4><<<1, 32, 65536>>>(L, out, 100, cyc);
    diag_solve<128, 8><<<1, 32, 65536>>>(L, out, 100, cyc);
    diag_solve<64, 2><<<1, 32, 16384>>>(L, out, 100, cyc);
    cudaDeviceSynchronize();
  }
  printf("shfl latency %lld cyc, ffma latency %lld cyc\n", cyc[0], cyc[1]);
  printf("diag TB=128 LPL=4: %lld cyc/block (%lld per round)\n", cyc[2], cyc[2] / 32);
  printf("diag TB=128 LPL=8: %lld cyc/block (%lld per round)\n", cyc[3], cyc[3] / 16);
  printf("diag TB=64 LPL=2: %lld cyc/block (%lld per round)\n", cyc[4], cyc[4] / 32);
  return 0;
}
