// Dev probe: cost of warp broadcasts inside an FFMA dependency chain (what one
// round of the TRSV diagonal solve pays), by mechanism: SHFL.IDX, shared-memory
// store + load, and how four staggered broadcasts per round pipeline.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false shfl_probe.cu -o bin/shfl_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float shfl_asm(float v, int src)
{
  float r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=f"(r) : "f"(v), "r"(src));
  return r;
}

template <int MODE>
__global__ void probe(float *out, long long *cyc, int iters)
{
  __shared__ float sm[64];
  const int lane = threadIdx.x;
  float v = 1.0f + lane * 1e-3f, a = 1.0001f, b = 1e-4f;
  float w1 = v, w2 = v, w3 = v;
  sm[lane] = v;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
  {
    const int m = i & 31;
    if constexpr (MODE == 0)
    {
      // fma -> bcast shfl
      v = __fmaf_rn(v, a, b);
      v = shfl_asm(v, m);
    }
    else if constexpr (MODE == 1)
    {
      // 4 fma chain, 4 shuffles (staggered), next round starts from the last
      const float s0 = __fmaf_rn(v, a, b);
      const float s1 = __fmaf_rn(s0, a, w1);
      const float s2 = __fmaf_rn(s1, a, w2);
      const float s3 = __fmaf_rn(s2, a, w3);
      const float x0 = shfl_asm(s0, m), x1 = shfl_asm(s1, m), x2 = shfl_asm(s2, m), x3 = shfl_asm(s3, m);
      w1 = x0;
      w2 = x1;
      w3 = x2;
      v = x3;
    }
    else if constexpr (MODE == 2)
    {
      // fma -> owner stores to smem -> everyone loads (broadcast)
      v = __fmaf_rn(v, a, b);
      if (lane == m)
        sm[0] = v;
      __syncwarp();
      v = sm[0];
      __syncwarp();
    }
    else if constexpr (MODE == 3)
    {
      // 4 fma chain then ONE shuffle of the last + three shuffles off the chain issued later
      const float s0 = __fmaf_rn(v, a, b);
      const float s1 = __fmaf_rn(s0, a, w1);
      const float s2 = __fmaf_rn(s1, a, w2);
      const float s3 = __fmaf_rn(s2, a, w3);
      v = shfl_asm(s3, m);
      w1 = s0;
      w2 = s1;
      w3 = s2;
    }
    else if constexpr (MODE == 4)
    {
      // one 64-bit-packed pair per shuffle? (two shuffles of packed halves is not possible for fp32;
      // here: 2 shuffles per round, 2-row rounds)
      const float s0 = __fmaf_rn(v, a, b);
      const float s1 = __fmaf_rn(s0, a, w1);
      const float x0 = shfl_asm(s0, m), x1 = shfl_asm(s1, m);
      w1 = x0;
      v = x1;
    }
    else if constexpr (MODE == 5)
    {
      // fma -> shfl -> fma -> shfl with lane-varying source
      v = __fmaf_rn(v, a, b);
      v = shfl_asm(v, (lane + m) & 31);
    }
    else if constexpr (MODE == 6)
    {
      // redux-style: owner value via match? use __shfl_sync builtin (compiler may pick uniform path)
      v = __fmaf_rn(v, a, b);
      v = __shfl_sync(0xffffffffu, v, m);
    }
  }
  long long t1 = clock64();
  if (lane == 0)
    cyc[MODE] = (t1 - t0) * 100 / iters;
  out[lane + 32 * MODE] = v + w1 + w2 + w3;
}

int main()
{
  float *out;
  long long *cyc;
  cudaMalloc(&out, 4096);
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  for (int r = 0; r < 2; ++r)
  {
    probe<0><<<1, 32>>>(out, cyc, 4096);
    probe<1><<<1, 32>>>(out, cyc, 4096);
    probe<2><<<1, 32>>>(out, cyc, 4096);
    probe<3><<<1, 32>>>(out, cyc, 4096);
    probe<4><<<1, 32>>>(out, cyc, 4096);
    probe<5><<<1, 32>>>(out, cyc, 4096);
    probe<6><<<1, 32>>>(out, cyc, 4096);
    cudaDeviceSynchronize();
  }
  printf("fma->bcast shfl                        : %.1f cyc/iter\n", cyc[0] / 100.0);
  printf("4 fma chain + 4 staggered bcast shfl    : %.1f cyc/iter\n", cyc[1] / 100.0);
  printf("fma->STS(owner)->LDS bcast              : %.1f cyc/iter\n", cyc[2] / 100.0);
  printf("4 fma chain + 1 bcast shfl              : %.1f cyc/iter\n", cyc[3] / 100.0);
  printf("2 fma chain + 2 staggered bcast shfl    : %.1f cyc/iter\n", cyc[4] / 100.0);
  printf("fma->shfl (lane-varying source)         : %.1f cyc/iter\n", cyc[5] / 100.0);
  printf("fma->__shfl_sync(uniform)               : %.1f cyc/iter\n", cyc[6] / 100.0);
  return 0;
}
