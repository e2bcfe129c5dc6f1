// Microbenchmark (dev tool, not product): the whole-panel speculation's
// diagonal-block factorization (lu_spec.cuh spec_diag_phase, one warp) and the
// row recurrences (spec_block_left) on one CTA, timed with clock64 and checked
// bit for bit against a sequential host LU without pivoting (fmaf / division).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -fmad=false \
//   --expt-relaxed-constexpr -I../../paper_2311_14616_b200/csrc panel_spec.cu -o bin/panel_spec
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

namespace mpirg
{
struct CudaError : std::runtime_error
{
  CudaError(cudaError_t, const char *, const char *, int) : std::runtime_error("cuda") {}
};
}  // namespace mpirg
#include "lu_spec.cuh"

using namespace mpirg;
using namespace mpirg::panel2;

constexpr int NB = 64, NTX = 256;

// A: column-major (ld = m) panel of m rows x NB columns; rows 0..63 = diagonal block.
template <int MODE>
__global__ void __launch_bounds__(NTX, 1) spec_kernel(const float *A, float *out, int m, long long *cyc, int *flags)
{
  extern __shared__ __align__(16) unsigned char dsm[];
  auto &sh = *reinterpret_cast<SpecShared<NB> *>(dsm);
  float *stash = reinterpret_cast<float *>(dsm + a16(sizeof(SpecShared<NB>))) + threadIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int NBLK = NB / 8;
  if (t == 0)
  {
    sh.prog = 0;
    sh.abort = 0;
    sh.zj = NB;
  }
  __syncthreads();
  bool beaten = false, stop = false;
  const long long t0 = clock64();
  if (warp == 0)
  {
    float D[2][NBLK][8];
#pragma unroll
    for (int c = 0; c < NB; ++c)
    {
      D[0][c / 8][c % 8] = A[(size_t)c * m + lane];
      D[1][c / 8][c % 8] = A[(size_t)c * m + lane + 32];
    }
    int zj = NB;
    const long long t1 = clock64();
    spec_diag_phase<NB, 0>(D, sh, lane, true, beaten, zj, stop);
    const long long t2 = clock64();
    spec_diag_phase<NB, 1>(D, sh, lane, true, beaten, zj, stop);
    const long long t3 = clock64();
    if (lane == 0)
    {
      cyc[0] = t1 - t0;
      cyc[1] = t2 - t1;
      cyc[2] = t3 - t2;
      flags[0] = sh.abort;
    }
  }
  if (MODE == 1 && warp != 0)
  {
    // rows 64 + (warp - 1) * 32 + lane ... one row per thread of warps 1..7
    const int row = 64 + (warp - 1) * 32 + lane;
    bool act[1] = {row < m};
    for (int c = 0; c < NB; ++c)
      stash[(size_t)c * NTX] = act[0] ? A[(size_t)c * m + row] : 0.0f;
    for (int b = 0; b < NBLK; ++b)
    {
      while (sh.prog < 8 * (b + 1) && !sh.abort)
        __nanosleep(40);
      if (sh.abort)
        break;
      __threadfence_block();
      spec_rows_block<NB, 1, NTX>(stash, act, sh.U, b, beaten);
    }
    if (t == NTX - 1)
      cyc[3] = clock64() - t0;
    if (act[0])
      for (int c = 0; c < NB; ++c)
        out[(size_t)c * m + row] = stash[(size_t)c * NTX];
    if (beaten)
      flags[1] = 1;
  }
  __syncthreads();
  for (int idx = t; idx < NB * NB; idx += NTX)
  {
    const int c = idx / NB, r = idx - c * NB;
    out[(size_t)c * m + r] = c >= r ? sh.U[r][c] : sh.Dg[r][c];
  }
}

int main()
{
  const int m = 64 + 7 * 32;
  std::vector<float> A((size_t)m * NB), ref;
  srand(7);
  for (int i = 0; i < m; ++i)
    for (int c = 0; c < NB; ++c)
      A[(size_t)c * m + i] = (float)rand() / RAND_MAX - 0.5f + (i == c ? 40.0f : 0.0f);
  ref = A;
  for (int k = 0; k < NB; ++k)
    for (int i = k + 1; i < m; ++i)
    {
      const float l = ref[(size_t)k * m + i] / ref[(size_t)k * m + k];
      ref[(size_t)k * m + i] = l;
      for (int c = k + 1; c < NB; ++c)
        ref[(size_t)c * m + i] = fmaf(-l, ref[(size_t)c * m + k], ref[(size_t)c * m + i]);
    }
  float *dA, *dout;
  long long *cyc;
  int *flags;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dout, A.size() * 4);
  cudaMallocManaged(&cyc, 64);
  cudaMallocManaged(&flags, 16);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = spec_dyn_smem<NB, 1, NTX>();
  cudaFuncSetAttribute(spec_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(spec_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 2; ++rep)
    {
      memset(cyc, 0, 64);
      flags[0] = flags[1] = 0;
      cudaMemset(dout, 0, A.size() * 4);
      if (mode == 0)
        spec_kernel<0><<<1, NTX, smem>>>(dA, dout, m, cyc, flags);
      else
        spec_kernel<1><<<1, NTX, smem>>>(dA, dout, m, cyc, flags);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> got(A.size());
      cudaMemcpy(got.data(), dout, A.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      const int rows = (mode & 1) == 0 ? 64 : m;
      for (int i = 0; i < rows; ++i)
        for (int c = 0; c < NB; ++c)
          bad += memcmp(&got[(size_t)c * m + i], &ref[(size_t)c * m + i], 4) != 0;
      if (rep == 1)
        printf("%s: load %lld  phase0 %lld  phase1 %lld  (diag total %lld, %.0f per step)  rows done at %lld  "
               "mismatches %d  abort %d beaten %d  %s\n",
               mode == 0 ? "diag warp alone   " : "diag + 7 row warps", cyc[0], cyc[1], cyc[2], cyc[1] + cyc[2],
               (cyc[1] + cyc[2]) / 64.0, cyc[3], bad, flags[0], flags[1], e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
