// Device-side problem generator: the Green's operator
// A = I - alpha G of proj/src/greens.cpp:11-59, written straight into device
// memory so config 5a's 34 GB matrix never has to be generated on the host
// and copied.
//
// Bitwise equal to the reference's build_operator: every entry is a fixed
// sequence of single IEEE operations (grid point i*h with the endpoint pinned
// to 1.0, the kernel y(1-x) or x(1-y), the trapezoid weight, the sign-flipped
// scaling, and 1.0 added on the diagonal after a store), spelled here with the
// _rn intrinsics so nothing is contracted. tests/test_gpu_kernels.py compares
// it with the host generator (which is pinned to the reference's own).
#include <cuda_runtime.h>

#include "../../include/mpir_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace mpirg
{
namespace
{
__device__ __forceinline__ double grid_point(int i, int n, double h)
{
  return i == n - 1 ? 1.0 : __dmul_rn((double)i, h);  // greens.cpp:21-24
}

__global__ void greens_operator_kernel(int n, double alpha, double h, int col0, int ncols,
                                       double *__restrict__ out, size_t ld)
{
  const int j = col0 + blockIdx.y;
  if (blockIdx.y >= ncols)
    return;
  const double y = grid_point(j, n, h);
  const double w = (j == 0 || j == n - 1) ? __dmul_rn(0.5, h) : h;  // greens.cpp:36
  double *c = out + (size_t)blockIdx.y * ld;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    const double x = grid_point(i, n, h);
    // greens.cpp:11-14: x > y ? y (1 - x) : x (1 - y)
    const double k = x > y ? __dmul_rn(y, __dsub_rn(1.0, x)) : __dmul_rn(x, __dsub_rn(1.0, y));
    const double g = __dmul_rn(k, w);              // greens.cpp:39
    double v = __dmul_rn(-alpha, g);               // greens.cpp:54
    if (i == j)
      v = __dadd_rn(v, 1.0);                       // greens.cpp:55
    c[i] = v;
  }
}
}  // namespace
}  // namespace mpirg

// Columns [col0, col0 + ncols) of I - alpha G (n x n) into out (device,
// column-major, leading dimension ld >= n: out[c * ld + i] is entry (i, col0 + c)).
extern "C" int mpirg_gen_greens_operator_device(int n, double alpha, int col0, int ncols,
                                                double *out, size_t ld, void *stream)
{
  using namespace mpirg;
  if (n < 3 || col0 < 0 || ncols < 0 || col0 + ncols > n || ld < (size_t)n || !out)
    return MPIRG_ERR_INVALID_SIZE;
  if (ncols == 0)
    return MPIRG_OK;
  const double h = 1.0 / (n - 1);  // greens.cpp:19 (host division, as in the reference)
  auto s = static_cast<cudaStream_t>(stream);
  const int gx = std::min(64, (n + 255) / 256);
  for (int c = 0; c < ncols; c += 65535)
  {
    const int nc = std::min(65535, ncols - c);
    greens_operator_kernel<<<dim3(gx, nc), 256, 0, s>>>(n, alpha, h, col0 + c, nc,
                                                        out + (size_t)c * ld, ld);
  }
  return cudaGetLastError() == cudaSuccess ? MPIRG_OK : MPIRG_ERR_CUDA;
}
