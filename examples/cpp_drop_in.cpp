// A reference-style C++ program on the B200 path: the same calls as
// proj/tests/acceptance.cpp check 2 (mp_lu<double,float> + ir_solve_report),
// with namespace mpir::gpu instead of mpir.
//   g++ -std=c++17 -Iinclude examples/cpp_drop_in.cpp -Lpaper_2311_14616_b200 -lmpir_gpu
#include <cstdio>

#include "mpir_gpu.hpp"

int main(int argc, char **argv)
{
  const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
  mpir::gpu::Matrix<double> a(n, n);
  mpirg_gen_greens_operator(n, 1.0, a.data());
  std::vector<double> ones(n, 1.0), b(n);
  mpirg_gen_matvec_compensated_f64(n, a.data(), ones.data(), b.data());
  try
  {
    mpir::gpu::FactorOptions opts;
    opts.on_the_fly = false;
    auto f = mpir::gpu::mp_lu<double, float>(a, opts);
    const auto rep = mpir::gpu::ir_solve_report(f, b);
    double err = 0.0;
    for (int i = 0; i < n; ++i)
      err = std::max(err, std::fabs(rep.sol[i] - 1.0));
    std::printf("n=%d reason=%d evals=%zu err=%.3e factor_ms=%.3f solve_ms=%.3f\n", n,
                static_cast<int>(rep.reason), rep.rhist.size(), err, f.last_factor_ms(),
                rep.device_ms);
    return (rep.reason == mpir::gpu::StopReason::SmallResidual && err <= 10 * 0x1p-52) ? 0 : 1;
  }
  catch (const mpir::gpu::Error &e)
  {
    std::printf("error: %s\n", e.what());
    return 2;
  }
}
