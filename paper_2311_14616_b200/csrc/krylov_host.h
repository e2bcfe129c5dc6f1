// Host scalar helpers of the GMRES correction (krylov_host.cpp).
#pragma once

#include <cstddef>

namespace mpirg
{
// The reference build vectorises its sequential reductions (dot, nrm2, the
// small back substitution) as fold-left reductions: the first
// reduction_unfused(count, ...) terms are rounded products added in order, the
// scalar tail is fused. half_step: the epilogue also takes a half vector.
int reduction_unfused(int count, int elem_bytes, bool half_step);
// Applies the stored rotations to Hessenberg column j (entries 0..j+1 filled),
// forms rotation j, updates g; returns |g[j+1]| (the residual estimate).
template <typename T>
double gmres_rotate(T *hess, int ld, T *cs, T *sn, T *g, int j);
// y = R^-1 g for the leading k x k triangle; true if a zero diagonal was met.
template <typename T>
bool gmres_backsolve(const T *hess, int ld, const T *g, T *y, int k);
template <typename T>
T host_sqrt(T v);
template <typename T>
T host_recip(T v);
}  // namespace mpirg
