// fast_math.cuh — the fast-mode reciprocal, square root and velocity shared by
// the stage kernels (kernels_fast.cu) and the fast step reductions
// (kernels_step.cu), so both compute identical bits from identical inputs.
#pragma once

#include <cuda_runtime.h>

namespace swdg_dev {
namespace {

// Fast reciprocal and reciprocal square root: the MUFU seed (rcp/rsqrt.approx)
// refined by two Newton steps in explicit round-to-nearest operations — within
// an ulp of the IEEE result, branch-free (no slow path), and bitwise identical
// at every call site (both sides of a face must see the same numbers).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}
__device__ __forceinline__ double frsqrt(double x) {  // x > 0
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = __fma_rn(-__dmul_rn(x, y), y, 1.0);
  y = __fma_rn(__dmul_rn(0.5, y), e, y);
  e = __fma_rn(-__dmul_rn(x, y), y, 1.0);
  return __fma_rn(__dmul_rn(0.5, y), e, y);
}
// sqrt(max(x, 0))
__device__ __forceinline__ double fsqrt0(double x) {
  return x > 0.0 ? __dmul_rn(x, frsqrt(x)) : 0.0;
}

// velocity desingularisation (physics.hpp:23-36): hard cut below h_des
// (branch-free: the reciprocal of the clamped height, then a select)
__device__ __forceinline__ void vel(double h, double hu, double hv, double h_des, double& u,
                                    double& v) {
  const bool wet = h >= h_des;
  const double r = frcp(wet ? h : 1.0);
  u = wet ? __dmul_rn(hu, r) : 0.0;
  v = wet ? __dmul_rn(hv, r) : 0.0;
}

// gravity wave speed sqrt(g max(h, 0)) (fluxes.hpp:150)
__device__ __forceinline__ double wave_c(double g, double h) {
  return fsqrt0(__dmul_rn(g, h));
}

}  // namespace
}  // namespace swdg_dev
