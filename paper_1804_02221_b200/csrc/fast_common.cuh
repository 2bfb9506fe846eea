// fast_common.cuh — device helpers shared by the fast-mode translation units
// (kernels_fast.cu and the kernels_pl_*.cu instantiations of stage_pl.cuh).
// Every TU that includes this gets its own copy of the constant operator table
// (internal linkage); upload_fast_ops fills all of them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fast_math.cuh"
#include "ptx_async.cuh"
#include "swdg_device.cuh"
#include "swdg_launch.h"

namespace swdg_dev {
extern int g_grid_cap;  // kernels_common.cu; 0 = no cap (test hook)
namespace {

// ---- constant operator tables --------------------------------------------
// per n1 = 2..16: D, Dtilde/4, Dtilde/8, Dhat, Vinv (n1^2 each) and w (n1)
__host__ __device__ constexpr int ops_offset(int n1) {
  int off = 0;
  for (int k = 2; k < n1; ++k) off += 5 * k * k + k;
  return off;
}
constexpr int kOpsTotal = ops_offset(17);
__constant__ double c_ops[kOpsTotal];  // per TU (anonymous namespace)

template <int N1>
struct Ops {
  static constexpr int base = ops_offset(N1);
  static __device__ __forceinline__ double D(int a, int b) { return c_ops[base + a * N1 + b]; }
  static __device__ __forceinline__ double D4(int a, int b) {
    return c_ops[base + N1 * N1 + a * N1 + b];
  }
  static __device__ __forceinline__ double D8(int a, int b) {
    return c_ops[base + 2 * N1 * N1 + a * N1 + b];
  }
  static __device__ __forceinline__ double Dh(int a, int b) {
    return c_ops[base + 3 * N1 * N1 + a * N1 + b];
  }
  static __device__ __forceinline__ double Vinv(int a, int b) {
    return c_ops[base + 4 * N1 * N1 + a * N1 + b];
  }
  static __device__ __forceinline__ double w(int a) { return c_ops[base + 5 * N1 * N1 + a]; }
};


__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// Minus-side outward normal and J_surf from the face metrics (compute_metrics,
// mesh.hpp:192-218): E/W faces take (y_eta, x_eta), S/N faces (y_xi, x_xi).
// One reciprocal square root; explicit _rn operations: bitwise the same on both
// sides of the face.
__device__ __forceinline__ void face_normal(int face, double m0, double m1, double& nx,
                                            double& ny, double& js) {
  const double m2 = __fma_rn(m0, m0, __dmul_rn(m1, m1));
  const double ri = frsqrt(m2);
  js = __dmul_rn(m2, ri);
  const double s = (face == 1 || face == 0) ? 1.0 : -1.0;  // E,S: +(m0,-m1); W,N: -(m0,-m1)
  nx = __dmul_rn(s * m0, ri);
  ny = __dmul_rn(-s * m1, ri);
}

// entropy-stable normal flux (fluxes.hpp:136-166) from both sides' states,
// velocities and wave speeds, algebraically simplified: R|Lambda|R^T applied
// directly (the zero/one entries of R dropped).
__device__ __forceinline__ void es_flux_pre(double hm, double um, double vm, double cm,
                                            double hp, double up, double vp, double cp,
                                            double bm, double bp, double nx, double ny,
                                            double g, double inv2g, double& f0, double& f1,
                                            double& f2) {
  const double unm = nx * um + ny * vm, utm = nx * vm - ny * um;
  const double unp = nx * up + ny * vp, utp = nx * vp - ny * up;
  const double havg = 0.5 * (hm + hp);
  const double h2avg = 0.5 * (hm * hm + hp * hp);
  const double uavg = 0.5 * (unm + unp), vavg = 0.5 * (utm + utp);
  const double cavg = 0.5 * (cm + cp);
  const double hu_ = havg * uavg;
  double a0 = hu_;
  double a1 = hu_ * uavg + 0.5 * g * h2avg;
  double a2 = hu_ * vavg;
  const double x1 = unp - unm, x2 = utp - utm;
  const double x0 = g * ((hp + bp) - (hm + bm)) - 0.5 * (x1 * (unp + unm)) -
                    0.5 * (x2 * (utp + utm));
  const double r10 = uavg + cavg, r12 = uavg - cavg;
  const double y0 = inv2g * fabs(r10) * (x0 + r10 * x1 + vavg * x2);
  const double y1 = fabs(hu_) * x2;
  const double y2 = inv2g * fabs(r12) * (x0 + r12 * x1 + vavg * x2);
  a0 -= 0.5 * (y0 + y2);
  a1 -= 0.5 * (r10 * y0 + r12 * y2);
  a2 -= 0.5 * (vavg * (y0 + y2) + y1);
  f0 = a0;
  f1 = nx * a1 - ny * a2;
  f2 = ny * a1 + nx * a2;
}

__device__ __forceinline__ void es_flux_fast(double hm, double hum, double hvm, double hp,
                                             double hup, double hvp, double bm, double bp,
                                             double nx, double ny, double g, double inv2g,
                                             double h_des, double& f0, double& f1,
                                             double& f2) {
  double um, vm, up, vp;
  vel(hm, hum, hvm, h_des, um, vm);
  vel(hp, hup, hvp, h_des, up, vp);
  es_flux_pre(hm, um, vm, wave_c(g, hm), hp, up, vp, wave_c(g, hp), bm, bp, nx, ny, g, inv2g,
              f0, f1, f2);
}

__device__ __forceinline__ uint32_t round16(size_t b) { return (uint32_t)((b + 15) & ~size_t(15)); }

// Per-device launch state: the dynamic shared-memory attribute and the
// occupancy are properties of (kernel, device context), so they are cached per
// device ordinal (a process may drive several B200s).
constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  return dev;
}

inline int device_sms(int dev) {
  static int sms[kMaxDevices] = {};
  if (sms[dev] == 0) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev];
}

// persistent grid: resident CTAs over all SMs (capped at the group count).
// `reserve_sms` SMs are left free for concurrent work (the halo exchange's
// NCCL kernels while a partition's interior runs).
template <class KERN>
int grid_for(KERN kern, int threads, size_t bytes, int groups, int (&cache)[kMaxDevices],
             int reserve_sms = 0) {
  const int dev = current_device();
  if (dev < 0) return 0;
  if (cache[dev] == 0) {  // resident CTAs per SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, bytes);
    cache[dev] = per_sm > 0 ? per_sm : 1;
  }
  const int sms = device_sms(dev);
  const int use = reserve_sms > 0 && reserve_sms < sms ? sms - reserve_sms : sms;
  int grid = cache[dev] * use;
  if (groups < grid) grid = groups;
  // test hook (swdg_gpu_set_grid_cap): fewer CTAs, so each loops over many groups
  if (g_grid_cap > 0 && grid > g_grid_cap) grid = g_grid_cap;
  return grid;
}

// this TU's copy of the operator tables
inline int upload_ops_local(int base, const double* tab, int len) {
  return cudaMemcpyToSymbol(c_ops, tab, len * sizeof(double), base * sizeof(double)) ==
                 cudaSuccess ? 0 : -2;
}

}  // namespace
}  // namespace swdg_dev
