// kernels_fast.cu — the throughput path (SWDG_MODE_FAST): one fused kernel per
// SSPRK3 stage on sm_100a, FP64 with FMA.
//
// Mapping: a CTA holds E elements; every element gets 2*(N+1) "line threads":
// thread l < N+1 owns the xi-line j=l, thread l >= N+1 the eta-line i=l-(N+1).
// A line thread keeps its line's nodal data and accumulators in registers and
// runs the split-form flux differencing (dg_rhs.hpp:23-71) over the UNORDERED
// node pairs of its line: the two-point flux F#(a,b) and the averaged metrics
// are symmetric, so each pair is evaluated once and scattered
// to both nodes with Dtilde(a,b) and Dtilde(b,a) — 19 DP instructions per
// pair instead of 2x16.  The same thread then adds its share of the split
// bathymetry source (dg_rhs.hpp:154-183: the xi or eta half) and the
// entropy-stable interface flux (fluxes.hpp:136-166) at its two line
// endpoints, which are exactly the element's face nodes.  After one barrier
// the node phase sums the xi/eta accumulators, applies -1/J, the SSPRK3
// update (timeloop.hpp:114-127), the element mean / Zhang-Shu limiter /
// dry-node zeroing (limiter.hpp:24-84) and the reject signal
// (timeloop.hpp:205-209), and writes the stage output once.  HBM traffic per
// node and stage: state in (24 B), W^n (24 B, stages 2-3), 6 geometry fields
// (48 B), state out (24 B) — face traces of neighbours are L2 hits.
//
// Operators live in __constant__ memory, one table set per N, so the fully
// unrolled pair loops issue DFMA with constant-bank operands.
#include <cuda_runtime.h>

#include <cstring>

#include "swdg_device.cuh"
#include "swdg_launch.h"

namespace swdg_dev {

// ---- constant operator tables --------------------------------------------
// per n1 = 2..16: D, Dtilde/4, Dtilde/8, Dhat, Vinv (n1^2 each) and w (n1)
__host__ __device__ constexpr int ops_offset(int n1) {
  int off = 0;
  for (int k = 2; k < n1; ++k) off += 5 * k * k + k;
  return off;
}
constexpr int kOpsTotal = ops_offset(17);
__constant__ double c_ops[kOpsTotal];

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

namespace {

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ void vel(double h, double hu, double hv, double h_des, double& u,
                                    double& v) {
  if (h >= h_des) {
    const double r = 1.0 / h;
    u = hu * r;
    v = hv * r;
  } else {
    u = 0.0;
    v = 0.0;
  }
}

// entropy-stable normal flux (fluxes.hpp:136-166), algebraically simplified:
// R|Lambda|R^T applied directly (the zero/one entries of R dropped).
__device__ __forceinline__ void es_flux_fast(double hm, double hum, double hvm, double hp,
                                             double hup, double hvp, double bm, double bp,
                                             double nx, double ny, double g, double inv2g,
                                             double h_des, double& f0, double& f1,
                                             double& f2) {
  double um, vm, up, vp;
  vel(hm, hum, hvm, h_des, um, vm);
  vel(hp, hup, hvp, h_des, up, vp);
  const double unm = nx * um + ny * vm, utm = nx * vm - ny * um;
  const double unp = nx * up + ny * vp, utp = nx * vp - ny * up;
  const double havg = 0.5 * (hm + hp);
  const double h2avg = 0.5 * (hm * hm + hp * hp);
  const double uavg = 0.5 * (unm + unp), vavg = 0.5 * (utm + utp);
  const double cavg = 0.5 * (sqrt(g * smax(hm, 0.0)) + sqrt(g * smax(hp, 0.0)));
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

// shared-memory slots per element: 10 nodal fields + 6 accumulators + 8 per
// line thread for the element reductions
template <int N1>
struct Smem {
  static constexpr int NP = N1 * N1;
  static constexpr int H = 0, U = 1, V = 2, HU = 3, HV = 4, YE = 5, XE = 6, YX = 7, XX = 8,
                       B = 9, AX = 10, AY = 13;
  static constexpr int kFields = 16;
  static constexpr int kRed = 8;
  static constexpr int per_elem = kFields * NP + kRed * 2 * N1;
};

template <int N1>
constexpr int elems_per_block() {
  return (128 / (2 * N1)) > 0 ? (128 / (2 * N1)) : 1;
}

// One RK stage for N1 <= 8 (a whole line in registers).
template <int N1, bool FORCE>
__global__ void __launch_bounds__(2 * N1 * elems_per_block<N1>())
    k_stage_lines(Mesh M, Phys P, StageArgs A, Flags* F) {
  constexpr int NP = N1 * N1, T = 2 * N1, E = elems_per_block<N1>();
  using S = Smem<N1>;
  using O = Ops<N1>;
  extern __shared__ double smem[];
  const int el = threadIdx.x / T, lt = threadIdx.x % T;
  const int e = blockIdx.x * E + el;
  const bool active = e < M.n_owned;
  double* sm = smem + el * S::per_elem;
  const long long base = (long long)e * NP;
  const double g = P.g, h_des = P.h_des;

  // ---- load phase: element fields -> smem (coalesced across the element)
  if (active) {
#pragma unroll 4
    for (int k = lt; k < NP; k += T) {
      const long long n = base + k;
      const double h = A.in.h[n], hu = A.in.hu[n], hv = A.in.hv[n];
      double u, v;
      vel(h, hu, hv, h_des, u, v);
      sm[S::H * NP + k] = h;
      sm[S::U * NP + k] = u;
      sm[S::V * NP + k] = v;
      sm[S::HU * NP + k] = hu;
      sm[S::HV * NP + k] = hv;
      sm[S::YE * NP + k] = M.ye[n];
      sm[S::XE * NP + k] = M.xe[n];
      sm[S::YX * NP + k] = M.yx[n];
      sm[S::XX * NP + k] = M.xx[n];
      sm[S::B * NP + k] = M.b[n];
    }
  }
  __syncthreads();

  // ---- line phase
  if (active) {
    const bool xi = lt < N1;
    const int li = xi ? lt : lt - N1;
    // node k of this line: xi-line j=li -> (k, li); eta-line i=li -> (li, k)
    auto idx = [&](int k) { return xi ? k * N1 + li : li * N1 + k; };
    double h[N1], u[N1], v[N1], hu[N1], hv[N1], Am[N1], Bm[N1];
    double r0[N1], r1[N1], r2[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int q = idx(k);
      h[k] = sm[S::H * NP + q];
      u[k] = sm[S::U * NP + q];
      v[k] = sm[S::V * NP + q];
      hu[k] = sm[S::HU * NP + q];
      hv[k] = sm[S::HV * NP + q];
      Am[k] = xi ? sm[S::YE * NP + q] : -sm[S::YX * NP + q];
      Bm[k] = xi ? sm[S::XE * NP + q] : -sm[S::XX * NP + q];
      r0[k] = r1[k] = r2[k] = 0.0;
    }
    const double g2 = 2.0 * g;
    // volume: unordered pairs (a<b) plus the two corner diagonals
#pragma unroll
    for (int a = 0; a < N1; ++a) {
#pragma unroll
      for (int b = a; b < N1; ++b) {
        if (a == b && a != 0 && a != N1 - 1) continue;  // Dtilde(i,i) = 0 inside
        const double Shu = hu[a] + hu[b], Shv = hv[a] + hv[b];
        const double Su = u[a] + u[b], Sv = v[a] + v[b];
        const double SA = Am[a] + Am[b], SB = Bm[a] + Bm[b];
        const double F0 = SA * Shu - SB * Shv;  // 4*Ftilde_0
        const double Q = g2 * h[a] * h[b];
        const double T1 = Su * F0 + Q * SA;     // 8*Ftilde_1
        const double T2 = Sv * F0 - Q * SB;     // 8*Ftilde_2
        r0[a] += O::D4(a, b) * F0;
        r1[a] += O::D8(a, b) * T1;
        r2[a] += O::D8(a, b) * T2;
        if (a != b) {
          r0[b] += O::D4(b, a) * F0;
          r1[b] += O::D8(b, a) * T1;
          r2[b] += O::D8(b, a) * T2;
        }
      }
    }
    // split bathymetry source, this direction's half (dg_rhs.hpp:171-176)
    {
      double bb[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) bb[k] = sm[S::B * NP + idx(k)];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double db = 0.0, dAb = 0.0, dBb = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const double d = O::D(k, m);
          db += d * bb[m];
          dAb += d * (Am[m] * bb[m]);
          dBb += d * (Bm[m] * bb[m]);
        }
        const double hg2 = 0.5 * g * h[k];
        r1[k] += hg2 * (Am[k] * db + dAb);
        r2[k] -= hg2 * (Bm[k] * db + dBb);
      }
    }
    // interface fluxes at the two line endpoints (dg_rhs.hpp:202-252)
    const double inv2g = 1.0 / (2.0 * g), iw0 = 1.0 / M.w0;
#pragma unroll
    for (int end = 0; end < 2; ++end) {
      const int k = end ? N1 - 1 : 0;
      const int face = xi ? (end ? 1 : 3) : (end ? 2 : 0);
      const int t = li;
      const int4 ef = M.ef[e * 4 + face];
      if (!(ef.y & EF_PRESENT)) continue;
      const double hm = h[k], hum = hu[k], hvm = hv[k], bo = sm[S::B * NP + idx(k)];
      double f0, f1, f2, js, sgn;
      if (ef.y & EF_WALL) {
        const long long fi = ((long long)e * 4 + face) * N1 + t;
        const double nx = M.fnx[fi], ny = M.fny[fi];
        js = M.fjs[fi];
        const double mn = hum * nx + hvm * ny;
        es_flux_fast(hm, hum, hvm, hm, hum - 2.0 * mn * nx, hvm - 2.0 * mn * ny, bo, bo, nx,
                     ny, g, inv2g, h_des, f0, f1, f2);
        sgn = 1.0;
      } else {
        const int nf = ef.y & EF_NBR_FACE_MASK;
        const int tp = (ef.y & EF_REVERSED) ? N1 - 1 - t : t;
        const long long nb = (long long)ef.x * NP + face_node(N1, nf, tp);
        const double hn = A.in.h[nb], hun = A.in.hu[nb], hvn = A.in.hv[nb], bn = M.b[nb];
        if (ef.y & EF_MINUS) {
          const long long fi = ((long long)e * 4 + face) * N1 + t;
          const double nx = M.fnx[fi], ny = M.fny[fi];
          js = M.fjs[fi];
          es_flux_fast(hm, hum, hvm, hn, hun, hvn, bo, bn, nx, ny, g, inv2g, h_des, f0, f1, f2);
          sgn = 1.0;
        } else {
          const long long fi = ((long long)ef.x * 4 + nf) * N1 + tp;
          const double nx = M.fnx[fi], ny = M.fny[fi];
          js = M.fjs[fi];
          es_flux_fast(hn, hun, hvn, hm, hum, hvm, bn, bo, nx, ny, g, inv2g, h_des, f0, f1, f2);
          sgn = -1.0;
        }
      }
      const double c = sgn * js * iw0;
      r0[k] += c * f0;
      r1[k] += c * f1;
      r2[k] += c * f2;
    }
    // publish this line's accumulators
    const int acc = xi ? S::AX : S::AY;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int q = idx(k);
      sm[(acc + 0) * NP + q] = r0[k];
      sm[(acc + 1) * NP + q] = r1[k];
      sm[(acc + 2) * NP + q] = r2[k];
    }
  }
  __syncthreads();

  // ---- node phase: dW/dt, SSPRK3 update, element mean
  double* red = sm + S::kFields * NP + lt * S::kRed;
  if (active) {
    double s_area = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0, mmin = 1.0e300;
#pragma unroll 2
    for (int k = lt; k < NP; k += T) {
      const long long n = base + k;
      const double jac = M.jac[n];
      const double ij = -1.0 / jac;
      double rh = (sm[S::AX * NP + k] + sm[S::AY * NP + k]) * ij;
      double rhu = (sm[(S::AX + 1) * NP + k] + sm[(S::AY + 1) * NP + k]) * ij;
      double rhv = (sm[(S::AX + 2) * NP + k] + sm[(S::AY + 2) * NP + k]) * ij;
      if (FORCE) {
        rh += A.fh[n];
        rhu += A.fhu[n];
        rhv += A.fhv[n];
      }
      if (A.rhs.h) {
        A.rhs.h[n] = rh;
        A.rhs.hu[n] = rhu;
        A.rhs.hv[n] = rhv;
      }
      double sh = sm[S::H * NP + k] + A.dt * rh;
      double shu = sm[S::HU * NP + k] + A.dt * rhu;
      double shv = sm[S::HV * NP + k] + A.dt * rhv;
      if (A.stage > 0) {
        sh = A.ca * A.wn.h[n] + A.cb * sh;
        shu = A.ca * A.wn.hu[n] + A.cb * shu;
        shv = A.ca * A.wn.hv[n] + A.cb * shv;
      }
      sm[S::H * NP + k] = sh;
      sm[S::HU * NP + k] = shu;
      sm[S::HV * NP + k] = shv;
      const int i = k / N1, j = k % N1;
      const double wj = O::w(i) * O::w(j) * jac;
      s_area += wj;
      s0 += wj * sh;
      s1 += wj * shu;
      s2 += wj * shv;
      mmin = smin(mmin, sh);
    }
    red[0] = s_area;
    red[1] = s0;
    red[2] = s1;
    red[3] = s2;
    red[4] = mmin;
  }
  __syncthreads();

  // ---- limiter (limit_element, limiter.hpp:43-84) and write-out.  No early
  // returns before the last barrier: every thread of the block reaches it.
  bool lim = active && A.update;
  double area = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, mmin = 1.0e300;
  const double* red0 = sm + S::kFields * NP;
  if (lim) {
#pragma unroll
    for (int q = 0; q < T; ++q) {
      area += red0[q * S::kRed + 0];
      a0 += red0[q * S::kRed + 1];
      a1 += red0[q * S::kRed + 2];
      a2 += red0[q * S::kRed + 3];
      mmin = smin(mmin, red0[q * S::kRed + 4]);
    }
  }
  const double inv = 1.0 / area;
  const double avg0 = inv * a0, avg1 = inv * a1, avg2 = inv * a2;
  if (lim && avg0 < 0.0) {
    if (lt == 0) {
      atomicExch(&F->reject, 1);
      if (!P.limiter) atomicExch(&F->abort, 1);
    }
    lim = false;
  }
  double theta = 1.0;
  if (lim && P.limiter && mmin < 0.0) {
    const double denom = avg0 - mmin;
    theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
  }
  if (lim && !P.limiter && mmin < 0.0 && lt == 0) atomicExch(&F->abort, 1);
  double mine = 1.0e300;
  if (lim) {
    for (int k = lt; k < NP; k += T) {
      const long long n = base + k;
      double sh = sm[S::H * NP + k], shu = sm[S::HU * NP + k], shv = sm[S::HV * NP + k];
      if (theta < 1.0) {
        sh = smax(theta * (sh - avg0) + avg0, 0.0);
        shu = theta * (shu - avg1) + avg1;
        shv = theta * (shv - avg2) + avg2;
      }
      if (P.limiter && sh < P.h_tol) {
        shu = 0.0;
        shv = 0.0;
      }
      A.out.h[n] = sh;
      A.out.hu[n] = shu;
      A.out.hv[n] = shv;
      mine = smin(mine, sh);
    }
  }
  red[5] = mine;
  __syncthreads();
  // per-element min and limited count, one atomic per element
  if (lim && lt == 0) {
    double m = red0[5];
    for (int q = 1; q < T; ++q) m = smin(m, red0[q * S::kRed + 5]);
    atomicMin(&F->min_h_key, order_key(m));
    if (theta < 1.0) atomicAdd(&F->n_limited, 1);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
static bool g_ops_set[17];
static double g_ops_host[kOpsTotal];

int upload_fast_ops(int n1, const double* D, const double* Dt, const double* Dh,
                    const double* Vinv, const double* w) {
  const int base = ops_offset(n1), np = n1 * n1;
  double tab[5 * 256 + 16];
  for (int k = 0; k < np; ++k) {
    tab[k] = D[k];
    tab[np + k] = 0.25 * Dt[k];
    tab[2 * np + k] = 0.125 * Dt[k];
    tab[3 * np + k] = Dh[k];
    tab[4 * np + k] = Vinv[k];
  }
  for (int k = 0; k < n1; ++k) tab[5 * np + k] = w[k];
  const int len = 5 * np + n1;
  if (g_ops_set[n1]) {
    if (std::memcmp(tab, g_ops_host + base, len * sizeof(double)) != 0) return -1;
    return 0;
  }
  if (cudaMemcpyToSymbol(c_ops, tab, len * sizeof(double), base * sizeof(double)) !=
      cudaSuccess)
    return -2;
  std::memcpy(g_ops_host + base, tab, len * sizeof(double));
  g_ops_set[n1] = true;
  return 0;
}

template <int N1>
static void launch_lines(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                         cudaStream_t st) {
  constexpr int E = elems_per_block<N1>(), T = 2 * N1;
  const size_t smem = (size_t)E * Smem<N1>::per_elem * sizeof(double);
  const unsigned grid = (unsigned)((M.n_owned + E - 1) / E);
  if (A.fh) {
    cudaFuncSetAttribute(k_stage_lines<N1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_stage_lines<N1, true><<<grid, E * T, smem, st>>>(M, P, A, F);
  } else {
    cudaFuncSetAttribute(k_stage_lines<N1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_stage_lines<N1, false><<<grid, E * T, smem, st>>>(M, P, A, F);
  }
}

bool fast_stage_supported(int n1) { return n1 >= 2 && n1 <= 8; }

int launch_fast_stage(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                      cudaStream_t st) {
  switch (M.n1) {
    case 2: launch_lines<2>(M, P, A, F, st); break;
    case 3: launch_lines<3>(M, P, A, F, st); break;
    case 4: launch_lines<4>(M, P, A, F, st); break;
    case 5: launch_lines<5>(M, P, A, F, st); break;
    case 6: launch_lines<6>(M, P, A, F, st); break;
    case 7: launch_lines<7>(M, P, A, F, st); break;
    case 8: launch_lines<8>(M, P, A, F, st); break;
    default: return 0;
  }
  return 1;
}

}  // namespace swdg_dev
