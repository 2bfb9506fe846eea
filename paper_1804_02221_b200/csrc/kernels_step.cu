// kernels_step.cu — per-step reductions of the device-resident driver, the
// positivity time-step bound (limiter.hpp:107-166) and the limiter entropy
// diagnostic, sm_100a FP64, compiled with --fmad=false (every per-node
// expression rounds like the reference's Release build).
//
//   k_step_diag    tile by tile: total_mass, total_entropy (field.hpp:39-61) as
//                  fixed-order block partials, min_height (field.hpp:63-67), the
//                  compute_dt candidates (timeloop.hpp:53-75) and the
//                  min_positivity_dt bounds (limiter.hpp:107-166) as
//                  order-independent minima.
//   k_step_final   the block partials in a fixed tree order (reproducible).
//   k_limiter_entropy  limited_entropy_check (limiter.hpp:88-101) for the
//                  elements post_stage limited (timeloop.hpp:221-229): the
//                  pre-limit stage state is rebuilt from the stage input, W^n
//                  and the stage's dW/dt with the reference's axpy/combine
//                  (timeloop.hpp:114-127), theta recomputed as limit_element
//                  does (limiter.hpp:43-84).
//
// The node pass reads h, hu, hv, J, b and the two CFL lengths once (56 B per
// node), the face pass the face arrays (n_x, n_y, a: 12 B per node at N=7) and
// the traces; a grid of a fixed number of CTAs with a static tile assignment
// makes the partial sums independent of the device and of timing, so a run is
// bitwise repeatable.
#include <cuda_runtime.h>

#include "fast_math.cuh"
#include "swdg_device.cuh"
#include "swdg_launch.h"

namespace swdg_dev {
namespace {

#ifndef SWDG_DIAG_BATCH
#define SWDG_DIAG_BATCH 2  // measured 0.2-0.5% per step faster than 1 (N=3, 7, 12); 4 slower
#endif
#ifndef SWDG_DIAG_FBATCH
#define SWDG_DIAG_FBATCH 1
#endif
constexpr int kSumThreads = 256;
constexpr int kSumBlocks = 148 * 8;  // fixed: the partial-sum order must not depend on the device

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// phys::velocity (physics.hpp:23-36)
__device__ __forceinline__ void velocity(double h, double hu, double hv, double h_des,
                                         double& u, double& v) {
  if (h >= h_des) {
    u = hu / h;
    v = hv / h;
  } else {
    u = 0.0;
    v = 0.0;
  }
}

// Fast-mode arithmetic (the step reductions of SWDG_MODE_FAST need not be
// bitwise): fast_math.cuh's reciprocal and square root (MUFU seeds and Newton
// steps in explicit round-to-nearest FMAs, within an ulp) and the stage
// kernels' velocity, instead of the IEEE division / square-root sequences this
// --fmad=false translation unit otherwise emits.
template <bool FAST>
__device__ __forceinline__ void vel_t(double h, double hu, double hv, double h_des, double& u,
                                      double& v) {
  if constexpr (FAST) {
    vel(h, hu, hv, h_des, u, v);
  } else {
    velocity(h, hu, hv, h_des, u, v);
  }
}

template <bool FAST>
__device__ __forceinline__ double div_t(double a, double b) {
  if constexpr (FAST) return __dmul_rn(a, frcp(b));
  else return a / b;
}

template <bool FAST>
__device__ __forceinline__ double sqrt_t(double x) {
  if constexpr (FAST) return fsqrt0(x);
  else return sqrt(x);
}

// phys::entropy (physics.hpp:47-62): h(u^2+v^2)/2 + g h^2/2 + g h b
__device__ __forceinline__ double entropy(double h, double hu, double hv, double b,
                                          const Phys& P) {
  double u, v;
  velocity(h, hu, hv, P.h_des, u, v);
  const double k = 0.5 * h * (u * u + v * v);
  return k + 0.5 * P.g * h * h + P.g * h * b;
}

// fixed-order block sum of two values (valid in thread 0)
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double s[2][32];
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s[0][w] = a;
    s[1][w] = b;
  }
  __syncthreads();
  if (w == 0) {
    a = (int)threadIdx.x < nw ? s[0][threadIdx.x] : 0.0;
    b = (int)threadIdx.x < nw ? s[1][threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
  }
}

// n / d for n < 2^31 by one 64-bit multiply and a shift (the round-up magic
// number, p = 31 + ceil(log2 d)): the per-node index arithmetic (element, node, face
// of an index) without integer divisions; the magic is formed once per thread
struct FDiv {
  unsigned long long m;
  int p;
  __device__ explicit FDiv(unsigned d) {
    const int l = d > 1 ? 32 - __clz(d - 1) : 0;
    p = 31 + l;
    m = ((1ull << p) + d - 1) / d;
  }
  __device__ __forceinline__ unsigned operator()(unsigned n) const {
    return (unsigned)(((unsigned long long)n * m) >> p);
  }
};

struct NodeAcc {
  double mass = 0.0, ent = 0.0;
  unsigned long long kmin = ~0ull, kdt = ~0ull, klen = ~0ull;
};

template <bool FAST>
__device__ __forceinline__ void node_terms(const Mesh& M, const Phys& P, double order, int loc,
                                           double h, double hu, double hv, double jac,
                                           double b, double lxi, double leta, NodeAcc& acc,
                                           const FDiv& div_n1) {
  const int i = (int)div_n1((unsigned)loc), j = loc - i * M.n1;
  const double wi = M.w[i], wj = M.w[j];
  // one phys::velocity per node serves both the entropy (physics.hpp:47-62) and
  // compute_dt (timeloop.hpp:58-71): the same call in the reference, same bits
  double u, v;
  vel_t<FAST>(h, hu, hv, P.h_des, u, v);
  const double kin = 0.5 * h * (u * u + v * v);
  const double en = kin + 0.5 * P.g * h * h + P.g * h * b;
  // total_mass: sum += h * J * w_i * w_j; total_entropy: e * J * w_i * w_j
  acc.mass += h * jac * wi * wj;
  acc.ent += en * jac * wi * wj;
  const unsigned long long kh = order_key(h);
  acc.kmin = kh < acc.kmin ? kh : acc.kmin;
  // compute_dt per node, lengths precomputed with glibc hypot
  const double c = sqrt_t<FAST>(P.g * smax(h, 0.0));
  double dt = __longlong_as_double(0x7ff0000000000000ll);
  const double lx = fabs(u) + c, ly = fabs(v) + c;
  if (lx > 1e-14) dt = smin(dt, div_t<FAST>(lxi, order * lx));
  if (ly > 1e-14) dt = smin(dt, div_t<FAST>(leta, order * ly));
  const unsigned long long a = order_key(dt), l = order_key(smin(lxi, leta));
  acc.kdt = a < acc.kdt ? a : acc.kdt;
  acc.klen = l < acc.klen ? l : acc.klen;
}

__global__ void __launch_bounds__(1024) k_step_final(const double* partial, int nparts,
                                                     double* out2) {
  double a = 0.0, b = 0.0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) {
    a += partial[2 * k];
    b += partial[2 * k + 1];
  }
  block_sum2(a, b);
  if (threadIdx.x == 0) {
    out2[0] = a;
    out2[1] = b;
  }
}

// limited_entropy_check for the elements this stage limited; the worst jump
// (e1 - e0) / max(1, |e0|) goes to *key (order key, atomicMax).  A rejected
// stage never reaches the limiter in the reference (post_stage returns first),
// so nothing is recorded for it.
__global__ void k_limiter_entropy(Mesh M, Phys P, StageArgs A, const Flags* F,
                                  unsigned long long* key) {
  const int e = M.e_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.n_owned || !P.limiter) return;
  if (*(volatile const int*)&F->reject) return;
  const int n1 = M.n1, np = M.np;
  const long long b0 = (long long)e * np;
  // the pre-limit stage state: W + dt R, then a W^n + b (.) for stages 2-3
  auto pre = [&](long long n, double& h, double& hu, double& hv) {
    h = A.in.h[n];
    hu = A.in.hu[n];
    hv = A.in.hv[n];
    h += A.dt * A.rhs.h[n];
    hu += A.dt * A.rhs.hu[n];
    hv += A.dt * A.rhs.hv[n];
    if (A.stage > 0) {
      h = A.ca * A.wn.h[n] + A.cb * h;
      hu = A.ca * A.wn.hu[n] + A.cb * hu;
      hv = A.ca * A.wn.hv[n] + A.cb * hv;
    }
  };
  double area = 0.0, a0 = 0.0, mmin = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      const long long n = b0 + i * n1 + j;
      double h, hu, hv;
      pre(n, h, hu, hv);
      const double w = M.jac[n] * M.w[i] * M.w[j];
      area += w;
      a0 += w * h;
      mmin = (i == 0 && j == 0) ? h : smin(mmin, h);
    }
  const double avg0 = (1.0 / area) * a0;
  if (avg0 < 0.0 || !(mmin < 0.0)) return;
  const double denom = avg0 - mmin;
  const double theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
  if (!(theta < 1.0)) return;
  double e_before = 0.0, e_after = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      const long long n = b0 + i * n1 + j;
      double h, hu, hv;
      pre(n, h, hu, hv);
      const double w = M.jac[n] * M.w[i] * M.w[j];
      const double bn = M.b[n];
      e_before += w * entropy(h, hu, hv, bn, P);
      e_after += w * entropy(A.out.h[n], A.out.hu[n], A.out.hv[n], bn, P);
    }
  const double jump = (e_after - e_before) / smax(1.0, fabs(e_before));
  atomicMax(key, order_key(jump));
}

// positivity_dt_bounds (limiter.hpp:107-130) evaluated by every owned
// element-face node from its own side (the reference evaluates the minus side
// and, for interior faces, the plus side with the plus normal: the same set).
template <bool FAST>
__device__ __forceinline__ double posdt_bound(const Mesh& M, const Phys& P, const CState& S,
                                               long long idx, const FDiv& div_n1) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int n1 = M.n1;
  const int q = (int)div_n1((unsigned)idx);  // idx / n1 = 4 e + face
  const int t = (int)idx - q * n1;
  const int face = q & 3;
  const int e = q >> 2;
  const int4 ef = M.ef[e * 4 + face];
  if (!(ef.y & EF_PRESENT)) return inf;
  const long long n = (long long)e * M.np + face_node(n1, face, t);
  const double nx = M.fnx[idx], ny = M.fny[idx], a_scale = M.fa[idx];
  const double hm = S.h[n], hum = S.hu[n], hvm = S.hv[n];
  double hp, hup, hvp;
  if (ef.y & EF_WALL) {
    const double mn = hum * nx + hvm * ny;
    hp = hm;
    hup = hum - 2.0 * mn * nx;
    hvp = hvm - 2.0 * mn * ny;
  } else {
    const int nf = ef.y & EF_NBR_FACE_MASK;
    const int tp = (ef.y & EF_REVERSED) ? M.degree - t : t;
    const long long nb = (long long)ef.x * M.np + face_node(n1, nf, tp);
    hp = S.h[nb];
    hup = S.hu[nb];
    hvp = S.hv[nb];
  }
  double um, vm, up, vp;
  vel_t<FAST>(hm, hum, hvm, P.h_des, um, vm);
  vel_t<FAST>(hp, hup, hvp, P.h_des, up, vp);
  const double unm = nx * um + ny * vm, unp = nx * up + ny * vp;
  const double uavg = 0.5 * (unm + unp);
  const double cavg = 0.5 * (sqrt_t<FAST>(P.g * smax(hm, 0.0)) + sqrt_t<FAST>(P.g * smax(hp, 0.0)));
  const double a = fabs(uavg + cavg) + fabs(uavg - cavg);
  const double bb = fabs(uavg + cavg) - fabs(uavg - cavg);
  const double den1 = a + 2.0 * uavg;
  double bound = den1 > 1e-300 ? div_t<FAST>(M.w0 * a_scale, den1) : inf;
  const double jump = unp - unm;
  if (hm > 0.0 && bb * jump < 0.0)
    bound = smin(bound, fabs(div_t<FAST>(M.w0 * a_scale * P.g * hm, cavg * bb * jump)));
  return bound;
}

// All StepDiagnostics reductions in one pass, element tile by element tile: a
// CTA owns a fixed (static) set of tiles of T elements; per tile it first runs
// the node terms (mass, entropy, min h, CFL candidates; coalesced loads) and then
// the tile's face-node positivity bounds, whose own-side state was just read
// (L1/L2 hits) and whose neighbour traces are mostly L2 hits (the tiles of all
// CTAs advance together).  Partial sums are per CTA in a fixed order.
template <int T, bool FAST>
__global__ void __launch_bounds__(kSumThreads) k_step_diag(Mesh M, Phys P, CState S,
                                                           double* partial, Flags* F) {
  const int np = M.np, n1 = M.n1;
  const int ntiles = (M.n_owned + T - 1) / T;
  const double order = 2.0 * M.degree + 1.0;
  NodeAcc acc;
  unsigned long long kpos = ~0ull;
  const FDiv div_n1((unsigned)n1), div_np((unsigned)np);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int e0 = tile * T, ne = min(T, M.n_owned - e0);
    const int n0 = e0 * np, nn = ne * np;
    // SWDG_DIAG_BATCH nodes per thread with all their loads issued before any
    // arithmetic (more bytes in flight per thread; the terms are then taken in
    // the same per-thread order as the one-node loop, so the partials are equal)
    constexpr int B = SWDG_DIAG_BATCH;
    for (int r0 = threadIdx.x; r0 < nn; r0 += B * blockDim.x) {
      double v[B][7];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int r = r0 + k * blockDim.x;
        const int n = n0 + (r < nn ? r : 0);
        v[k][0] = __ldg(S.h + n);
        v[k][1] = __ldg(S.hu + n);
        v[k][2] = __ldg(S.hv + n);
        v[k][3] = __ldg(M.jac + n);
        v[k][4] = __ldg(M.b + n);
        v[k][5] = __ldg(M.len_xi + n);
        v[k][6] = __ldg(M.len_eta + n);
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int r = r0 + k * blockDim.x;
        if (r < nn)  // n0 is a multiple of np: the node's position is r mod np
          node_terms<FAST>(M, P, order, r - (int)div_np((unsigned)r) * np, v[k][0], v[k][1],
                           v[k][2], v[k][3], v[k][4], v[k][5], v[k][6], acc, div_n1);
      }
    }
    const long long f0 = (long long)e0 * 4 * n1;
    const int nf = ne * 4 * n1;
    constexpr int BF = SWDG_DIAG_FBATCH;  // face nodes per thread per pass (unrolled)
    for (int r0 = threadIdx.x; r0 < nf; r0 += BF * blockDim.x) {
      double bnd[BF];
#pragma unroll
      for (int k = 0; k < BF; ++k) {
        const int r = r0 + k * blockDim.x;
        bnd[k] = posdt_bound<FAST>(M, P, S, f0 + (r < nf ? r : 0), div_n1);
      }
#pragma unroll
      for (int k = 0; k < BF; ++k) {
        const unsigned long long key = order_key(bnd[k]);
        if (r0 + k * blockDim.x < nf) kpos = key < kpos ? key : kpos;
      }
    }
  }
  block_sum2(acc.mass, acc.ent);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = acc.mass;
    partial[2 * blockIdx.x + 1] = acc.ent;
  }
  const unsigned long long kmin = block_min_key(acc.kmin);
  const unsigned long long kdt = block_min_key(acc.kdt);
  const unsigned long long klen = block_min_key(acc.klen);
  const unsigned long long kp = block_min_key(kpos);
  if (threadIdx.x == 0) {
    if (kmin != ~0ull) atomicMin(&F->min_h_key, kmin);
    if (kdt != ~0ull) atomicMin(&F->dt_key, kdt);
    if (klen != ~0ull) atomicMin(&F->minlen_key, klen);
    if (kp != ~0ull) atomicMin(&F->posdt_key, kp);
  }
}

// compute_dt's two reductions (timeloop.hpp:57-74): the CFL candidate minimum and
// the all-dry fallback length, with the same per-node arithmetic as the step
// reductions (so the driver's first dt and the step reports' next dt agree
// bitwise in both modes)
template <bool FAST>
__global__ void __launch_bounds__(kSumThreads) k_cfl_dt(Mesh M, Phys P, CState S, Flags* F) {
  const int nn = M.n_owned * M.np;
  const double order = 2.0 * M.degree + 1.0;
  unsigned long long kdt = ~0ull, klen = ~0ull;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < nn; n += gridDim.x * blockDim.x) {
    const double h = __ldg(S.h + n), lxi = __ldg(M.len_xi + n), leta = __ldg(M.len_eta + n);
    double u, v;
    vel_t<FAST>(h, __ldg(S.hu + n), __ldg(S.hv + n), P.h_des, u, v);
    const double c = sqrt_t<FAST>(P.g * smax(h, 0.0));
    double dt = __longlong_as_double(0x7ff0000000000000ll);
    const double lx = fabs(u) + c, ly = fabs(v) + c;
    if (lx > 1e-14) dt = smin(dt, div_t<FAST>(lxi, order * lx));
    if (ly > 1e-14) dt = smin(dt, div_t<FAST>(leta, order * ly));
    const unsigned long long a = order_key(dt), l = order_key(smin(lxi, leta));
    kdt = a < kdt ? a : kdt;
    klen = l < klen ? l : klen;
  }
  kdt = block_min_key(kdt);
  klen = block_min_key(klen);
  if (threadIdx.x == 0) {
    if (kdt != ~0ull) atomicMin(&F->dt_key, kdt);
    if (klen != ~0ull) atomicMin(&F->minlen_key, klen);
  }
}

// total_mass / total_entropy in the reference's own order (field.hpp:39-61: one
// serial sum over e, i, j): exact mode's diagnostics are then bitwise the
// reference's.  One warp: the lanes form 32 consecutive terms, lane 0 adds them
// in node order.
__global__ void __launch_bounds__(32) k_serial_sums(Mesh M, Phys P, CState S, double* out2) {
  const int nn = M.n_owned * M.np;
  const int lane = threadIdx.x;
  double mass = 0.0, ent = 0.0;
  for (int base = 0; base < nn; base += 32) {
    const int n = base + lane;
    double tm = 0.0, te = 0.0;
    if (n < nn) {
      const int loc = n % M.np, i = loc / M.n1, j = loc - i * M.n1;
      const double jac = M.jac[n], wi = M.w[i], wj = M.w[j], h = S.h[n];
      tm = h * jac * wi * wj;
      te = entropy(h, S.hu[n], S.hv[n], M.b[n], P) * jac * wi * wj;
    }
    const int cnt = nn - base < 32 ? nn - base : 32;
    for (int k = 0; k < cnt; ++k) {
      const double a = __shfl_sync(0xffffffffu, tm, k);
      const double b = __shfl_sync(0xffffffffu, te, k);
      mass += a;
      ent += b;
    }
  }
  if (lane == 0) {
    out2[0] = mass;
    out2[1] = ent;
  }
}

}  // namespace

int step_sum_partials() { return kSumBlocks; }


// StepDiagnostics reductions of a state (driver.hpp:117-127): mass, entropy,
// min h and the CFL candidates, then the positivity bound.  serial = the
// reference's summation order (exact mode).
int launch_diagnostics(const Mesh& M, const Phys& P, CState S, double* partial, double* out2,
                       Flags* F, cudaStream_t st, bool serial) {
  // tiles of ~1024 nodes (4 per thread): T = 1024 / (N+1)^2 elements
  const int T = M.np <= 16 ? 64 : M.np <= 64 ? 16 : M.np <= 128 ? 8 : 4;
  // fast mode: fast reciprocals / square roots (the exact mode keeps the IEEE
  // operations, bitwise the reference)
#define SWDG_DIAG(t)                                                                 \
  case t:                                                                            \
    if (serial) k_step_diag<t, false><<<kSumBlocks, kSumThreads, 0, st>>>(M, P, S, partial, F); \
    else k_step_diag<t, true><<<kSumBlocks, kSumThreads, 0, st>>>(M, P, S, partial, F);        \
    break;
  switch (T) {
    SWDG_DIAG(64)
    SWDG_DIAG(16)
    SWDG_DIAG(8)
    default: SWDG_DIAG(4)
  }
#undef SWDG_DIAG
  k_step_final<<<1, 1024, 0, st>>>(partial, kSumBlocks, out2);
  if (serial) {  // exact mode: the reference's serial summation order
    k_serial_sums<<<1, 32, 0, st>>>(M, P, S, out2);
    return 3;
  }
  return 2;
}

int launch_cfl_dt(const Mesh& M, const Phys& P, CState S, Flags* F, cudaStream_t st, bool fast) {
  if (fast) k_cfl_dt<true><<<kSumBlocks, kSumThreads, 0, st>>>(M, P, S, F);
  else k_cfl_dt<false><<<kSumBlocks, kSumThreads, 0, st>>>(M, P, S, F);
  return 1;
}

int launch_limiter_entropy(const Mesh& M, const Phys& P, const StageArgs& A, const Flags* F,
                           unsigned long long* key, cudaStream_t st) {
  const int ne = M.n_owned - M.e_lo;
  if (ne <= 0) return 0;
  k_limiter_entropy<<<(ne + 127) / 128, 128, 0, st>>>(M, P, A, F, key);
  return 1;
}

}  // namespace swdg_dev
