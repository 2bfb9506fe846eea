// kernels_bench.cu — the paper's §5 kernel comparison on the B200: one pass of
// the split-form (entropy-conservative flux differencing with Dtilde,
// dg_rhs.hpp:23-71) or the standard (pointwise contravariant fluxes times D,
// dg_rhs.hpp:75-117) volume kernel over K elements, the buffers of the
// reference harness (bench.hpp:101-131 KernelBuffers), out += volume term.
//
// Both are node-per-thread with the element group staged in shared memory, so
// the comparison isolates the arithmetic: the split kernel evaluates the
// reference's 2(N+1) ordered two-point fluxes per node (bench.hpp:91-94, the
// flux-evaluation count the paper's table reports), the standard kernel one
// pointwise flux per node plus the 2(N+1)-term D contractions.  This harness is
// not the product stage path (kernels_fast.cu evaluates unordered pairs once).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/swdg_gpu.h"

extern "C" int swdg_operators(int degree, double* nodes, double* weights, double* deriv,
                              double* deriv_modified, double* deriv_weak, double* vand,
                              double* vand_inv);

namespace {

constexpr int kMaxNp = 256;
__constant__ double c_dt[kMaxNp];  // Dtilde of the current degree (split)
__constant__ double c_d[kMaxNp];   // D (standard)

template <int N1>
struct BP {
  static constexpr int NP = N1 * N1;
  static constexpr int E = (256 / NP) > 0 ? (256 / NP) : 1;
  static constexpr int THREADS = E * NP;
};

__device__ __forceinline__ void vel(double h, double hu, double hv, double h_des, double& u,
                                    double& v) {
  // phys::velocity (physics.hpp:23-36)
  if (h >= h_des) {
    u = hu / h;
    v = hv / h;
  } else {
    u = 0.0;
    v = 0.0;
  }
}

template <int N1>
__global__ void __launch_bounds__(BP<N1>::THREADS)
    k_volume_split(int64_t K, double g, double h_des, const double* __restrict__ h,
                   const double* __restrict__ hu, const double* __restrict__ hv,
                   const double* __restrict__ ye, const double* __restrict__ xe,
                   const double* __restrict__ yx, const double* __restrict__ xx, double* oh,
                   double* ohu, double* ohv) {
  using P = BP<N1>;
  constexpr int NP = P::NP;
  __shared__ double s[9][P::THREADS];  // h hu hv u v ye xe yx xx
  const int tid = threadIdx.x, el = tid / NP, loc = tid - el * NP;
  const int i = loc / N1, j = loc - i * N1;
  const int64_t e = (int64_t)blockIdx.x * P::E + el;
  const bool ok = e < K;
  const int64_t n = e * NP + loc;
  double hn = 0, hun = 0, hvn = 0, un = 0, vn = 0;
  if (ok) {
    hn = h[n];
    hun = hu[n];
    hvn = hv[n];
    vel(hn, hun, hvn, h_des, un, vn);
    s[0][tid] = hn;
    s[1][tid] = hun;
    s[2][tid] = hvn;
    s[3][tid] = un;
    s[4][tid] = vn;
    s[5][tid] = ye[n];
    s[6][tid] = xe[n];
    s[7][tid] = yx[n];
    s[8][tid] = xx[n];
  }
  __syncthreads();
  if (!ok) return;
  const double yen = s[5][tid], xen = s[6][tid], yxn = s[7][tid], xxn = s[8][tid];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int b = el * NP;
#pragma unroll 4
  for (int m = 0; m < N1; ++m) {
    // xi: (i,j) with (m,j); eta: (i,j) with (i,m) -- volume_flux_pair (fluxes.hpp:21-39)
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
      const int q = b + (dir == 0 ? m * N1 + j : i * N1 + m);
      const double hq = s[0][q], huq = s[1][q], hvq = s[2][q], uq = s[3][q], vq = s[4][q];
      const double havg = 0.5 * (hn + hq), uavg = 0.5 * (un + uq), vavg = 0.5 * (vn + vq);
      const double huavg = 0.5 * (hun + huq), hvavg = 0.5 * (hvn + hvq);
      const double h2avg = 0.5 * (hn * hn + hq * hq);
      const double press = g * havg * havg - 0.5 * g * h2avg;
      const double f0 = huavg, f1 = huavg * uavg + press, f2 = huavg * vavg;
      const double g0 = hvavg, g1 = hvavg * uavg, g2 = hvavg * vavg + press;
      if (dir == 0) {
        const double ya = 0.5 * (yen + s[5][q]), xa = 0.5 * (xen + s[6][q]);
        const double d = c_dt[i * N1 + m];
        a0 += d * (ya * f0 - xa * g0);
        a1 += d * (ya * f1 - xa * g1);
        a2 += d * (ya * f2 - xa * g2);
      } else {
        const double ya = 0.5 * (yxn + s[7][q]), xa = 0.5 * (xxn + s[8][q]);
        const double d = c_dt[j * N1 + m];
        a0 += d * (xa * g0 - ya * f0);
        a1 += d * (xa * g1 - ya * f1);
        a2 += d * (xa * g2 - ya * f2);
      }
    }
  }
  oh[n] += a0;
  ohu[n] += a1;
  ohv[n] += a2;
}

template <int N1>
__global__ void __launch_bounds__(BP<N1>::THREADS)
    k_volume_standard(int64_t K, double g, double h_des, const double* __restrict__ h,
                      const double* __restrict__ hu, const double* __restrict__ hv,
                      const double* __restrict__ ye, const double* __restrict__ xe,
                      const double* __restrict__ yx, const double* __restrict__ xx, double* oh,
                      double* ohu, double* ohv) {
  using P = BP<N1>;
  constexpr int NP = P::NP;
  __shared__ double s[6][P::THREADS];  // ft0..2, gt0..2
  const int tid = threadIdx.x, el = tid / NP, loc = tid - el * NP;
  const int i = loc / N1, j = loc - i * N1;
  const int64_t e = (int64_t)blockIdx.x * P::E + el;
  const bool ok = e < K;
  const int64_t n = e * NP + loc;
  if (ok) {
    double u, v;
    const double hn = h[n];
    vel(hn, hu[n], hv[n], h_des, u, v);
    const double pr = 0.5 * g * hn * hn;
    const double fx0 = hn * u, fx1 = hn * u * u + pr, fx2 = hn * u * v;
    const double fy0 = hn * v, fy1 = hn * u * v, fy2 = hn * v * v + pr;
    const double yen = ye[n], xen = xe[n], yxn = yx[n], xxn = xx[n];
    s[0][tid] = yen * fx0 - xen * fy0;
    s[1][tid] = yen * fx1 - xen * fy1;
    s[2][tid] = yen * fx2 - xen * fy2;
    s[3][tid] = xxn * fy0 - yxn * fx0;
    s[4][tid] = xxn * fy1 - yxn * fx1;
    s[5][tid] = xxn * fy2 - yxn * fx2;
  }
  __syncthreads();
  if (!ok) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int b = el * NP;
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    const double di = c_d[i * N1 + m], dj = c_d[j * N1 + m];
    const int qx = b + m * N1 + j, qe = b + i * N1 + m;
    a0 += di * s[0][qx] + dj * s[3][qe];
    a1 += di * s[1][qx] + dj * s[4][qe];
    a2 += di * s[2][qx] + dj * s[5][qe];
  }
  oh[n] += a0;
  ohu[n] += a1;
  ohv[n] += a2;
}

template <int N1>
void launch(int kind, int64_t K, double g, const double* const* in, double* const* out,
            cudaStream_t st) {
  using P = BP<N1>;
  const unsigned grid = (unsigned)((K + P::E - 1) / P::E);
  if (kind == 0)
    k_volume_split<N1><<<grid, P::THREADS, 0, st>>>(K, g, 1e-8, in[0], in[1], in[2], in[3],
                                                    in[4], in[5], in[6], out[0], out[1], out[2]);
  else
    k_volume_standard<N1><<<grid, P::THREADS, 0, st>>>(K, g, 1e-8, in[0], in[1], in[2], in[3],
                                                       in[4], in[5], in[6], out[0], out[1],
                                                       out[2]);
}

int g_loaded_degree = -1;
int g_loaded_device = -1;

}  // namespace

extern "C" int swdg_gpu_volume_kernel(int kind, int degree, int64_t k, const double* const* in,
                                  double* const* out, double g, void* stream) {
  if (kind < 0 || kind > 1 || degree < 1 || degree > 15 || k < 1) return SWDG_ERR_INPUT;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SWDG_ERR_CUDA;
  if (degree != g_loaded_degree || dev != g_loaded_device) {
    const int n1 = degree + 1, np = n1 * n1;
    double nodes[16], w[16], D[kMaxNp], Dt[kMaxNp], Dh[kMaxNp], V[kMaxNp], Vi[kMaxNp];
    swdg_operators(degree, nodes, w, D, Dt, Dh, V, Vi);
    if (cudaMemcpyToSymbol(c_dt, Dt, np * sizeof(double)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_d, D, np * sizeof(double)) != cudaSuccess)
      return SWDG_ERR_CUDA;
    g_loaded_degree = degree;
    g_loaded_device = dev;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (degree + 1) {
#define SWDG_BK(n) \
  case n: launch<n>(kind, k, g, in, out, st); break;
    SWDG_BK(2) SWDG_BK(3) SWDG_BK(4) SWDG_BK(5) SWDG_BK(6) SWDG_BK(7) SWDG_BK(8) SWDG_BK(9)
    SWDG_BK(10) SWDG_BK(11) SWDG_BK(12) SWDG_BK(13) SWDG_BK(14) SWDG_BK(15) SWDG_BK(16)
#undef SWDG_BK
    default: return SWDG_ERR_INPUT;
  }
  return cudaGetLastError() == cudaSuccess ? SWDG_OK : SWDG_ERR_CUDA;
}
