// kernels_common.cu — per-step diagnostics shared by both arithmetic modes:
// total_mass / total_entropy / min_height (field.hpp:39-68) and the advisory
// mean-positivity time-step bound min_positivity_dt (limiter.hpp:107-166).
// Sums use a fixed-order two-level reduction (element-serial, then a fixed
// strided/tree pass), so repeated runs are bitwise reproducible; they agree
// with the reference's fully serial sums to rounding.
#include <cuda_runtime.h>

#include "swdg_device.cuh"
#include "swdg_launch.h"

namespace swdg_dev {
namespace {

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

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

__device__ __forceinline__ double elem_sums(const Mesh& M, const Phys& P, const CState& S,
                                            double* partial, int e);

__global__ void k_elem_sums(Mesh M, Phys P, CState S, double* partial, Flags* F) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long key = ~0ull;
  if (e < M.n_owned) key = order_key(elem_sums(M, P, S, partial, e));
  key = block_min_key(key);
  if (threadIdx.x == 0) atomicMin(&F->min_h_key, key);
}

__device__ __forceinline__ double elem_sums(const Mesh& M, const Phys& P, const CState& S,
                                            double* partial, int e) {
  const int n1 = M.n1;
  const long long b = (long long)e * M.np;
  double mass = 0.0, ent = 0.0, mn = S.h[b];
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      const long long n = b + i * n1 + j;
      const double h = S.h[n], wij = M.jac[n] * M.w[i] * M.w[j];
      double u, v;
      velocity(h, S.hu[n], S.hv[n], P.h_des, u, v);
      const double k = 0.5 * h * (u * u + v * v);
      const double en = k + 0.5 * P.g * h * h + P.g * h * M.b[n];
      mass += h * wij;
      ent += en * wij;
      mn = smin(mn, h);
    }
  partial[2 * e] = mass;
  partial[2 * e + 1] = ent;
  return mn;
}

__global__ void k_sum_partials(const double* partial, int K, double* out2) {
  __shared__ double sm[2][1024];
  const int t = threadIdx.x;
  double a = 0.0, c = 0.0;
  for (int e = t; e < K; e += blockDim.x) {
    a += partial[2 * e];
    c += partial[2 * e + 1];
  }
  sm[0][t] = a;
  sm[1][t] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) {
      sm[0][t] += sm[0][t + s];
      sm[1][t] += sm[1][t + s];
    }
    __syncthreads();
  }
  if (t == 0) {
    out2[0] = sm[0][0];
    out2[1] = sm[1][0];
  }
}

// positivity_dt_bounds (limiter.hpp:107-130) evaluated by every owned
// element-face node from its own side (the reference evaluates the minus side
// and, for interior faces, the plus side with the plus normal: the same set).
__device__ __forceinline__ double posdt_bound(const Mesh& M, const Phys& P, const CState& S,
                                               long long idx);

__global__ void k_posdt(Mesh M, Phys P, CState S, Flags* F) {
  unsigned long long key = ~0ull;
  const long long nf = (long long)M.n_owned * 4 * M.n1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < nf;
       idx += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = order_key(posdt_bound(M, P, S, idx));
    key = k < key ? k : key;
  }
  key = block_min_key(key);  // one atomic per block
  if (threadIdx.x == 0) atomicMin(&F->posdt_key, key);
}

__device__ __forceinline__ double posdt_bound(const Mesh& M, const Phys& P, const CState& S,
                                               long long idx) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int n1 = M.n1;
  const int t = (int)(idx % n1);
  const int face = (int)((idx / n1) % 4);
  const int e = (int)(idx / (4 * n1));
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
  velocity(hm, hum, hvm, P.h_des, um, vm);
  velocity(hp, hup, hvp, P.h_des, up, vp);
  const double unm = nx * um + ny * vm, unp = nx * up + ny * vp;
  const double uavg = 0.5 * (unm + unp);
  const double cavg = 0.5 * (sqrt(P.g * smax(hm, 0.0)) + sqrt(P.g * smax(hp, 0.0)));
  const double a = fabs(uavg + cavg) + fabs(uavg - cavg);
  const double bb = fabs(uavg + cavg) - fabs(uavg - cavg);
  const double den1 = a + 2.0 * uavg;
  double bound = den1 > 1e-300 ? M.w0 * a_scale / den1 : inf;
  const double jump = unp - unm;
  if (hm > 0.0 && bb * jump < 0.0)
    bound = smin(bound, fabs(M.w0 * a_scale * P.g * hm / (cavg * bb * jump)));
  return bound;
}

// halo pack/unpack: node-major [i][field] so each peer's block is contiguous
__global__ void k_halo_pack(const int* idx, long long n, int nf, const double* f0,
                            const double* f1, const double* f2, const double* f3, double* buf) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = idx[i];
  buf[i * nf + 0] = f0[k];
  buf[i * nf + 1] = f1[k];
  buf[i * nf + 2] = f2[k];
  if (nf > 3) buf[i * nf + 3] = f3[k];
}

__global__ void k_halo_unpack(const int* idx, long long n, int nf, double* f0, double* f1,
                              double* f2, double* f3, const double* buf) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = idx[i];
  f0[k] = buf[i * nf + 0];
  f1[k] = buf[i * nf + 1];
  f2[k] = buf[i * nf + 2];
  if (nf > 3) f3[k] = buf[i * nf + 3];
}

}  // namespace

int launch_halo_pack(const int* idx, long long n, int nf, const double* const* f, double* buf,
                     cudaStream_t st) {
  if (n == 0) return 0;
  k_halo_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n, nf, f[0], f[1], f[2],
                                                          nf > 3 ? f[3] : f[0], buf);
  return 1;
}

int launch_halo_unpack(const int* idx, long long n, int nf, double* const* f, const double* buf,
                       cudaStream_t st) {
  if (n == 0) return 0;
  k_halo_unpack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n, nf, f[0], f[1], f[2],
                                                            nf > 3 ? f[3] : f[0], buf);
  return 1;
}

int launch_diagnostics(const Mesh& M, const Phys& P, CState S, double* partial, double* out2,
                       Flags* F, cudaStream_t st) {
  k_elem_sums<<<(M.n_owned + 127) / 128, 128, 0, st>>>(M, P, S, partial, F);
  k_sum_partials<<<1, 1024, 0, st>>>(partial, M.n_owned, out2);
  const long long nf = (long long)M.n_owned * 4 * M.n1;
  const long long pb = (nf + 255) / 256;
  k_posdt<<<(unsigned)(pb < 148 * 16 ? pb : 148 * 16), 256, 0, st>>>(M, P, S, F);
  return 3;
}

}  // namespace swdg_dev

namespace swdg_dev {
int g_grid_cap = 0;
}  // namespace swdg_dev
