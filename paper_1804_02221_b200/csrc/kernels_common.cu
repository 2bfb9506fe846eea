// kernels_common.cu — mode-independent kernels: the halo pack/unpack of the
// partitioned (multi-GPU) step and the grid-cap test hook.
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


}  // namespace swdg_dev

namespace swdg_dev {
int g_grid_cap = 0;
}  // namespace swdg_dev
