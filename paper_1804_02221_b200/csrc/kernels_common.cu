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

// direct peer-memory exchange: pack straight into the receiving rank's mailbox
// (a CUDA IPC mapping: NVLink / NVSwitch stores between GPUs), then raise the
// receiver's sequence flag with a system-scope release once every block of the
// pack has finished (stream order + the fences)
__global__ void k_halo_push(const int* idx, long long n, int nf, const double* f0,
                            const double* f1, const double* f2, const double* f3, double* dst) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    const long long k = idx[i];
    dst[i * nf + 0] = f0[k];
    dst[i * nf + 1] = f1[k];
    dst[i * nf + 2] = f2[k];
    if (nf > 3) dst[i * nf + 3] = f3[k];
  }
  __threadfence_system();
}

// sequence numbers are `seq`, or `*base + seq` when the caller keeps the base on
// the device (graph replays: the captured kernels carry offsets, a kernel at the
// end of each replay advances the base)
__global__ void k_flag_release(unsigned long long* flag, const unsigned long long* base,
                               unsigned long long seq) {
  __threadfence_system();
  const unsigned long long v = (base ? *base : 0ull) + seq;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

__global__ void k_seq_advance(unsigned long long* base, unsigned long long by) { *base += by; }

// the receiver: one lane per peer polls its flag (system-scope acquire) until the
// peer's data of exchange `seq` has landed; a peer that never arrives sets *err
// after timeout_ns instead of hanging the stream
__global__ void k_flags_wait(const unsigned long long* flags, int n,
                             const unsigned long long* base, unsigned long long seq,
                             unsigned long long timeout_ns, int* err) {
  const int i = threadIdx.x;
  if (base) seq += *base;
  if (i < n) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
      if (v >= seq) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

}  // namespace

int launch_halo_push(const int* idx, long long n, int nf, const double* const* f, double* dst,
                     unsigned long long* flag, const unsigned long long* base,
                     unsigned long long seq, cudaStream_t st) {
  int launches = 0;
  if (n > 0) {
    k_halo_push<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n, nf, f[0], f[1], f[2],
                                                            nf > 3 ? f[3] : f[0], dst);
    ++launches;
  }
  k_flag_release<<<1, 1, 0, st>>>(flag, base, seq);
  return launches + 1;
}

int launch_seq_advance(unsigned long long* base, unsigned long long by, cudaStream_t st) {
  k_seq_advance<<<1, 1, 0, st>>>(base, by);
  return 1;
}

int launch_flags_wait(const unsigned long long* flags, int n, const unsigned long long* base,
                      unsigned long long seq, unsigned long long timeout_ns, int* err,
                      cudaStream_t st) {
  if (n <= 0) return 0;
  k_flags_wait<<<1, ((n + 31) / 32) * 32, 0, st>>>(flags, n, base, seq, timeout_ns, err);
  return 1;
}

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

// fast-mode dispatch over the degree-range objects of kernels_fast.cu
static int fast_part(int n1) { return n1 <= 7 ? 0 : (n1 <= 11 ? 1 : 2); }

bool fast_stage_supported(int n1) { return n1 >= 2 && n1 <= 16; }

int upload_fast_ops(int n1, const double* D, const double* Dt, const double* Dh,
                    const double* Vinv, const double* w) {
  // every object has its own table; all get the degree (the source-geometry
  // kernel of part 0 serves every degree)
  for (auto up : {upload_fast_ops_p0, upload_fast_ops_p1, upload_fast_ops_p2}) {
    const int rc = up(n1, D, Dt, Dh, Vinv, w);
    if (rc) return rc;
  }
  return 0;
}

int launch_source_geometry(const Mesh& M, double* sx, double* sy, cudaStream_t st) {
  return launch_source_geometry_p0(M, sx, sy, st);
}

int launch_fast_visc_pre(const Mesh& M, const Phys& P, CState S, double* eps, double* fvu,
                         double* fvv, double* gvu, double* gvv, Flags* F, cudaStream_t st) {
  switch (fast_part(M.n1)) {
    case 0: return launch_fast_visc_pre_p0(M, P, S, eps, fvu, fvv, gvu, gvv, F, st);
    case 1: return launch_fast_visc_pre_p1(M, P, S, eps, fvu, fvv, gvu, gvv, F, st);
    default: return launch_fast_visc_pre_p2(M, P, S, eps, fvu, fvv, gvu, gvv, F, st);
  }
}

int launch_fast_stage(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                      cudaStream_t st) {
  switch (fast_part(M.n1)) {
    case 0: return launch_fast_stage_p0(M, P, A, F, st);
    case 1: return launch_fast_stage_p1(M, P, A, F, st);
    default: return launch_fast_stage_p2(M, P, A, F, st);
  }
}
}  // namespace swdg_dev
