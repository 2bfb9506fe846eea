// swdg_launch.h — host-side launch interface between the C-ABI context and the
// kernel translation units (exact: kernels_exact.cu built --fmad=false; fast:
// kernels_fast.cu).  Each launcher returns the number of kernels it launched.
#pragma once

#include <cuda_runtime.h>

#include "swdg_device.cuh"

namespace swdg_dev {

struct StageArgs {
  CState in;       // stage input W^(k)
  CState wn;       // W^n for the SSPRK3 convex combination
  State out;       // stage output (update != 0)
  State rhs;       // optional dW/dt output (h == nullptr: not written)
  double dt, ca, cb, t;
  int stage;       // 0,1,2 (ssprk3_combination timeloop.hpp:80-81)
  int update;      // write out = combine(axpy(in, dt, rhs))
  const double* eps;                        // per element viscosity
  const double *fvu, *fvv, *gvu, *gvv;      // viscous flux pairs (nullptr: inviscid)
  const double *fh, *fhu, *fhv;             // nodal forcing (nullptr: none)
  // persistent stage kernels claim element groups from this counter (zeroed
  // before each launch) so the CTAs sweep the mesh as one wavefront and the
  // neighbour face traces they gather are still in L2 when reused
  int* gctr;
  // SMs the persistent stage kernels leave free (0: use all): a partition's
  // interior launch runs while NCCL moves the halo, whose kernels need SMs
  int reserve_sms;
};

// exact mode (kernels_exact.cu)
int launch_exact_indicator(const Mesh& M, CState S, double* r, cudaStream_t st);
int launch_exact_grad(const Mesh& M, const Phys& P, CState S, const double* eps, double* fvu,
                      double* fvv, double* gvu, double* gvv, cudaStream_t st);
int launch_exact_rhs_stage(const Mesh& M, const Phys& P, const StageArgs& A, cudaStream_t st);
int launch_exact_limit(const Mesh& M, const Phys& P, State S, Flags* F, cudaStream_t st);

// fast mode: dispatch (kernels_common.cu) over the three degree-range objects of
// kernels_fast.cu (SWDG_PART 0/1/2: N+1 in [2,7], [8,11], [12,16])
int upload_fast_ops(int n1, const double* D, const double* Dt, const double* Dh,
                    const double* Vinv, const double* w);
bool fast_stage_supported(int n1);
int launch_source_geometry(const Mesh& M, double* sx, double* sy, cudaStream_t st);
int launch_fast_visc_pre(const Mesh& M, const Phys& P, CState S, double* eps, double* fvu,
                         double* fvv, double* gvu, double* gvv, Flags* F, cudaStream_t st);
int launch_fast_stage(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                      cudaStream_t st);
#define SWDG_FAST_PART_DECL(p)                                                              \
  int upload_fast_ops_##p(int n1, const double* D, const double* Dt, const double* Dh,      \
                          const double* Vinv, const double* w);                             \
  int launch_source_geometry_##p(const Mesh& M, double* sx, double* sy, cudaStream_t st);   \
  int launch_fast_visc_pre_##p(const Mesh& M, const Phys& P, CState S, double* eps,         \
                               double* fvu, double* fvv, double* gvu, double* gvv, Flags* F, \
                               cudaStream_t st);                                            \
  int launch_fast_stage_##p(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,     \
                            cudaStream_t st);
SWDG_FAST_PART_DECL(p0)
SWDG_FAST_PART_DECL(p1)
SWDG_FAST_PART_DECL(p2)
#undef SWDG_FAST_PART_DECL

// per-step reductions (kernels_step.cu, --fmad=false): mass/entropy partials
// (step_sum_partials() pairs) for launch_diagnostics
int step_sum_partials();
// compute_dt's CFL candidates (fast: the fast arithmetic of the fast step reductions)
int launch_cfl_dt(const Mesh& M, const Phys& P, CState S, Flags* F, cudaStream_t st, bool fast);
// limited_entropy_check of the elements a stage limited (A.rhs holds its dW/dt)
int launch_limiter_entropy(const Mesh& M, const Phys& P, const StageArgs& A, const Flags* F,
                           unsigned long long* key, cudaStream_t st);

// test hook: cap on the persistent stage kernels' grid (0 = none), kernels_common.cu
extern int g_grid_cap;

// mode-independent (kernels_common.cu)
int launch_halo_push(const int* idx, long long n, int nf, const double* const* f, double* dst,
                     unsigned long long* flag, const unsigned long long* base,
                     unsigned long long seq, cudaStream_t st);
int launch_flags_wait(const unsigned long long* flags, int n, const unsigned long long* base,
                      unsigned long long seq, unsigned long long timeout_ns, int* err,
                      cudaStream_t st);
int launch_seq_advance(unsigned long long* base, unsigned long long by, cudaStream_t st);
int launch_halo_pack(const int* idx, long long n, int nf, const double* const* f, double* buf,
                     cudaStream_t st);
int launch_halo_unpack(const int* idx, long long n, int nf, double* const* f, const double* buf,
                       cudaStream_t st);
int launch_diagnostics(const Mesh& M, const Phys& P, CState S, double* partial, double* out2,
                       Flags* F, cudaStream_t st, bool serial);

}  // namespace swdg_dev
