// swdg_gpu.cu — the C ABI (include/swdg_gpu.h): context, device buffers and the
// SSPRK3 stage pipeline (timeloop.hpp:88-108, 146-234) driving the exact
// (kernels_exact.cu) or fast (kernels_fast.cu) kernels on one B200.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "../../include/swdg_gpu.h"
#include "swdg_device.cuh"
#include "swdg_host.h"
#include "swdg_launch.h"
#include "swdg_mesh.h"

using namespace swdg_dev;

extern "C" int swdg_operators(int degree, double* nodes, double* weights, double* deriv,
                              double* deriv_modified, double* deriv_weak, double* vand,
                              double* vand_inv);

namespace {
thread_local std::string g_create_error;

constexpr double kCa[3] = {0.0, 3.0 / 4.0, 1.0 / 3.0};  // ssprk3_combination (timeloop.hpp:80)
constexpr double kCb[3] = {1.0, 1.0 / 4.0, 2.0 / 3.0};
constexpr double kCt[3] = {0.0, 1.0, 0.5};              // ssprk3_stage_times (timeloop.hpp:82)

struct CudaError {
  cudaError_t e;
  const char* where;
};

inline void ck(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw CudaError{e, where};
}

// every kernel launch is checked: a failed launch (bad configuration, a missing
// shared-memory attribute on a new device, ...) must never read as an accepted step
inline int launched(int n, const char* what) {
  ck(cudaGetLastError(), what);
  return n;
}

struct InputError {
  std::string msg;
};

constexpr int kDiagFlags = 3;  // Flags slot of the step reductions (0-2: stages)
// SMs a partition's interior stage leaves to the concurrent halo exchange (NCCL
// P2P kernels: one or two CTAs per peer and direction)
constexpr int kHaloReserveSms = 8;

struct Report {
  Flags f[4];
  double sums[2];  // total_mass, total_entropy
};
}  // namespace

struct swdg_gpu {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  swdg_params params{};
  Phys phys{};
  Mesh M{};
  long long nn = 0, nf = 0;
  int64_t launches = 0;
  std::string err;
  bool fast = false;   // fused fast stage kernel in use

  std::vector<void*> allocations;
  std::vector<void*> ipc_opened;  // peer mailboxes mapped by swdg_gpu_ipc_open
  int* ipc_err = nullptr;         // set by a flag wait that timed out
  double* geo = nullptr;   // 8 nodal + 4 face arrays
  double* xy = nullptr;    // device x,y (structured meshes)
  double* W[3] = {};       // current state
  double* A[3] = {};
  double* B[3] = {};
  double* R[3] = {};       // rhs output
  double *eps = nullptr, *r_ind = nullptr;
  double *fvu = nullptr, *fvv = nullptr, *gvu = nullptr, *gvv = nullptr;
  double *fh = nullptr, *fhu = nullptr, *fhv = nullptr;
  double *partial = nullptr, *sums = nullptr;
  int int_lo = 0, int_hi = 0;   // interior element range (halo overlap), empty by default
  int reserve_sms = 0;          // SMs the next stage launch leaves free
  bool no_graphs = std::getenv("SWDG_NO_GRAPHS") != nullptr;  // A/B: eager launches
  int* gctr = nullptr;          // device group counter of the persistent stage kernels
  // device report: Flags[4] (one per stage + one for the step reductions) and the
  // mass/entropy sums, contiguous so one copy (one host sync) reads a whole step
  Report* rep = nullptr;        // device
  Report* rep_h = nullptr;      // pinned host mirror
  Flags* flags = nullptr;       // rep->f
  Flags* flags_init = nullptr;  // device, reset image (4)
  Flags* flags_h = nullptr;     // rep_h->f
  double* sums_h = nullptr;     // rep_h->sums
  // TimeIntegrator::track_limiter_entropy (timeloop.hpp:197): the worst
  // per-element limiter entropy jump, accumulated over the context's life
  bool track_entropy = false;
  unsigned long long* ent_key = nullptr;  // device, order key
  // asynchronous snapshot: a D2H copy of the state on its own stream, overlapping
  // the following steps; the buffer it reads is fenced (snap_done) before any
  // launch or copy writes it again
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t snap_ready = nullptr, snap_done = nullptr;
  const double* snap_buf = nullptr;  // W[0] when the copy was issued; null when none pending
  // CUDA graph of two device-resident steps (the W/A ping-pong returns to its
  // starting assignment after two) for fixed-dt stepping: one launch per two
  // steps instead of ~2 x (3 stage kernels + 3 counter memsets + reductions)
  cudaStream_t graph_stream = nullptr;
  cudaEvent_t graph_in = nullptr, graph_out = nullptr;
  cudaGraphExec_t graph = nullptr;
  double graph_dt = 0.0;
  bool graph_red = false;
  const double* graph_w0 = nullptr;
  int64_t graph_launches = 0;  // kernels per replay

  std::vector<double> x, y, eps_h, r_h, fbuf;
  swdg_forcing_fn forcing = nullptr;
  void* forcing_user = nullptr;
  swdg_step_info last{};

  // partitioned runs: halo node lists (device) and the split-step state
  int* send_idx = nullptr;
  int* recv_idx = nullptr;
  long long n_send = 0, n_recv = 0;
  double split_max_eps = 0.0;

  template <class T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    allocations.push_back(p);
    return static_cast<T*>(p);
  }
  ~swdg_gpu() {
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (void* p : allocations) cudaFree(p);
    if (rep_h) cudaFreeHost(rep_h);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (graph) cudaGraphExecDestroy(graph);
    if (graph_stream) cudaStreamDestroy(graph_stream);
    if (graph_in) cudaEventDestroy(graph_in);
    if (graph_out) cudaEventDestroy(graph_out);
    if (snap_ready) cudaEventDestroy(snap_ready);
    if (snap_done) cudaEventDestroy(snap_done);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {

int fail(swdg_gpu* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

template <class F>
int guarded(swdg_gpu* c, F&& body) {
  if (!c) return SWDG_ERR_INPUT;
  try {
    cudaSetDevice(c->device);
    return body();
  } catch (const CudaError& e) {
    return fail(c, SWDG_ERR_CUDA, std::string(e.where) + ": " + cudaGetErrorString(e.e));
  } catch (const InputError& e) {
    return fail(c, SWDG_ERR_INPUT, e.msg);
  } catch (const std::exception& e) {
    return fail(c, SWDG_ERR_CUDA, e.what());
  }
}

// viscosity_coefficient (viscosity.hpp:69-78) on the host with the same libm
// the reference uses; sigma = log10(r) finishes shock_indicator (:64).
double ramp(double r, const swdg_params& p) {
  const double sigma = r <= 0.0 ? -std::numeric_limits<double>::infinity() : std::log10(r);
  if (sigma < p.sigma_min) return 0.0;
  if (sigma >= p.sigma_max) return p.epsilon0;
  const double delta =
      1.0 + std::sin(M_PI * (sigma - 0.5 * (p.sigma_max + p.sigma_min)) / (p.sigma_max - p.sigma_min));
  return 0.5 * p.epsilon0 * delta;
}

void reset_flags(swdg_gpu* c) {
  ck(cudaMemcpyAsync(c->flags, c->flags_init, 4 * sizeof(Flags), cudaMemcpyDeviceToDevice,
                     c->stream), "reset flags");
}

// the whole device report (stage flags, step reductions, sums): one copy, one sync
void read_flags(swdg_gpu* c) {
  ck(cudaMemcpyAsync(c->rep_h, c->rep, sizeof(Report), cudaMemcpyDeviceToHost, c->stream),
     "read flags");
  ck(cudaStreamSynchronize(c->stream), "sync flags");
}

// compute_dt's result (timeloop.hpp:72-74) from the reduced candidates in the
// step-reduction flags: the CFL minimum, or the all-dry fallback
double cfl_dt(swdg_gpu* c, double cfl) {
  const Flags& f = c->flags_h[kDiagFlags];
  double d = key_value(f.dt_key);
  if (!std::isfinite(d)) {
    const double order = 2.0 * c->M.degree + 1.0;
    d = key_value(f.minlen_key) / (order * std::sqrt(c->params.g * std::max(c->params.h_ref, 1e-12)));
  }
  return cfl * d;
}

void diag_out(swdg_gpu* c, swdg_diagnostics* out) {
  out->mass = c->sums_h[0];
  out->entropy = c->sums_h[1];
  out->min_h = key_value(c->flags_h[kDiagFlags].min_h_key);
  out->positivity_dt = key_value(c->flags_h[kDiagFlags].posdt_key);
}

// Before anything writes the state buffer `buf` (three fields at one base), the
// compute stream waits for a pending snapshot copy that reads it.
void fence_snapshot(swdg_gpu* c, double* const* buf) {
  if (c->snap_buf && c->snap_buf == buf[0]) {
    ck(cudaStreamWaitEvent(c->stream, c->snap_done, 0), "snapshot fence");
    c->snap_buf = nullptr;
  }
}

CState cs(double* const* a) { return CState{a[0], a[1], a[2]}; }
State st(double* const* a) { return State{a[0], a[1], a[2]}; }

// Per-stage viscosity (compute_viscosity viscosity.hpp:250-259 + the velocity
// loop and br1/viscous flux pairs of evaluate_rhs timeloop.hpp:176-187).
// Returns max eps.
double stage_viscosity(swdg_gpu* c, CState in) {
  c->launches += launched(launch_exact_indicator(c->M, in, c->r_ind, c->stream), "launch_exact_indicator");
  ck(cudaMemcpyAsync(c->r_h.data(), c->r_ind, sizeof(double) * c->M.K, cudaMemcpyDeviceToHost,
                     c->stream), "indicator D2H");
  ck(cudaStreamSynchronize(c->stream), "indicator sync");
  // owned elements only: a partition's ghost elements hold only face traces (their
  // viscous flux pairs arrive by the halo exchange), so their eps is 0, not a ramp
  // of stale interior data
  double mx = 0.0;
  for (int e = 0; e < c->M.K; ++e) {
    c->eps_h[e] = e < c->M.n_owned ? ramp(c->r_h[e], c->params) : 0.0;
    mx = std::max(mx, c->eps_h[e]);
  }
  ck(cudaMemcpyAsync(c->eps, c->eps_h.data(), sizeof(double) * c->M.K, cudaMemcpyHostToDevice,
                     c->stream), "eps H2D");
  c->launches += launched(launch_exact_grad(c->M, c->phys, in, c->eps, c->fvu, c->fvv, c->gvu, c->gvv,
                                   c->stream), "launch_exact_grad");
  return mx;
}

void ensure_xy(swdg_gpu* c) {
  if (!c->x.empty() || !c->xy) return;
  c->x.resize(c->nn);
  c->y.resize(c->nn);
  ck(cudaMemcpy(c->x.data(), c->xy, c->nn * sizeof(double), cudaMemcpyDeviceToHost), "x D2H");
  ck(cudaMemcpy(c->y.data(), c->xy + c->nn, c->nn * sizeof(double), cudaMemcpyDeviceToHost),
     "y D2H");
}

bool stage_forcing(swdg_gpu* c, double ts) {
  if (!c->forcing) return false;
  const long long nn = c->nn;
  c->forcing(c->forcing_user, ts, nn, c->x.data(), c->y.data(), c->fbuf.data(),
             c->fbuf.data() + nn, c->fbuf.data() + 2 * nn);
  ck(cudaMemcpyAsync(c->fh, c->fbuf.data(), sizeof(double) * 3 * nn, cudaMemcpyHostToDevice,
                     c->stream), "forcing H2D");
  // the host buffer is reused at the next stage: make the copy complete
  ck(cudaStreamSynchronize(c->stream), "forcing sync");
  return true;
}

// dW/dt of `in` (+ optional stage update into `out`, limiter into flags[k]).
// Returns max eps.
// Viscous pre-pass of a stage input: eps, BR1 gradients and the flux pairs into
// c->fvu.. (fast: one device kernel, max eps into F; exact: indicator on the
// device, ramp on the host).  Returns the host-side max eps (exact mode).
double stage_visc(swdg_gpu* c, CState in, Flags* F, const Mesh* range = nullptr) {
  if (c->fast) {
    if (range && range->n_owned <= range->e_lo) return 0.0;  // empty boundary slab
    c->launches += launched(launch_fast_visc_pre(range ? *range : c->M, c->phys, in, c->eps, c->fvu, c->fvv, c->gvu,
                                        c->gvv, F, c->stream), "launch_fast_visc_pre");
    return 0.0;
  }
  return stage_viscosity(c, in);
}

// The stage proper: dW/dt of `in` (+ update into `out` and the limiter/reject
// flags in F), consuming the flux pairs of a preceding stage_visc.
void stage_main(swdg_gpu* c, CState in, double* const* out, int k, double t, double dt,
                bool viscous, double* const* rhs, Flags* F, const Mesh* range = nullptr) {
  StageArgs a{};
  a.in = in;
  a.wn = cs(c->W);
  a.dt = dt;
  a.ca = kCa[k];
  a.cb = kCb[k];
  a.stage = k;
  a.t = t + kCt[k] * dt;
  a.update = out != nullptr;
  if (out) a.out = st(out);
  if (rhs) a.rhs = st(rhs);
  // limiter entropy tracking needs the stage's dW/dt to rebuild the pre-limit state
  const bool track = c->track_entropy && out && c->params.limiter_enabled;
  if (track && !rhs) a.rhs = st(c->R);
  if (viscous) {
    a.eps = c->eps;
    a.fvu = c->fvu;
    a.fvv = c->fvv;
    a.gvu = c->gvu;
    a.gvv = c->gvv;
  }
  if (stage_forcing(c, a.t)) {
    a.fh = c->fh;
    a.fhu = c->fhu;
    a.fhv = c->fhv;
  }
  const Mesh& M = range ? *range : c->M;
  a.reserve_sms = c->reserve_sms;
  if (out) fence_snapshot(c, out);
  if (c->fast) {
    ck(cudaMemsetAsync(c->gctr, 0, sizeof(int), c->stream), "group counter");
    a.gctr = c->gctr;
    if (M.n_owned > M.e_lo) c->launches += launched(launch_fast_stage(M, c->phys, a, F, c->stream), "launch_fast_stage");
  } else {
    c->launches += launched(launch_exact_rhs_stage(c->M, c->phys, a, c->stream), "launch_exact_rhs_stage");
    if (out) c->launches += launched(launch_exact_limit(c->M, c->phys, st(out), F, c->stream), "launch_exact_limit");
  }
  if (track)
    c->launches += launched(launch_limiter_entropy(c->fast ? M : c->M, c->phys, a, F, c->ent_key,
                                                   c->stream), "launch_limiter_entropy");
}

double stage(swdg_gpu* c, CState in, double* const* out, int k, double t, double dt,
             bool viscous, double* const* rhs, Flags* F) {
  const double mx = viscous ? stage_visc(c, in, F) : 0.0;
  stage_main(c, in, out, k, t, dt, viscous, rhs, F);
  return mx;
}

void upload(double* dst, const double* src, size_t n, const char* what) {
  if (!src) throw InputError{std::string("mesh view: missing array ") + what};
  ck(cudaMemcpy(dst, src, n * sizeof(double), cudaMemcpyHostToDevice), what);
}

void validate_params(const swdg_params* p, int N) {
  if (N < 1 || N > 15) throw InputError{"degree must be in [1, 15]"};
  if (p->visc_enabled && N < 2)
    throw InputError{"artificial viscosity requires polynomial degree >= 2"};
  if (p->visc_enabled && !(p->sigma_min < p->sigma_max))
    throw InputError{"viscosity: sigma_min must be < sigma_max"};
  if (p->visc_enabled && p->epsilon0 < 0.0) throw InputError{"viscosity: epsilon0 must be >= 0"};
  if (p->mode != SWDG_MODE_EXACT && p->mode != SWDG_MODE_FAST)
    throw InputError{"unknown arithmetic mode"};
  if (p->scheme != SWDG_SCHEME_ES && p->scheme != SWDG_SCHEME_STANDARD)
    throw InputError{"unknown scheme"};
}

// element-face connectivity from MeshTopology::faces (mesh.hpp:46-54)
std::vector<int4> connectivity(int K, const swdg_face* faces, int n_faces) {
  std::vector<int4> ef(4 * (size_t)K, int4{-1, 0, 0, 0});
  auto claim = [&](int e, int f, int4 v) {
    if (e < 0 || e >= K || f < 0 || f > 3) throw InputError{"face list: element/face out of range"};
    if (ef[4 * e + f].y & EF_PRESENT) throw InputError{"face list: element face listed twice"};
    ef[4 * e + f] = v;
  };
  for (int i = 0; i < n_faces; ++i) {
    const swdg_face& f = faces[i];
    const int rev = f.reversed ? EF_REVERSED : 0;
    if (f.tag == SWDG_TAG_WALL) {
      claim(f.elem_minus, f.face_minus, int4{-1, EF_PRESENT | EF_MINUS | EF_WALL, i, 0});
    } else if (f.tag == SWDG_TAG_INTERIOR) {
      if (f.face_plus < 0 || f.face_plus > 3) throw InputError{"face list: bad plus face"};
      claim(f.elem_minus, f.face_minus,
            int4{f.elem_plus, EF_PRESENT | EF_MINUS | rev | f.face_plus, i, 0});
      claim(f.elem_plus, f.face_plus, int4{f.elem_minus, EF_PRESENT | rev | f.face_minus, i, 0});
    } else {
      throw InputError{"exterior_state: unknown boundary tag"};
    }
  }
  return ef;
}

// Device allocation shared by both constructors.  Geometry arrays are left for
// the caller to fill.
void allocate(swdg_gpu* c, int K, int n_owned, int N, const std::vector<int4>& ef,
              const double* ops_w, const double* ops_d, const double* ops_dt,
              const double* ops_dh, const double* ops_vinv) {
  const int n1 = N + 1, np = n1 * n1;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw CudaError{cudaErrorNoDevice, "no CUDA device (there is no CPU fallback)"};
  ck(cudaSetDevice(c->device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
  c->own_stream = true;
  const long long nn = (long long)K * np, nf = (long long)K * 4 * n1;
  c->nn = nn;
  c->nf = nf;
  // nodal arrays sit at a padded stride: every array starts 16-byte aligned,
  // a bulk copy of the last partial element group may round up by 8 bytes, and
  // consecutive arrays are staggered by an odd multiple of 256 bytes so the
  // same node of different fields does not land on the same DRAM channel
  static const long long kStagger = [] {  // SWDG_NNP_PAD: experiments only
    const char* s = getenv("SWDG_NNP_PAD");
    return s ? (atoll(s) & ~1ll) : 544ll;
  }();
  const long long nnp = ((nn + 511) & ~511ll) + kStagger;
  c->geo = c->dalloc<double>(10 * nnp + 4 * nf);
  double* ops = c->dalloc<double>(n1 + 4 * np);
  upload(ops, ops_w, n1, "weights");
  upload(ops + n1, ops_d, np, "deriv");
  upload(ops + n1 + np, ops_dt, np, "deriv_modified");
  upload(ops + n1 + 2 * np, ops_dh, np, "deriv_weak");
  upload(ops + n1 + 3 * np, ops_vinv, np, "vandermonde_inv");
  int4* def = c->dalloc<int4>(ef.size());
  ck(cudaMemcpy(def, ef.data(), ef.size() * sizeof(int4), cudaMemcpyHostToDevice), "ef");

  Mesh& M = c->M;
  M.K = K;
  M.n_owned = n_owned;
  M.e_lo = 0;
  M.n1 = n1;
  M.np = np;
  M.degree = N;
  M.w0 = ops_w[0];
  M.w = ops;
  M.D = ops + n1;
  M.Dt = ops + n1 + np;
  M.Dh = ops + n1 + 2 * np;
  M.Vinv = ops + n1 + 3 * np;
  double* geo = c->geo;
  M.ye = geo;
  M.xe = geo + nnp;
  M.yx = geo + 2 * nnp;
  M.xx = geo + 3 * nnp;
  M.jac = geo + 4 * nnp;
  M.b = geo + 5 * nnp;
  M.len_xi = geo + 6 * nnp;
  M.len_eta = geo + 7 * nnp;
  M.sx = geo + 8 * nnp;
  M.sy = geo + 9 * nnp;
  double* fgeo = geo + 10 * nnp;
  M.fnx = fgeo;
  M.fny = fgeo + nf;
  M.fjs = fgeo + 2 * nf;
  M.fa = fgeo + 3 * nf;
  M.ef = def;

  if (c->params.mode == SWDG_MODE_FAST) {
    const int rc = upload_fast_ops(n1, ops_d, ops_dt, ops_dh, ops_vinv, ops_w);
    if (rc == -1) throw InputError{"fast mode: operators differ from the LGL operators of this degree"};
    if (rc < 0) throw CudaError{cudaErrorInvalidSymbol, "upload operators"};
    c->fast = fast_stage_supported(n1);
  }

  double* sbuf = c->dalloc<double>(12 * nnp);
  for (int k = 0; k < 3; ++k) {
    c->W[k] = sbuf + k * nnp;
    c->A[k] = sbuf + (3 + k) * nnp;
    c->B[k] = sbuf + (6 + k) * nnp;
    c->R[k] = sbuf + (9 + k) * nnp;
  }
  ck(cudaMemset(sbuf, 0, 12 * nnp * sizeof(double)), "memset state");
  c->eps = c->dalloc<double>(K);
  c->r_ind = c->dalloc<double>(K);
  ck(cudaMemset(c->eps, 0, K * sizeof(double)), "memset eps");
  if (c->params.visc_enabled) {
    // padded stride like the state buffers: 16-byte aligned bases and slack for
    // the node kernel's bulk copies (one double before, one after a group)
    double* vb = c->dalloc<double>(4 * nnp);
    c->fvu = vb;
    c->fvv = vb + nnp;
    c->gvu = vb + 2 * nnp;
    c->gvv = vb + 3 * nnp;
  }
  c->partial = c->dalloc<double>(2 * (size_t)std::max(K, step_sum_partials()));
  c->rep = c->dalloc<Report>(1);
  c->flags = c->rep->f;
  c->sums = c->rep->sums;
  c->gctr = c->dalloc<int>(1);
  c->flags_init = c->dalloc<Flags>(4);
  c->ent_key = c->dalloc<unsigned long long>(1);
  ck(cudaMallocHost(&c->rep_h, sizeof(Report)), "pinned report");
  std::memset(c->rep_h, 0, sizeof(Report));
  c->flags_h = c->rep_h->f;
  c->sums_h = c->rep_h->sums;
  {
    const unsigned long long k0 = order_key(0.0);  // worst jump starts at 0 (timeloop.hpp:261)
    ck(cudaMemcpy(c->ent_key, &k0, sizeof(k0), cudaMemcpyHostToDevice), "ent key");
  }
  Flags f{};
  f.min_h_key = ~0ull;
  f.dt_key = ~0ull;
  f.minlen_key = ~0ull;
  f.posdt_key = ~0ull;
  f.max_eps_key = 0ull;  // atomicMax target (eps >= 0)
  for (int k = 0; k < 4; ++k) c->flags_h[k] = f;
  ck(cudaMemcpy(c->flags_init, c->flags_h, 4 * sizeof(Flags), cudaMemcpyHostToDevice), "flags");
  c->eps_h.assign(K, 0.0);
  c->r_h.assign(K, 0.0);
}

// The libm-dependent geometry of a device-generated mesh, with the host's glibc
// as the reference computes it: the face arrays (compute_metrics mesh.hpp:192-218:
// hypot, normals, J_surf, a = J / J_surf), the compute_dt lengths 2J/hypot
// (timeloop.hpp:62-65) and the sine bathymetries (sample_bathymetry :223-232).
// Chunks of elements, threads over elements; the polynomial work stays on the
// device.
void finish_mesh_on_host(swdg_gpu* c, const swdg_structured_spec& spec, int n1) {
  const Mesh& M = c->M;
  const int np = n1 * n1, K = M.K;
  const bool bathy = bathy_needs_libm(spec.bathy_kind);
  const int chunk = std::max(1, (1 << 22) / np);  // ~4M nodes per chunk
  std::vector<double> ye, xe, yx, xx, jac, x, y, lx, le, b, fj, fx, fy, fa;
  auto dl = [&](std::vector<double>& h, const double* d, long long off, long long n) {
    h.resize(n);
    ck(cudaMemcpy(h.data(), d + off, n * sizeof(double), cudaMemcpyDeviceToHost), "geometry D2H");
  };
  auto ul = [&](double* d, const std::vector<double>& h, long long off) {
    ck(cudaMemcpy(d + off, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice),
       "geometry H2D");
  };
  const unsigned nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  for (int e0 = 0; e0 < K; e0 += chunk) {
    const int ne = std::min(chunk, K - e0);
    const long long n0 = (long long)e0 * np, nn = (long long)ne * np;
    const long long f0 = (long long)e0 * 4 * n1, nf = (long long)ne * 4 * n1;
    dl(ye, M.ye, n0, nn);
    dl(xe, M.xe, n0, nn);
    dl(yx, M.yx, n0, nn);
    dl(xx, M.xx, n0, nn);
    dl(jac, M.jac, n0, nn);
    if (bathy) {
      dl(x, c->xy, n0, nn);
      dl(y, c->xy + c->nn, n0, nn);
      b.resize(nn);
    }
    lx.resize(nn);
    le.resize(nn);
    fj.resize(nf);
    fx.resize(nf);
    fy.resize(nf);
    fa.resize(nf);
    const double* p = spec.bathy;
    auto work = [&](int t) {
      for (int el = t; el < ne; el += (int)nthreads) {
        const long long a = (long long)el * np;
        for (int q = 0; q < np; ++q) {
          const long long n = a + q;
          lx[n] = 2.0 * jac[n] / std::hypot(xe[n], ye[n]);
          le[n] = 2.0 * jac[n] / std::hypot(xx[n], yx[n]);
          if (bathy)
            b[n] = spec.bathy_kind == 4
                       ? 0.1 + 0.05 * std::sin(2.0 * M_PI * x[n]) * std::sin(2.0 * M_PI * y[n])
                       : p[0] + p[1] * std::sin(p[2] * x[n]) * std::sin(p[2] * y[n]);
        }
        for (int face = 0; face < 4; ++face)
          for (int tt = 0; tt < n1; ++tt) {
            const long long n = a + face_node(n1, face, tt);
            const long long f = ((long long)el * 4 + face) * n1 + tt;
            double js, nx, ny;
            if (face == 1) {  // east
              js = std::hypot(ye[n], xe[n]);
              nx = ye[n] / js;
              ny = -xe[n] / js;
            } else if (face == 3) {  // west
              js = std::hypot(ye[n], xe[n]);
              nx = -ye[n] / js;
              ny = xe[n] / js;
            } else if (face == 2) {  // north
              js = std::hypot(yx[n], xx[n]);
              nx = -yx[n] / js;
              ny = xx[n] / js;
            } else {  // south
              js = std::hypot(yx[n], xx[n]);
              nx = yx[n] / js;
              ny = -xx[n] / js;
            }
            fj[f] = js;
            fx[f] = nx;
            fy[f] = ny;
            fa[f] = jac[n] / js;
          }
      }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nthreads; ++t) pool.emplace_back(work, (int)t);
    work(0);
    for (auto& th : pool) th.join();
    auto wr = [](const double* q) { return const_cast<double*>(q); };
    ul(wr(M.len_xi), lx, n0);
    ul(wr(M.len_eta), le, n0);
    ul(wr(M.fjs), fj, f0);
    ul(wr(M.fnx), fx, f0);
    ul(wr(M.fny), fy, f0);
    ul(wr(M.fa), fa, f0);
    if (bathy) ul(wr(M.b), b, n0);
  }
}

swdg_gpu* new_context(const swdg_params* p, int device) {
  auto* c = new swdg_gpu;
  c->device = device;
  c->params = *p;
  // the standard scheme has no artificial viscosity (evaluate_rhs
  // timeloop.hpp:178 adds it for SchemeMode::es only) and runs the exact kernels
  if (p->scheme == SWDG_SCHEME_STANDARD) {
    c->params.visc_enabled = 0;
    c->params.mode = SWDG_MODE_EXACT;
  }
  c->phys = Phys{p->g, p->h_tol, p->h_des, p->h_ref, p->epsilon0, p->sigma_min,
                 p->sigma_max, c->params.visc_enabled, p->limiter_enabled,
                 p->scheme == SWDG_SCHEME_STANDARD ? 1 : 0};
  return c;
}

template <class F>
int create_guarded(swdg_gpu* c, swdg_gpu** out, F&& body) {
  try {
    body();
    // fast mode: geometry-only split-source coefficients, once per mesh
    if (c->params.mode == SWDG_MODE_FAST)
      c->launches += launched(launch_source_geometry(c->M, const_cast<double*>(c->M.sx),
                                            const_cast<double*>(c->M.sy), c->stream), "launch_source_geometry");
    ck(cudaDeviceSynchronize(), "create sync");
  } catch (const CudaError& e) {
    g_create_error = std::string(e.where) + ": " + cudaGetErrorString(e.e);
    delete c;
    return SWDG_ERR_CUDA;
  } catch (const InputError& e) {
    g_create_error = e.msg;
    delete c;
    return SWDG_ERR_INPUT;
  }
  *out = c;
  return SWDG_OK;
}

}  // namespace

extern "C" {

const char* swdg_gpu_create_error(void) { return g_create_error.c_str(); }

int swdg_gpu_create(const swdg_mesh_view* mv, const swdg_params* p, int device,
                    swdg_gpu** out) {
  *out = nullptr;
  g_create_error.clear();
  if (!mv || !p) {
    g_create_error = "null mesh or params";
    return SWDG_ERR_INPUT;
  }
  swdg_gpu* c = new_context(p, device);
  return create_guarded(c, out, [&] {
    const int N = mv->degree, n1 = N + 1, np = n1 * n1, K = mv->n_elem;
    validate_params(p, N);
    if (K < 1) throw InputError{"mesh has no elements"};
    const int n_owned = mv->n_owned > 0 ? mv->n_owned : K;
    if (n_owned > K) throw InputError{"n_owned exceeds n_elem"};
    const std::vector<int4> ef = connectivity(K, mv->faces, mv->n_faces);
    // check_unit_normal (physics.hpp:71-74) for every face node a flux visits
    for (int i = 0; i < mv->n_faces; ++i) {
      const swdg_face& f = mv->faces[i];
      for (int t = 0; t < n1; ++t) {
        const long long fm = ((long long)f.elem_minus * 4 + f.face_minus) * n1 + t;
        const double nx = mv->face_nx[fm], ny = mv->face_ny[fm];
        if (std::abs(std::sqrt(nx * nx + ny * ny) - 1.0) > 1e-10)
          throw InputError{"normal vector is not unit length"};
      }
    }
    allocate(c, K, n_owned, N, ef, mv->weights, mv->deriv, mv->deriv_modified, mv->deriv_weak,
             mv->vandermonde_inv);
    const long long nn = (long long)K * np, nf = (long long)K * 4 * n1;
    Mesh& M = c->M;
    upload(const_cast<double*>(M.ye), mv->y_eta, nn, "y_eta");
    upload(const_cast<double*>(M.xe), mv->x_eta, nn, "x_eta");
    upload(const_cast<double*>(M.yx), mv->y_xi, nn, "y_xi");
    upload(const_cast<double*>(M.xx), mv->x_xi, nn, "x_xi");
    upload(const_cast<double*>(M.jac), mv->jac, nn, "jac");
    upload(const_cast<double*>(M.b), mv->b, nn, "b");
    {
      // compute_dt lengths 2J/|(x_eta,y_eta)|, 2J/|(x_xi,y_xi)| (timeloop.hpp:62-65),
      // geometry-only: evaluated once with the reference's libm hypot
      std::vector<double> lx(nn), le(nn);
      for (long long n = 0; n < nn; ++n) {
        lx[n] = 2.0 * mv->jac[n] / std::hypot(mv->x_eta[n], mv->y_eta[n]);
        le[n] = 2.0 * mv->jac[n] / std::hypot(mv->x_xi[n], mv->y_xi[n]);
      }
      upload(const_cast<double*>(M.len_xi), lx.data(), nn, "len_xi");
      upload(const_cast<double*>(M.len_eta), le.data(), nn, "len_eta");
    }
    upload(const_cast<double*>(M.fnx), mv->face_nx, nf, "face_nx");
    upload(const_cast<double*>(M.fny), mv->face_ny, nf, "face_ny");
    upload(const_cast<double*>(M.fjs), mv->face_jsurf, nf, "face_jsurf");
    upload(const_cast<double*>(M.fa), mv->face_a, nf, "face_a");
    if (mv->x && mv->y) {
      c->x.assign(mv->x, mv->x + nn);
      c->y.assign(mv->y, mv->y + nn);
    }
  });
}

int swdg_gpu_create_structured(const swdg_structured_spec* s, const swdg_params* p, int device,
                               swdg_gpu** out) {
  return swdg_gpu_create_structured_part(s, p, device, 0, 0, nullptr, 0, nullptr, out);
}

int swdg_gpu_create_structured_part(const swdg_structured_spec* s, const swdg_params* p,
                                    int device, int32_t n_local, int32_t n_owned,
                                    const int32_t* local_to_global, int32_t n_faces,
                                    const swdg_face* local_faces, swdg_gpu** out) {
  *out = nullptr;
  g_create_error.clear();
  if (!s || !p) {
    g_create_error = "null spec or params";
    return SWDG_ERR_INPUT;
  }
  swdg_gpu* c = new_context(p, device);
  return create_guarded(c, out, [&] {
    const int N = s->degree, n1 = N + 1, np = n1 * n1;
    validate_params(p, N);
    if (s->kx < 1 || s->ky < 1) throw InputError{"mesh: element counts must be >= 1"};
    if (s->kind < 0 || s->kind > 2) throw InputError{"unknown mesh kind"};
    const long long Kg = (long long)s->kx * s->ky;
    const bool part = local_to_global != nullptr;
    const long long Kl = part ? n_local : Kg;
    if (Kl * np > (1ll << 31) - 1) throw InputError{"mesh too large for int32 node indices"};
    const int K = (int)Kl;
    std::vector<swdg_face> faces;
    if (part) {
      if (n_owned < 1 || n_owned > n_local) throw InputError{"partition: bad n_owned"};
      for (int i = 0; i < n_local; ++i)
        if (local_to_global[i] < 0 || local_to_global[i] >= Kg)
          throw InputError{"partition: global id out of range"};
      faces.assign(local_faces, local_faces + n_faces);
    } else {
      faces = swdg_host::structured_faces(s->kx, s->ky, s->periodic_x != 0, s->periodic_y != 0);
    }
    const std::vector<int4> ef = connectivity(K, faces.data(), (int)faces.size());
    std::vector<double> nodes(n1), w(n1), D(np), Dt(np), Dh(np), V(np), Vi(np);
    swdg_operators(N, nodes.data(), w.data(), D.data(), Dt.data(), Dh.data(), V.data(), Vi.data());
    allocate(c, K, part ? n_owned : K, N, ef, w.data(), D.data(), Dt.data(), Dh.data(),
             Vi.data());
    const long long nn = c->nn;
    c->xy = c->dalloc<double>(2 * nn);
    double* dnodes = c->dalloc<double>(n1);
    ck(cudaMemcpy(dnodes, nodes.data(), n1 * sizeof(double), cudaMemcpyHostToDevice), "nodes");
    int* bad = c->dalloc<int>(1);
    ck(cudaMemset(bad, 0, sizeof(int)), "memset");
    int* gid = nullptr;
    if (part) {
      gid = c->dalloc<int>(n_local);
      ck(cudaMemcpy(gid, local_to_global, n_local * sizeof(int), cudaMemcpyHostToDevice), "gid");
    }
    MeshSpecDev sd{s->kind, s->kx, s->ky, s->bathy_kind, s->x0, s->x1, s->y0, s->y1, s->extra,
                   {s->bathy[0], s->bathy[1], s->bathy[2], s->bathy[3]}, gid, Kl,
                   nullptr, nullptr, nullptr, nullptr};
    if (s->kind == SWDG_MESH_WAVY) {
      // sin(2 pi u) of every u the edge curves sample, with the host's libm
      // (build_wavy_mesh mesh.hpp:370-379 via structured_mesh :313-327)
      auto table = [&](int k, std::vector<double>& samp, std::vector<double>& edge) {
        samp.assign((size_t)k * (n1 + 2), 0.0);
        edge.assign((size_t)k + 1, 0.0);
        for (int e = 0; e <= k; ++e) edge[e] = std::sin(2.0 * M_PI * (static_cast<double>(e) / k));
        for (int e = 0; e < k; ++e) {
          const double a = static_cast<double>(e) / k, b = static_cast<double>(e + 1) / k;
          for (int q = 0; q < n1 + 2; ++q) {
            const double r = q < n1 ? nodes[q] : (q == n1 ? -1.0 : 1.0);
            const double t = 0.5 * (1.0 + r);
            samp[(size_t)e * (n1 + 2) + q] = std::sin(2.0 * M_PI * (a + t * (b - a)));
          }
        }
      };
      std::vector<double> su, sue, sv, sve;
      table(s->kx, su, sue);
      table(s->ky, sv, sve);
      double* tb = c->dalloc<double>(su.size() + sue.size() + sv.size() + sve.size());
      size_t off = 0;
      for (const std::vector<double>* v : {&su, &sue, &sv, &sve}) {
        ck(cudaMemcpy(tb + off, v->data(), v->size() * sizeof(double), cudaMemcpyHostToDevice),
           "sin table");
        off += v->size();
      }
      sd.sin_u = tb;
      sd.sin_ue = tb + su.size();
      sd.sin_v = sd.sin_ue + sue.size();
      sd.sin_ve = sd.sin_v + sv.size();
    }
    const Mesh& M = c->M;
    auto wr = [](const double* p) { return const_cast<double*>(p); };
    MeshOut o{c->xy, c->xy + nn, wr(M.xx), wr(M.xe), wr(M.yx), wr(M.ye), wr(M.jac), wr(M.b),
              wr(M.len_xi), wr(M.len_eta), wr(M.fnx), wr(M.fny), wr(M.fjs), wr(M.fa), bad};
    c->launches += launched(launch_structured_mesh(sd, dnodes, c->M.D, n1, o, c->stream), "launch_structured_mesh");
    int hbad = 0;
    ck(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "bad D2H");
    ck(cudaStreamSynchronize(c->stream), "mesh sync");
    if (hbad) throw InputError{"mesh rejected: nonpositive Jacobian"};
    finish_mesh_on_host(c, *s, n1);
  });
}

void swdg_gpu_destroy(swdg_gpu* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  delete c;
}

const char* swdg_gpu_last_error(const swdg_gpu* c) { return c ? c->err.c_str() : "null context"; }

int swdg_gpu_set_stream(swdg_gpu* c, void* stream) {
  return guarded(c, [&] {
    if (c->own_stream && c->stream) {
      ck(cudaStreamSynchronize(c->stream), "sync old stream");
      cudaStreamDestroy(c->stream);
      c->own_stream = false;
      c->stream = nullptr;
    }
    // the caller's stream, NULL included (the legacy default stream): kernels,
    // copies and the caller's own work (NCCL, events) are then stream-ordered
    c->stream = static_cast<cudaStream_t>(stream);
    return SWDG_OK;
  });
}

int swdg_gpu_synchronize(swdg_gpu* c) {
  return guarded(c, [&] {
    ck(cudaStreamSynchronize(c->stream), "synchronize");
    return SWDG_OK;
  });
}

int swdg_gpu_upload_state(swdg_gpu* c, const double* h, const double* hu, const double* hv) {
  return guarded(c, [&] {
    fence_snapshot(c, c->W);
    const double* src[3] = {h, hu, hv};
    for (int k = 0; k < 3; ++k)
      ck(cudaMemcpyAsync(c->W[k], src[k], c->nn * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream), "upload state");
    ck(cudaStreamSynchronize(c->stream), "upload sync");
    return SWDG_OK;
  });
}

int swdg_gpu_download_state(swdg_gpu* c, double* h, double* hu, double* hv) {
  return guarded(c, [&] {
    double* dst[3] = {h, hu, hv};
    for (int k = 0; k < 3; ++k)
      ck(cudaMemcpyAsync(dst[k], c->W[k], c->nn * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream), "download state");
    ck(cudaStreamSynchronize(c->stream), "download sync");
    return SWDG_OK;
  });
}

int swdg_gpu_device_state(swdg_gpu* c, double** h, double** hu, double** hv) {
  return guarded(c, [&] {
    *h = c->W[0];
    *hu = c->W[1];
    *hv = c->W[2];
    return SWDG_OK;
  });
}

int swdg_gpu_download_geometry(swdg_gpu* c, const char* name, double* out) {
  return guarded(c, [&] {
    const std::string n(name);
    const double* src = nullptr;
    long long len = c->nn;
    const Mesh& M = c->M;
    if (n == "y_eta") src = M.ye;
    else if (n == "x_eta") src = M.xe;
    else if (n == "y_xi") src = M.yx;
    else if (n == "x_xi") src = M.xx;
    else if (n == "jac") src = M.jac;
    else if (n == "b") src = M.b;
    else if (n == "x" && c->xy) src = c->xy;
    else if (n == "y" && c->xy) src = c->xy + c->nn;
    else {
      len = c->nf;
      if (n == "face_nx") src = M.fnx;
      else if (n == "face_ny") src = M.fny;
      else if (n == "face_jsurf") src = M.fjs;
      else if (n == "face_a") src = M.fa;
    }
    if (!src) throw InputError{"unknown geometry array " + n};
    ck(cudaMemcpy(out, src, len * sizeof(double), cudaMemcpyDeviceToHost), "geometry D2H");
    return SWDG_OK;
  });
}

static int rhs_common(swdg_gpu* c, double t, double* rh, double* rhu, double* rhv,
                      bool viscous) {
  return guarded(c, [&] {
    reset_flags(c);
    stage(c, cs(c->W), nullptr, 0, t, 0.0, viscous, c->R, c->flags);
    double* dst[3] = {rh, rhu, rhv};
    for (int k = 0; k < 3; ++k)
      ck(cudaMemcpyAsync(dst[k], c->R[k], c->nn * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream), "rhs D2H");
    ck(cudaStreamSynchronize(c->stream), "rhs sync");
    return SWDG_OK;
  });
}

int swdg_gpu_evaluate_rhs(swdg_gpu* c, double t, double* rh, double* rhu, double* rhv) {
  return rhs_common(c, t, rh, rhu, rhv, c && c->params.visc_enabled);
}

int swdg_gpu_assemble_rhs(swdg_gpu* c, double t, double* rh, double* rhu, double* rhv) {
  if (!c) return SWDG_ERR_INPUT;
  swdg_forcing_fn saved = c->forcing;
  c->forcing = nullptr;
  const int rc = rhs_common(c, t, rh, rhu, rhv, false);
  c->forcing = saved;
  return rc;
}

int swdg_gpu_compute_dt(swdg_gpu* c, double cfl, double* dt) {
  return guarded(c, [&] {
    if (!(cfl > 0.0) || cfl > 1.0) throw InputError{"compute_dt: cfl must be in (0, 1]"};
    reset_flags(c);
    c->launches += launched(launch_cfl_dt(c->M, c->phys, cs(c->W), c->flags + kDiagFlags,
                                          c->stream, c->fast), "launch_cfl_dt");
    read_flags(c);
    *dt = cfl_dt(c, cfl);
    return SWDG_OK;
  });
}

// Fold per-stage flags into the reference's try_step report.  Returns the
// index of the first rejecting stage (3 = none).
static int fold_flags(swdg_gpu* c, swdg_step_info& r, int& code) {
  for (int k = 0; k < 3; ++k) {
    const Flags& f = c->flags_h[k];
    // eps of every evaluated stage counts, the rejected one included (timeloop.hpp:177-180)
    if (c->params.visc_enabled) r.max_eps = std::max(r.max_eps, key_value(f.max_eps_key));
    if (f.abort) {
      code = fail(c, SWDG_ERR_ABORT, "negative water height without limiter");
      return k;
    }
    if (f.reject) return k;
    if (c->params.limiter_enabled) r.n_limited = f.n_limited;
    r.min_stage_h = std::min(r.min_stage_h, key_value(f.min_h_key));
  }
  return 3;
}

// One SSPRK3 step of the device state (try_step timeloop.hpp:156-170).  With
// `diag`, the step reductions of the stage-3 output (the next state if the step
// is accepted) are queued behind the stages, so the device-resident driver reads
// flags, diagnostics and the next CFL candidate with ONE host synchronisation.
// Returns the error code; r.accepted says whether W advanced.
static int try_step_impl(swdg_gpu* c, double t, double dt, swdg_step_info& r, bool diag) {
  r = swdg_step_info{};
  r.min_stage_h = std::numeric_limits<double>::infinity();
  double* const* outs[3] = {c->A, c->B, c->A};
  CState in = cs(c->W);
  const bool viscous = c->params.visc_enabled != 0;
  int code = SWDG_OK;
  reset_flags(c);
  if (c->fast && !c->forcing) {
    // device-resident: three stages back to back, one flag read per step
    for (int k = 0; k < 3; ++k) {
      stage(c, in, outs[k], k, t, dt, viscous, nullptr, c->flags + k);
      in = cs(outs[k]);
    }
    if (diag)
      c->launches += launched(launch_diagnostics(c->M, c->phys, cs(c->A), c->partial, c->sums,
                                                 c->flags + kDiagFlags, c->stream, !c->fast),
                              "launch_diagnostics");
    read_flags(c);
    r.accepted = fold_flags(c, r, code) == 3 && code == SWDG_OK;
  } else {
    for (int k = 0; k < 3; ++k) {
      const double mx = stage(c, in, outs[k], k, t, dt, viscous, nullptr, c->flags + k);
      r.max_eps = std::max(r.max_eps, mx);
      read_flags(c);
      const Flags& f = c->flags_h[k];
      if (f.abort) {
        code = fail(c, SWDG_ERR_ABORT, "negative water height without limiter");
        break;
      }
      if (f.reject) break;
      if (c->params.limiter_enabled) r.n_limited = f.n_limited;
      r.min_stage_h = std::min(r.min_stage_h, key_value(f.min_h_key));
      in = cs(outs[k]);
      if (k == 2) r.accepted = 1;
    }
    if (diag && r.accepted) {
      c->launches += launched(launch_diagnostics(c->M, c->phys, cs(c->A), c->partial, c->sums,
                                                 c->flags + kDiagFlags, c->stream, !c->fast),
                              "launch_diagnostics");
      read_flags(c);
    }
  }
  if (r.accepted)
    for (int k = 0; k < 3; ++k) std::swap(c->W[k], c->A[k]);
  c->last = r;
  return code;
}

int swdg_gpu_try_step(swdg_gpu* c, double t, double dt, swdg_step_info* info) {
  return guarded(c, [&] {
    swdg_step_info r{};
    const int code = try_step_impl(c, t, dt, r, false);
    if (info) *info = r;
    return code;
  });
}

int swdg_gpu_step_device(swdg_gpu* c, double t, double dt, double cfl, swdg_step_report* out) {
  return guarded(c, [&] {
    if (!(cfl > 0.0) || cfl > 1.0) throw InputError{"compute_dt: cfl must be in (0, 1]"};
    swdg_step_report rep{};
    const int code = try_step_impl(c, t, dt, rep.info, true);
    if (rep.info.accepted) {
      diag_out(c, &rep.diag);
      rep.next_dt = cfl_dt(c, cfl);
    }
    if (out) *out = rep;
    return code;
  });
}

int swdg_gpu_run_steps_ex(swdg_gpu* c, int nsteps, double t, double dt, int flags) {
  return guarded(c, [&] {
    const bool viscous = c->params.visc_enabled != 0;
    const bool reductions = (flags & SWDG_RUN_STEP_REDUCTIONS) != 0;
    if (!(c->fast && !c->forcing)) {
      for (int s = 0; s < nsteps; ++s) {
        swdg_step_info r{};
        const int rc = try_step_impl(c, t + s * dt, dt, r, reductions);
        if (rc) return rc;
        if (!r.accepted) return SWDG_OK;  // c->last holds the reject
      }
      return SWDG_OK;
    }
    // device-resident: no host synchronisation; reject/abort/min h accumulate
    // over the run in the per-stage flags and are folded at the end
    reset_flags(c);
    double* const* outs[3] = {c->A, c->B, c->A};
    auto one_step = [&](double ts) {
      CState in = cs(c->W);
      for (int k = 0; k < 3; ++k) {
        stage(c, in, outs[k], k, ts, dt, viscous, nullptr, c->flags + k);
        in = cs(outs[k]);
      }
      // the per-step StepDiagnostics reductions and the next CFL candidate of the
      // new state, as the driver needs them every step (driver.hpp:92, 117-127)
      if (reductions)
        c->launches += launched(launch_diagnostics(c->M, c->phys, cs(c->A), c->partial, c->sums,
                                                   c->flags + kDiagFlags, c->stream, false),
                                "launch_diagnostics");
      for (int k = 0; k < 3; ++k) std::swap(c->W[k], c->A[k]);
    };
    int s0 = 0;
    if (nsteps >= 2 && !c->no_graphs) {
      // replay the two-step graph (re-captured when dt, the reductions flag or the
      // buffer assignment changed); the kernels' time argument only feeds forcing,
      // which this path excludes
      if (c->snap_buf) {  // a pending snapshot copy reads W: let it land first
        ck(cudaEventSynchronize(c->snap_done), "snapshot sync");
        c->snap_buf = nullptr;
      }
      if (!c->graph_stream) {
        ck(cudaStreamCreateWithFlags(&c->graph_stream, cudaStreamNonBlocking), "graph stream");
        ck(cudaEventCreateWithFlags(&c->graph_in, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->graph_out, cudaEventDisableTiming), "event");
      }
      bool stale = !c->graph || c->graph_dt != dt || c->graph_red != reductions;
      if (!stale && c->graph_w0 != c->W[0]) {  // odd step count last time: realign
        one_step(t);
        s0 = 1;
      }
      if (stale) {
        // one eager step first: first-launch work (shared-memory attributes,
        // occupancy queries) stays out of the capture
        one_step(t);
        s0 = 1;
        if (c->graph) cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
        cudaStream_t user = c->stream;
        c->stream = c->graph_stream;
        const int64_t l0 = c->launches;
        const double* w0 = c->W[0];
        ck(cudaStreamBeginCapture(c->graph_stream, cudaStreamCaptureModeThreadLocal), "capture");
        try {
          one_step(t + s0 * dt);
          one_step(t + (s0 + 1) * dt);
        } catch (...) {
          cudaGraph_t g = nullptr;
          cudaStreamEndCapture(c->graph_stream, &g);
          if (g) cudaGraphDestroy(g);
          c->stream = user;
          throw;
        }
        cudaGraph_t g = nullptr;
        ck(cudaStreamEndCapture(c->graph_stream, &g), "end capture");
        c->stream = user;
        ck(cudaGraphInstantiate(&c->graph, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        c->graph_launches = c->launches - l0;
        c->launches = l0;
        c->graph_dt = dt;
        c->graph_red = reductions;
        c->graph_w0 = w0;
      }
      ck(cudaEventRecord(c->graph_in, c->stream), "graph in");
      ck(cudaStreamWaitEvent(c->graph_stream, c->graph_in, 0), "graph wait");
      if (c->graph_w0 != c->W[0]) throw CudaError{cudaErrorUnknown, "graph buffer assignment"};
      for (; s0 + 2 <= nsteps; s0 += 2) {
        ck(cudaGraphLaunch(c->graph, c->graph_stream), "graph launch");
        c->launches += c->graph_launches;
      }
      ck(cudaEventRecord(c->graph_out, c->graph_stream), "graph out");
      ck(cudaStreamWaitEvent(c->stream, c->graph_out, 0), "graph join");
    }
    for (int s = s0; s < nsteps; ++s) one_step(t + s * dt);
    read_flags(c);
    swdg_step_info r{};
    r.min_stage_h = std::numeric_limits<double>::infinity();
    int code = SWDG_OK;
    r.accepted = fold_flags(c, r, code) == 3 && code == SWDG_OK;
    c->last = r;
    return code;
  });
}

int swdg_gpu_run_steps(swdg_gpu* c, int nsteps, double t, double dt) {
  return swdg_gpu_run_steps_ex(c, nsteps, t, dt, 0);
}

int swdg_gpu_last_info(swdg_gpu* c, swdg_step_info* info) {
  return guarded(c, [&] {
    *info = c->last;
    return SWDG_OK;
  });
}

int swdg_gpu_last_eps(swdg_gpu* c, double* eps) {
  return guarded(c, [&] {
    if (c->fast) {  // eps lives on the device in fast mode
      ck(cudaMemcpyAsync(eps, c->eps, sizeof(double) * c->M.K, cudaMemcpyDeviceToHost,
                         c->stream), "eps D2H");
      ck(cudaStreamSynchronize(c->stream), "eps sync");
    } else {
      std::memcpy(eps, c->eps_h.data(), sizeof(double) * c->M.K);
    }
    return SWDG_OK;
  });
}

int swdg_gpu_diagnostics(swdg_gpu* c, swdg_diagnostics* out) {
  return guarded(c, [&] {
    reset_flags(c);
    c->launches += launched(launch_diagnostics(c->M, c->phys, cs(c->W), c->partial, c->sums,
                                               c->flags + kDiagFlags, c->stream, !c->fast),
                            "launch_diagnostics");
    read_flags(c);
    diag_out(c, out);
    return SWDG_OK;
  });
}

int swdg_gpu_set_forcing(swdg_gpu* c, swdg_forcing_fn fn, void* user) {
  return guarded(c, [&] {
    if (fn) ensure_xy(c);
    if (fn && c->x.empty()) throw InputError{"forcing needs the mesh x/y arrays"};
    c->forcing = fn;
    c->forcing_user = user;
    if (fn && !c->fh) {
      double* fb = c->dalloc<double>(3 * c->nn);
      c->fh = fb;
      c->fhu = fb + c->nn;
      c->fhv = fb + 2 * c->nn;
      c->fbuf.assign(3 * c->nn, 0.0);
    }
    return SWDG_OK;
  });
}

int64_t swdg_gpu_launch_count(const swdg_gpu* c) { return c ? c->launches : 0; }

int swdg_gpu_set_grid_cap(int32_t max_ctas) {
  if (max_ctas < 0) return SWDG_ERR_INPUT;
  swdg_dev::g_grid_cap = max_ctas;
  return SWDG_OK;
}

// ---- stage buffers, per-stage report, limiter entropy tracking ------------

static double* const* stage_input(swdg_gpu* c, int k) {
  return k == 0 ? c->W : (k == 1 ? c->A : c->B);
}
static double* const* stage_output(swdg_gpu* c, int k) { return k == 1 ? c->B : c->A; }

int swdg_gpu_upload_stage_input(swdg_gpu* c, int k, const double* h, const double* hu,
                                const double* hv) {
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"upload_stage_input: bad stage"};
    const double* src[3] = {h, hu, hv};
    double* const* dst = stage_input(c, k);
    fence_snapshot(c, dst);
    for (int f = 0; f < 3; ++f)
      ck(cudaMemcpyAsync(dst[f], src[f], c->nn * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream), "upload stage input");
    ck(cudaStreamSynchronize(c->stream), "upload stage sync");
    return SWDG_OK;
  });
}

int swdg_gpu_download_stage_output(swdg_gpu* c, int k, double* h, double* hu, double* hv) {
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"download_stage_output: bad stage"};
    double* dst[3] = {h, hu, hv};
    double* const* src = stage_output(c, k);
    for (int f = 0; f < 3; ++f)
      ck(cudaMemcpyAsync(dst[f], src[f], c->nn * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream), "download stage output");
    ck(cudaStreamSynchronize(c->stream), "download stage sync");
    return SWDG_OK;
  });
}

int swdg_gpu_stage_info(swdg_gpu* c, int k, swdg_step_info* info) {
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"stage_info: bad stage"};
    read_flags(c);
    const Flags& f = c->flags_h[k];
    swdg_step_info r{};
    r.min_stage_h = key_value(f.min_h_key);
    r.max_eps = c->fast ? key_value(f.max_eps_key) : c->split_max_eps;
    r.n_limited = f.n_limited;
    r.accepted = !(f.reject || f.abort);
    *info = r;
    return f.abort ? fail(c, SWDG_ERR_ABORT, "negative water height without limiter") : SWDG_OK;
  });
}

int swdg_gpu_snapshot_async(swdg_gpu* c, double* h, double* hu, double* hv) {
  return guarded(c, [&] {
    if (!c->copy_stream) {
      ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
      ck(cudaEventCreateWithFlags(&c->snap_ready, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->snap_done, cudaEventDisableTiming), "event");
    }
    if (c->snap_buf) ck(cudaStreamWaitEvent(c->stream, c->snap_done, 0), "snapshot fence");
    ck(cudaEventRecord(c->snap_ready, c->stream), "snapshot ready");
    ck(cudaStreamWaitEvent(c->copy_stream, c->snap_ready, 0), "snapshot wait");
    double* dst[3] = {h, hu, hv};
    for (int f = 0; f < 3; ++f)
      ck(cudaMemcpyAsync(dst[f], c->W[f], c->nn * sizeof(double), cudaMemcpyDeviceToHost,
                         c->copy_stream), "snapshot D2H");
    ck(cudaEventRecord(c->snap_done, c->copy_stream), "snapshot done");
    c->snap_buf = c->W[0];
    return SWDG_OK;
  });
}

void* swdg_gpu_alloc_pinned(size_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}

void swdg_gpu_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

int swdg_gpu_snapshot_wait(swdg_gpu* c) {
  return guarded(c, [&] {
    if (c->snap_done) ck(cudaEventSynchronize(c->snap_done), "snapshot sync");
    return SWDG_OK;
  });
}

int swdg_gpu_set_track_limiter_entropy(swdg_gpu* c, int on) {
  return guarded(c, [&] {
    c->track_entropy = on != 0;
    return SWDG_OK;
  });
}

int swdg_gpu_worst_limiter_entropy_jump(swdg_gpu* c, double* out) {
  return guarded(c, [&] {
    unsigned long long k = 0;
    ck(cudaMemcpyAsync(&k, c->ent_key, sizeof(k), cudaMemcpyDeviceToHost, c->stream), "ent D2H");
    ck(cudaStreamSynchronize(c->stream), "ent sync");
    *out = key_value(k);
    return SWDG_OK;
  });
}

// ---- partitioned runs: halo exchange hooks and the split SSPRK3 step -------

int swdg_gpu_halo_setup(swdg_gpu* c, int64_t n_send, const int32_t* send_idx, int64_t n_recv,
                        const int32_t* recv_idx) {
  return guarded(c, [&] {
    const long long lim = c->nn;
    for (int64_t i = 0; i < n_send; ++i)
      if (send_idx[i] < 0 || send_idx[i] >= lim) throw InputError{"halo: send index out of range"};
    for (int64_t i = 0; i < n_recv; ++i)
      if (recv_idx[i] < 0 || recv_idx[i] >= lim) throw InputError{"halo: recv index out of range"};
    c->send_idx = c->dalloc<int>(n_send);
    c->recv_idx = c->dalloc<int>(n_recv);
    if (n_send)
      ck(cudaMemcpy(c->send_idx, send_idx, n_send * sizeof(int), cudaMemcpyHostToDevice), "send idx");
    if (n_recv)
      ck(cudaMemcpy(c->recv_idx, recv_idx, n_recv * sizeof(int), cudaMemcpyHostToDevice), "recv idx");
    c->n_send = n_send;
    c->n_recv = n_recv;
    return SWDG_OK;
  });
}

// what: 0 = state of stage k's input (3 fields), 1 = viscous flux pairs (4 fields)
int swdg_gpu_halo_pack(swdg_gpu* c, int what, int k, double* send_buf) {
  return guarded(c, [&] {
    if (k < 0 || k > 2 || what < 0 || what > 1) throw InputError{"halo_pack: bad stage/what"};
    if (what == 1 && !c->fvu) throw InputError{"halo_pack: viscosity is off"};
    double* const* in = stage_input(c, k);
    const double* f[4] = {in[0], in[1], in[2], nullptr};
    if (what == 1) {
      f[0] = c->fvu;
      f[1] = c->fvv;
      f[2] = c->gvu;
      f[3] = c->gvv;
    }
    c->launches += launched(launch_halo_pack(c->send_idx, c->n_send, what ? 4 : 3, f, send_buf, c->stream), "launch_halo_pack");
    return SWDG_OK;
  });
}

int swdg_gpu_halo_unpack(swdg_gpu* c, int what, int k, const double* recv_buf) {
  return guarded(c, [&] {
    if (k < 0 || k > 2 || what < 0 || what > 1) throw InputError{"halo_unpack: bad stage/what"};
    if (what == 1 && !c->fvu) throw InputError{"halo_unpack: viscosity is off"};
    double* const* in = stage_input(c, k);
    double* f[4] = {in[0], in[1], in[2], nullptr};
    if (what == 1) {
      f[0] = c->fvu;
      f[1] = c->fvv;
      f[2] = c->gvu;
      f[3] = c->gvv;
    }
    c->launches += launched(launch_halo_unpack(c->recv_idx, c->n_recv, what ? 4 : 3, f, recv_buf,
                                      c->stream), "launch_halo_unpack");
    return SWDG_OK;
  });
}

// ---- direct peer-memory halo exchange (CUDA IPC) --------------------------

int swdg_gpu_ipc_alloc(swdg_gpu* c, int64_t bytes, void** dptr, void* handle) {
  return guarded(c, [&] {
    if (bytes <= 0 || !dptr || !handle) throw InputError{"ipc_alloc: bad arguments"};
    char* p = c->dalloc<char>((size_t)bytes);
    ck(cudaMemset(p, 0, (size_t)bytes), "ipc_alloc memset");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof h);
    *dptr = p;
    return SWDG_OK;
  });
}

int swdg_gpu_ipc_open(swdg_gpu* c, const void* handle, void** dptr) {
  return guarded(c, [&] {
    if (!handle || !dptr) throw InputError{"ipc_open: bad arguments"};
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* p = nullptr;
    ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    c->ipc_opened.push_back(p);
    *dptr = p;
    return SWDG_OK;
  });
}

int swdg_gpu_halo_push(swdg_gpu* c, int what, int k, int64_t first, int64_t count, double* dst,
                       uint64_t* flag, const uint64_t* seq_base, uint64_t seq) {
  return guarded(c, [&] {
    if (k < 0 || k > 2 || what < 0 || what > 1) throw InputError{"halo_push: bad stage/what"};
    if (what == 1 && !c->fvu) throw InputError{"halo_push: viscosity is off"};
    if (first < 0 || count < 0 || first + count > c->n_send) throw InputError{"halo_push: bad range"};
    if (!flag || (count > 0 && !dst)) throw InputError{"halo_push: null destination"};
    double* const* in = stage_input(c, k);
    const double* f[4] = {in[0], in[1], in[2], nullptr};
    if (what == 1) {
      f[0] = c->fvu;
      f[1] = c->fvv;
      f[2] = c->gvu;
      f[3] = c->gvv;
    }
    c->launches += launched(launch_halo_push(c->send_idx + first, count, what ? 4 : 3, f, dst,
                                             reinterpret_cast<unsigned long long*>(flag),
                                             reinterpret_cast<const unsigned long long*>(seq_base),
                                             seq, c->stream), "launch_halo_push");
    return SWDG_OK;
  });
}

int swdg_gpu_halo_wait(swdg_gpu* c, const uint64_t* flags, int32_t n, const uint64_t* seq_base,
                       uint64_t seq, double timeout_s) {
  return guarded(c, [&] {
    if (n < 0 || (n > 0 && !flags)) throw InputError{"halo_wait: bad arguments"};
    if (!c->ipc_err) {
      c->ipc_err = c->dalloc<int>(1);
      ck(cudaMemset(c->ipc_err, 0, sizeof(int)), "ipc_err");
    }
    const unsigned long long tns = (unsigned long long)(std::max(timeout_s, 1e-3) * 1e9);
    c->launches += launched(launch_flags_wait(reinterpret_cast<const unsigned long long*>(flags), n,
                                              reinterpret_cast<const unsigned long long*>(seq_base),
                                              seq, tns, c->ipc_err, c->stream), "launch_flags_wait");
    return SWDG_OK;
  });
}

int swdg_gpu_seq_advance(swdg_gpu* c, uint64_t* seq_base, uint64_t by) {
  return guarded(c, [&] {
    if (!seq_base) throw InputError{"seq_advance: null base"};
    c->launches += launched(launch_seq_advance(reinterpret_cast<unsigned long long*>(seq_base), by,
                                               c->stream), "launch_seq_advance");
    return SWDG_OK;
  });
}

int swdg_gpu_halo_status(swdg_gpu* c, int32_t* timed_out) {
  return guarded(c, [&] {
    int v = 0;
    if (c->ipc_err) {
      ck(cudaStreamSynchronize(c->stream), "halo_status sync");
      ck(cudaMemcpy(&v, c->ipc_err, sizeof(int), cudaMemcpyDeviceToHost), "halo_status");
      if (v) ck(cudaMemset(c->ipc_err, 0, sizeof(int)), "halo_status reset");
    }
    *timed_out = v;
    return SWDG_OK;
  });
}

// compute_dt's two reductions before the cross-rank min (timeloop.hpp:57-74):
// min over owned nodes of the CFL candidates (inf if none) and of the lengths
int swdg_gpu_dt_candidates(swdg_gpu* c, double* dt_min, double* min_len) {
  return guarded(c, [&] {
    reset_flags(c);
    c->launches += launched(launch_cfl_dt(c->M, c->phys, cs(c->W), c->flags, c->stream, c->fast),
                            "launch_cfl_dt");
    read_flags(c);
    *dt_min = key_value(c->flags_h[0].dt_key);
    *min_len = key_value(c->flags_h[0].minlen_key);
    return SWDG_OK;
  });
}

int swdg_gpu_step_begin(swdg_gpu* c) {
  return guarded(c, [&] {
    reset_flags(c);
    c->split_max_eps = 0.0;
    return SWDG_OK;
  });
}

int swdg_gpu_stage_visc(swdg_gpu* c, int k, double t, double dt) {
  (void)t;
  (void)dt;
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"stage_visc: bad stage"};
    if (!c->params.visc_enabled) return SWDG_OK;
    const double mx = stage_visc(c, cs(stage_input(c, k)), c->flags + k);
    c->split_max_eps = std::max(c->split_max_eps, mx);
    return SWDG_OK;
  });
}

int swdg_gpu_stage_run(swdg_gpu* c, int k, double t, double dt) {
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"stage_run: bad stage"};
    stage_main(c, cs(stage_input(c, k)), stage_output(c, k), k, t, dt,
               c->params.visc_enabled != 0, nullptr, c->flags + k);
    return SWDG_OK;
  });
}

int swdg_gpu_stage_visc_part(swdg_gpu* c, int k, double t, double dt, int part) {
  (void)t;
  (void)dt;
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"stage_visc_part: bad stage"};
    if (part < 0 || part > 2) throw InputError{"stage_visc_part: bad part"};
    if (!c->params.visc_enabled) return SWDG_OK;
    const CState in = cs(stage_input(c, k));
    if (part == 0 || !c->fast || c->int_hi <= c->int_lo) {
      // exact mode (host ramp over all elements) and partitions without an
      // interior: everything after the exchange
      if (part != 1) c->split_max_eps = std::max(c->split_max_eps, stage_visc(c, in, c->flags + k));
      return SWDG_OK;
    }
    Mesh r = c->M;
    if (part == 1) {
      r.e_lo = c->int_lo;
      r.n_owned = c->int_hi;
      c->reserve_sms = kHaloReserveSms;
      stage_visc(c, in, c->flags + k, &r);
      c->reserve_sms = 0;
    } else {
      r.e_lo = 0;
      r.n_owned = c->int_lo;
      stage_visc(c, in, c->flags + k, &r);
      r.e_lo = c->int_hi;
      r.n_owned = c->M.n_owned;
      stage_visc(c, in, c->flags + k, &r);
    }
    return SWDG_OK;
  });
}

int swdg_gpu_set_interior(swdg_gpu* c, int32_t lo, int32_t hi) {
  return guarded(c, [&] {
    if (lo < 0 || hi < lo || hi > c->M.n_owned) throw InputError{"set_interior: bad range"};
    // even bounds keep the stage kernels' element groups 16-byte aligned
    lo = (lo + 1) & ~1;
    hi = hi & ~1;
    c->int_lo = lo;
    c->int_hi = hi > lo ? hi : lo;
    return SWDG_OK;
  });
}

int swdg_gpu_stage_run_part(swdg_gpu* c, int k, double t, double dt, int part) {
  return guarded(c, [&] {
    if (k < 0 || k > 2) throw InputError{"stage_run_part: bad stage"};
    if (part < 0 || part > 2) throw InputError{"stage_run_part: bad part"};
    const CState in = cs(stage_input(c, k));
    double* const* out = stage_output(c, k);
    const bool visc = c->params.visc_enabled != 0;
    if (part == 0 || !c->fast || c->int_hi <= c->int_lo) {
      // everything at once (exact mode and partitions without an interior run
      // all of it after the exchange)
      if (part != 1) stage_main(c, in, out, k, t, dt, visc, nullptr, c->flags + k);
      return SWDG_OK;
    }
    Mesh r = c->M;
    if (part == 1) {
      r.e_lo = c->int_lo;
      r.n_owned = c->int_hi;
      c->reserve_sms = kHaloReserveSms;  // the exchange runs concurrently
      stage_main(c, in, out, k, t, dt, visc, nullptr, c->flags + k, &r);
      c->reserve_sms = 0;
    } else {
      r.e_lo = 0;
      r.n_owned = c->int_lo;
      stage_main(c, in, out, k, t, dt, visc, nullptr, c->flags + k, &r);
      r.e_lo = c->int_hi;
      r.n_owned = c->M.n_owned;
      stage_main(c, in, out, k, t, dt, visc, nullptr, c->flags + k, &r);
    }
    return SWDG_OK;
  });
}

int swdg_gpu_step_flags(swdg_gpu* c, int32_t* reject, int32_t* abort) {
  return guarded(c, [&] {
    read_flags(c);
    *reject = 0;
    *abort = 0;
    // stage order, stopping at the first signal: the reference never evaluates
    // the stages after a reject (ssprk3_step timeloop.hpp:97-105)
    for (int k = 0; k < 3; ++k) {
      if (c->flags_h[k].abort) {
        *abort = 1;
        break;
      }
      if (c->flags_h[k].reject) {
        *reject = 1;
        break;
      }
    }
    return SWDG_OK;
  });
}

int swdg_gpu_step_commit(swdg_gpu* c, int accept, swdg_step_info* info) {
  return guarded(c, [&] {
    swdg_step_info r{};
    r.min_stage_h = std::numeric_limits<double>::infinity();
    int code = SWDG_OK;
    fold_flags(c, r, code);
    if (!c->fast) r.max_eps = std::max(r.max_eps, c->split_max_eps);
    r.accepted = accept ? 1 : 0;
    if (accept)
      for (int k = 0; k < 3; ++k) std::swap(c->W[k], c->A[k]);
    c->last = r;
    if (info) *info = r;
    return SWDG_OK;
  });
}

}  // extern "C"
