/*
 * swdg_gpu.h — C ABI of the B200 (sm_100a) ES-DGSEM shallow-water stage path.
 *
 * Drop-in boundary for the reference solver `swdg` (arXiv 1804.02221,
 * /root/reference/proj/include/swdg).  The reference has no plugin registry;
 * its seams are the free functions and the TimeIntegrator class below.  Each
 * entry point names the reference interface it replaces:
 *
 *   swdg_gpu_create          TimeIntegrator ctor          timeloop.hpp:148-151
 *                            (+ Mesh/Operators1D inputs   mesh.hpp:35-112, operators.hpp:35-52)
 *   swdg_gpu_try_step        TimeIntegrator::try_step     timeloop.hpp:156-170
 *                            ssprk3_step                  timeloop.hpp:88-108
 *                            post_stage (reject+limiter)  timeloop.hpp:202-234
 *   swdg_gpu_evaluate_rhs    TimeIntegrator::evaluate_rhs timeloop.hpp:173-190
 *   swdg_gpu_assemble_rhs    assemble_rhs (inviscid)      dg_rhs.hpp:267-303
 *   swdg_gpu_compute_dt      compute_dt                   timeloop.hpp:53-75
 *   swdg_gpu_diagnostics     total_mass/total_entropy/min_height  field.hpp:39-68
 *                            min_positivity_dt            limiter.hpp:135-166
 *   swdg_gpu_last_eps        TimeIntegrator::last_eps     timeloop.hpp:192
 *   swdg_gpu_set_forcing     TimeIntegrator::forcing      timeloop.hpp:198 (ForcingFn dg_rhs.hpp:255)
 *   swdg_gpu_set_track_limiter_entropy  TimeIntegrator::track_limiter_entropy timeloop.hpp:199
 *   swdg_gpu_worst_limiter_entropy_jump TimeIntegrator::worst_limiter_entropy_jump timeloop.hpp:196,
 *                            limited_entropy_check        limiter.hpp:88-101
 *   swdg_gpu_step_device     one run_simulation loop body driver.hpp:91-127
 *                            (try_step + total_mass/total_entropy/min_height/
 *                            min_positivity_dt + the next compute_dt)
 *
 * Conventions
 *   - Return codes: SWDG_OK; SWDG_ERR_INPUT mirrors SwdgError (core.hpp:63);
 *     SWDG_ERR_ABORT mirrors NumericalAbort (timeloop.hpp:46); these match the
 *     CLI exit codes 2/3 (tools/swdg_main.cpp:168-185).  SWDG_ERR_CUDA is a
 *     device/runtime failure (no reference counterpart).
 *   - All arrays are FP64, layouts exactly as in the reference: nodal arrays
 *     element-major e*(N+1)^2 + i*(N+1) + j (core.hpp:39-42), face arrays
 *     (e*4+face)*(N+1)+t (mesh.hpp:70-75), matrices row-major (operators.hpp:30-33).
 *   - Every host pointer is borrowed for the duration of the call only; the
 *     context deep-copies mesh data to the device and owns all device memory.
 *   - A context is single-threaded (the reference is single-threaded).
 *   - There is no CPU fallback: without a CUDA device every call that needs
 *     one returns SWDG_ERR_CUDA.
 */
#ifndef SWDG_GPU_H
#define SWDG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWDG_OK 0
#define SWDG_ERR_CUDA 1
#define SWDG_ERR_INPUT 2
#define SWDG_ERR_ABORT 3

/* Arithmetic modes.  EXACT replays the reference expression trees and
 * accumulation orders without FMA contraction (bitwise parity with the
 * reference built at its own flags, proj/CMakeLists.txt:6-8).  FAST is the
 * fused throughput kernel (FMA, symmetric two-point flux evaluation),
 * validated at 1e-12 normwise per stage. */
#define SWDG_MODE_EXACT 0
#define SWDG_MODE_FAST 1

/* Discretisation, SchemeMode (dg_rhs.hpp:14, RunConfig::mode timeloop.hpp:27).
 * ES: split-form entropy-conservative volume + entropy-stable interface flux
 * (the throughput path).  STANDARD: pointwise fluxes differentiated with D
 * (standard_volume_element dg_rhs.hpp:75-117) + the local Lax-Friedrichs
 * interface flux in strong form (llf_surface_flux fluxes.hpp:192-202,
 * surface_terms dg_rhs.hpp:228-246), no artificial viscosity (evaluate_rhs
 * timeloop.hpp:178).  STANDARD always runs the exact-mode kernels: it is the
 * paper's comparison scheme, bitwise with the reference, not a throughput path. */
#define SWDG_SCHEME_ES 0
#define SWDG_SCHEME_STANDARD 1

/* Face tags, BoundaryTag (mesh.hpp:30). */
#define SWDG_TAG_INTERIOR 0
#define SWDG_TAG_WALL 1

/* FaceInfo (mesh.hpp:35-44) without the periodic offsets (watertightness
 * diagnostics only, never read on the stage path). */
typedef struct swdg_face {
  int32_t elem_minus, face_minus, elem_plus, face_plus;
  int32_t reversed; /* plus-side nodes run opposite (MeshTopology::partner_node mesh.hpp:51) */
  int32_t tag;      /* SWDG_TAG_* */
} swdg_face;

/* Borrowed view of a reference Mesh (mesh.hpp:101-112): Operators1D
 * matrices, MeshGeometry arrays and MeshTopology.faces.  The metric-
 * premultiplied bathymetry products b_yeta... (mesh.hpp:67-68) are not
 * passed: sample_bathymetry (mesh.hpp:223-232) defines them as metric*b and
 * the device recomputes that product bitwise. */
typedef struct swdg_mesh_view {
  int32_t n_elem; /* K (elements stored, owned first) */
  int32_t degree; /* N */
  int32_t n_owned; /* elements [0,n_owned) are advanced; the rest are halo
                      (ghost) elements filled by swdg_gpu_halo_*; 0 = all */
  int32_t n_faces;
  const swdg_face* faces;
  /* Operators1D, n1 or n1*n1 entries */
  const double* weights;         /* LGL weights w */
  const double* deriv;           /* D */
  const double* deriv_modified;  /* Dtilde = 2D + S */
  const double* deriv_weak;      /* Dhat = -M^-1 D^T M */
  const double* vandermonde_inv; /* V^-1 */
  /* MeshGeometry nodal arrays, K*n1*n1 entries */
  const double *x, *y;
  const double *x_xi, *x_eta, *y_xi, *y_eta;
  const double* jac;
  const double* b;
  /* MeshGeometry face arrays, K*4*n1 entries */
  const double *face_jsurf, *face_nx, *face_ny, *face_a;
} swdg_mesh_view;

/* PhysicsParams (physics.hpp:11-16) + ViscosityConfig (viscosity.hpp:14-19)
 * + the stage-relevant RunConfig fields (timeloop.hpp:23-44). */
typedef struct swdg_params {
  double g, h_tol, h_des, h_ref;
  double epsilon0, sigma_min, sigma_max;
  int32_t visc_enabled;
  int32_t limiter_enabled;
  int32_t mode;   /* SWDG_MODE_* */
  int32_t scheme; /* SWDG_SCHEME_* (0 = ES) */
} swdg_params;

/* Per-try_step report: TimeIntegrator::last_limited_count / last_max_eps /
 * last_min_stage_h (timeloop.hpp:192-195). */
typedef struct swdg_step_info {
  double min_stage_h;
  double max_eps;
  int32_t n_limited;
  int32_t accepted;
} swdg_step_info;

/* StepDiagnostics fields computed from a state (driver.hpp:115-127). */
typedef struct swdg_diagnostics {
  double mass;
  double entropy;
  double min_h;
  double positivity_dt;
} swdg_diagnostics;

/* Host forcing callback standing in for ForcingFn (dg_rhs.hpp:255): fill
 * (fh,fhu,fhv)[n] = forcing(x[n], y[n], t) for n < count. */
typedef void (*swdg_forcing_fn)(void* user, double t, int64_t count, const double* x,
                                const double* y, double* fh, double* fhu, double* fhv);

typedef struct swdg_gpu swdg_gpu;

/* Context lifetime (TimeIntegrator ctor, timeloop.hpp:148-151: viscosity
 * needs degree >= 2).  `device` is the CUDA ordinal; *out is NULL on error
 * and swdg_gpu_create_error() holds the message. */
int swdg_gpu_create(const swdg_mesh_view* mesh, const swdg_params* params, int device,
                    swdg_gpu** out);
const char* swdg_gpu_create_error(void);
void swdg_gpu_destroy(swdg_gpu* ctx);
const char* swdg_gpu_last_error(const swdg_gpu* ctx);

/* Run every launch and copy of this context on `stream` (a cudaStream_t; NULL
 * is the legacy default stream).  A new context uses its own non-blocking
 * stream; callers that order the context against their own work (CUDA events,
 * NCCL, torch) pass their stream here. */
int swdg_gpu_set_stream(swdg_gpu* ctx, void* stream);
int swdg_gpu_synchronize(swdg_gpu* ctx);

/* State transfer: State h/hu/hv (field.hpp:12-34), K*n1*n1 each, host memory
 * (pinned memory gives full PCIe bandwidth). */
int swdg_gpu_upload_state(swdg_gpu* ctx, const double* h, const double* hu, const double* hv);
int swdg_gpu_download_state(swdg_gpu* ctx, double* h, double* hu, double* hv);
/* Device pointers of the current state (for device-resident callers). */
int swdg_gpu_device_state(swdg_gpu* ctx, double** h, double** hu, double** hv);

/* dW/dt of the current state at time t, downloaded to host buffers. */
int swdg_gpu_evaluate_rhs(swdg_gpu* ctx, double t, double* rh, double* rhu, double* rhv);
int swdg_gpu_assemble_rhs(swdg_gpu* ctx, double t, double* rh, double* rhu, double* rhv);

/* CFL time step of the current state (compute_dt): SWDG_ERR_INPUT unless
 * 0 < cfl <= 1. */
int swdg_gpu_compute_dt(swdg_gpu* ctx, double cfl, double* dt);

/* One SSPRK3 step of the current device state.  info->accepted = 0 leaves
 * the state untouched (reject signal, timeloop.hpp:205-209).  Returns
 * SWDG_ERR_ABORT when the limiter is disabled and a stage goes negative
 * (timeloop.hpp:211-218). */
int swdg_gpu_try_step(swdg_gpu* ctx, double t, double dt, swdg_step_info* info);

/* Device-resident throughput entry: `nsteps` SSPRK3 steps with fixed dt and
 * no host synchronisation (reject flags accumulate on the device; read them
 * with swdg_gpu_last_info). */
int swdg_gpu_run_steps(swdg_gpu* ctx, int nsteps, double t, double dt);
/* run_steps with options: SWDG_RUN_STEP_REDUCTIONS also queues, after every
 * step, the per-step reductions a driver needs (the StepDiagnostics sums and
 * minima and the next compute_dt candidate, driver.hpp:92, :117-127) on the
 * device -- the throughput metric "with dt and diagnostics amortised".  After a
 * rejected run (last_info accepted = 0) the device state is undefined. */
#define SWDG_RUN_STEP_REDUCTIONS 1
int swdg_gpu_run_steps_ex(swdg_gpu* ctx, int nsteps, double t, double dt, int flags);
int swdg_gpu_last_info(swdg_gpu* ctx, swdg_step_info* info);

int swdg_gpu_last_eps(swdg_gpu* ctx, double* eps);
int swdg_gpu_diagnostics(swdg_gpu* ctx, swdg_diagnostics* out);

/* TimeIntegrator::track_limiter_entropy (timeloop.hpp:199, post_stage :221-229):
 * when on, every stage that limits records the worst per-element
 * (e_after - e_before) / max(1, |e_before|) of limited_entropy_check
 * (limiter.hpp:88-101); worst_limiter_entropy_jump returns the maximum over the
 * context's life (starts at 0, timeloop.hpp:261).  Costs one dW/dt write and one
 * element pass per stage while on. */
int swdg_gpu_set_track_limiter_entropy(swdg_gpu* ctx, int on);
int swdg_gpu_worst_limiter_entropy_jump(swdg_gpu* ctx, double* jump);

/* The device-resident driver step (driver.hpp:91-127 without the host State):
 * try_step of the device state, then, if accepted, the StepDiagnostics fields
 * of the new state (total_mass, total_entropy, min_height, min_positivity_dt,
 * field.hpp:39-68, limiter.hpp:135-166) and the next step's compute_dt(cfl)
 * (timeloop.hpp:53-75).  Fast mode queues the reductions behind the three
 * stages and synchronises once. */
typedef struct swdg_step_report {
  swdg_step_info info;
  swdg_diagnostics diag; /* valid when info.accepted */
  double next_dt;        /* compute_dt(new state, cfl); valid when info.accepted */
} swdg_step_report;
int swdg_gpu_step_device(swdg_gpu* ctx, double t, double dt, double cfl, swdg_step_report* out);

/* Forcing: a host callback evaluated at the stage times t, t+dt, t+dt/2
 * (ssprk3_stage_times timeloop.hpp:82) and uploaded, or NULL to clear. */
int swdg_gpu_set_forcing(swdg_gpu* ctx, swdg_forcing_fn fn, void* user);

/* Number of kernels this context has launched (instrumentation). */
int64_t swdg_gpu_launch_count(const swdg_gpu* ctx);

/* ---- the paper's §5 kernel comparison (bench.hpp:133-157, 255-291) --------
 * One pass of the split-form volume kernel (kind 0: Dtilde flux differencing
 * with the entropy-conservative two-point flux, kernels::split_volume_element
 * dg_rhs.hpp:23-71) or the standard one (kind 1: pointwise contravariant
 * fluxes times D, standard_volume_element dg_rhs.hpp:75-117) over k elements of
 * DEVICE arrays in[7] = (h, hu, hv, y_eta, x_eta, y_xi, x_xi) with out[3] +=
 * the volume term, on `stream` (a cudaStream_t, NULL = legacy default).  The
 * harness kernels of the paper's table, not the stage path. */
int swdg_gpu_volume_kernel(int kind, int degree, int64_t k, const double* const* in,
                           double* const* out, double g, void* stream);

/* ---- standalone inputs (no reference headers needed) -------------------- */

/* make_operators (operators.hpp:148-188): LGL nodes/weights, D, Dtilde, Dhat,
 * V, V^-1 for degree N (bitwise the reference's). */
int swdg_operators(int degree, double* nodes, double* weights, double* deriv,
                   double* deriv_modified, double* deriv_weak, double* vandermonde,
                   double* vandermonde_inv);

/* structured_topology (mesh.hpp:237-290): face list of a kx*ky grid. */
int64_t swdg_structured_face_count(int kx, int ky, int periodic_x, int periodic_y);
int swdg_structured_faces(int kx, int ky, int periodic_x, int periodic_y, swdg_face* out);

#define SWDG_MESH_CARTESIAN 0  /* build_cartesian_mesh  mesh.hpp:342 */
#define SWDG_MESH_CURVED_DAM 1 /* build_curved_dam_mesh mesh.hpp:352 */
#define SWDG_MESH_WAVY 2       /* build_wavy_mesh       mesh.hpp:370 */

/* Generator spec of the reference's structured meshes plus a bathymetry:
 * bathy_kind 0 none, 1 constant p0, 2 linear p0 x + p1 y + p2, 3 paraboloid
 * p0 (x^2+y^2), 4 0.1 + 0.05 sin(2 pi x) sin(2 pi y) (validate.hpp:103),
 * 5 step x < p0 ? p1 : p2, 6 p0 + p1 sin(p2 x) sin(p2 y). */
typedef struct swdg_structured_spec {
  int32_t kind, degree, kx, ky;
  int32_t periodic_x, periodic_y;
  int32_t bathy_kind, reserved;
  double x0, x1, y0, y1;
  double extra; /* dam_fraction (curved dam) or amplitude (wavy) */
  double bathy[4];
} swdg_structured_spec;

/* Context whose mesh is generated on the device (the 1M-element throughput
 * meshes never touch host memory).  Geometry agrees with the host-built
 * reference mesh to rounding (device libm + FMA), not bitwise. */
int swdg_gpu_create_structured(const swdg_structured_spec* spec, const swdg_params* params,
                               int device, swdg_gpu** out);

/* One partition of a structured mesh generated on the device: local element i
 * is global element local_to_global[i]; [0, n_owned) are owned, the rest are
 * halo (ghost) copies; local_faces is the partition's face list in local ids
 * (paper_1804_02221_b200/partition.py build_plan). */
int swdg_gpu_create_structured_part(const swdg_structured_spec* spec, const swdg_params* params,
                                    int device, int32_t n_local, int32_t n_owned,
                                    const int32_t* local_to_global, int32_t n_faces,
                                    const swdg_face* local_faces, swdg_gpu** out);

/* Copy a device geometry array ("y_eta", "jac", "b", "face_nx", "x", ...) to host. */
int swdg_gpu_download_geometry(swdg_gpu* ctx, const char* name, double* out);

/* ---- partitioned (multi-GPU) runs ----------------------------------------
 * The reference has no decomposition; a partition is a mesh view whose
 * elements [n_owned, n_elem) are ghost copies of off-rank neighbours
 * (paper_1804_02221_b200/partition.py builds them).  Between stages the caller
 * moves face-node data between ranks (NCCL): pack -> send/recv -> unpack.
 *
 * halo_setup: local node ids to send (owner side) and to fill (ghost side),
 * concatenated over peers in the partition plan's order.
 * halo_pack/unpack: what 0 = stage k's input state (3 doubles per node,
 * node-major), what 1 = the viscous flux pairs (4 doubles per node); buffers
 * are device memory owned by the caller.
 * The split step: step_begin; for k in 0..2 { [exchange state]; stage_visc;
 * [exchange flux pairs]; stage_run }; step_flags (local reject/abort, sync);
 * the caller reduces them over ranks; step_commit(accept). */
int swdg_gpu_halo_setup(swdg_gpu* ctx, int64_t n_send, const int32_t* send_idx, int64_t n_recv,
                        const int32_t* recv_idx);
int swdg_gpu_halo_pack(swdg_gpu* ctx, int what, int stage, double* send_buf);
int swdg_gpu_halo_unpack(swdg_gpu* ctx, int what, int stage, const double* recv_buf);
/* Direct peer-memory halo exchange (no NCCL): every rank owns a mailbox in
 * device memory exported through CUDA IPC (ipc_alloc: zeroed, 64-byte
 * cudaIpcMemHandle_t out) and maps its peers' (ipc_open; NVLink / NVSwitch
 * between GPUs, plain device memory between processes sharing one GPU).
 * halo_push packs send entries [first, first+count) of `what` (as halo_pack)
 * straight into `dst` (a peer's mailbox slot) and then stores the sequence
 * number to `flag` (the peer's flag for this rank) with a system-scope release.
 * halo_wait queues a device-side wait until each of the n flags (this rank's
 * mailbox) reaches the sequence number -- no host synchronisation; after
 * timeout_s it gives up and halo_status reports it (synchronises the stream;
 * clears the report).  The sequence number is `seq`, or `*seq_base + seq` with a
 * device-resident base (seq_base non-NULL): a captured CUDA graph then carries
 * offsets and seq_advance (queued at the end of each replay) moves the base. */
int swdg_gpu_ipc_alloc(swdg_gpu* ctx, int64_t bytes, void** dptr, void* handle);
int swdg_gpu_ipc_open(swdg_gpu* ctx, const void* handle, void** dptr);
int swdg_gpu_halo_push(swdg_gpu* ctx, int what, int stage, int64_t first, int64_t count,
                       double* dst, uint64_t* flag, const uint64_t* seq_base, uint64_t seq);
int swdg_gpu_halo_wait(swdg_gpu* ctx, const uint64_t* flags, int32_t n, const uint64_t* seq_base,
                       uint64_t seq, double timeout_s);
int swdg_gpu_seq_advance(swdg_gpu* ctx, uint64_t* seq_base, uint64_t by);
int swdg_gpu_halo_status(swdg_gpu* ctx, int32_t* timed_out);
int swdg_gpu_dt_candidates(swdg_gpu* ctx, double* dt_min, double* min_len);
int swdg_gpu_step_begin(swdg_gpu* ctx);
int swdg_gpu_stage_visc(swdg_gpu* ctx, int stage, double t, double dt);
int swdg_gpu_stage_run(swdg_gpu* ctx, int stage, double t, double dt);
int swdg_gpu_step_flags(swdg_gpu* ctx, int32_t* reject, int32_t* abort);
int swdg_gpu_step_commit(swdg_gpu* ctx, int accept, swdg_step_info* info);

/* Asynchronous snapshot (driver.hpp:129-135 with the state on the device): copy
 * the current device state into caller-owned host buffers on a copy stream
 * (pinned buffers make it truly asynchronous), overlapping the following steps;
 * the context fences the buffer before it is overwritten.  snapshot_wait blocks
 * until the last copy has landed in host memory. */
int swdg_gpu_snapshot_async(swdg_gpu* ctx, double* h, double* hu, double* hv);
int swdg_gpu_snapshot_wait(swdg_gpu* ctx);
/* Page-locked host memory for snapshot buffers (NULL on failure). */
void* swdg_gpu_alloc_pinned(size_t bytes);
void swdg_gpu_free_pinned(void* p);

/* Stage buffers of the split step: stage k reads W (k = 0), A (k = 1) or B
 * (k = 2) and writes A (k = 0, 2) or B (k = 1), W^n staying in W.  With
 * upload_state (W^n) and upload_stage_input a single stage can be run from any
 * input (step_begin; stage_visc; stage_run) and its kernel-written output --
 * update, SSPRK3 combine, limiter, dry-node cut -- downloaded; stage_info is
 * that stage's report (n_limited, min h after limiting, max eps, accepted = no
 * negative element mean). */
int swdg_gpu_upload_stage_input(swdg_gpu* ctx, int stage, const double* h, const double* hu,
                                const double* hv);
int swdg_gpu_download_stage_output(swdg_gpu* ctx, int stage, double* h, double* hu, double* hv);
int swdg_gpu_stage_info(swdg_gpu* ctx, int stage, swdg_step_info* info);

/* Overlap of the halo exchange with interior work.  set_interior names an
 * owned element range [lo, hi) none of whose faces touches a ghost element
 * (lo is rounded up and hi down to even indices); stage_run_part then runs
 * part 1 = that range, which needs no halo data and may run while the state
 * exchange is in flight, and part 2 = the rest of the owned elements, after the
 * unpack (part 0 = all, like stage_run).  Exact mode runs everything in part 2. */
int swdg_gpu_set_interior(swdg_gpu* ctx, int32_t lo, int32_t hi);
int swdg_gpu_stage_run_part(swdg_gpu* ctx, int stage, double t, double dt, int part);
/* The viscous pre-pass of a stage in the same two parts: part 1 (the interior:
 * its BR1 face corrections need no ghost state) while the state exchange is in
 * flight, part 2 after the unpack; then the flux-pair exchange overlaps the
 * interior stage (stage_run_part 1).  Exact mode runs it whole in part 2. */
int swdg_gpu_stage_visc_part(swdg_gpu* ctx, int stage, double t, double dt, int part);

#ifdef __cplusplus
}
#endif

#endif /* SWDG_GPU_H */
