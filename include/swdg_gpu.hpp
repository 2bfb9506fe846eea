// swdg_gpu.hpp — header-only C++ mirror of the reference's TimeIntegrator
// (proj/include/swdg/timeloop.hpp:146-262) backed by the sm_100a C ABI in
// swdg_gpu.h.  Include it next to the reference headers; it borrows the
// reference's Mesh/State/RunConfig types unchanged, so a caller switches with
//
//     swdg::TimeIntegrator      integ(mesh, cfg);   // CPU reference
//     swdg::gpu::TimeIntegrator integ(mesh, cfg);   // B200
//
// Same member functions, same return values, same exceptions (SwdgError for
// bad input, NumericalAbort when the limiter is off and a stage goes
// negative), including the public `forcing` and `track_limiter_entropy` members
// and worst_limiter_entropy_jump().  Link with paper_1804_02221_b200/_lib/libswdg_gpu.so.
#pragma once

#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "swdg/timeloop.hpp"  // reference: Mesh, State, RunConfig, NumericalAbort
#include "swdg_gpu.h"

namespace swdg {
namespace gpu {

class TimeIntegrator {
 public:
  // `exact` selects SWDG_MODE_EXACT (bitwise parity with the reference build);
  // otherwise the fused fast kernels (1e-12 per stage).
  TimeIntegrator(const Mesh& mesh, const RunConfig& cfg, bool exact = true, int device = 0)
      : mesh_(mesh), cfg_(cfg) {
    faces_.reserve(mesh.topo.faces.size());
    for (const FaceInfo& f : mesh.topo.faces)
      faces_.push_back(swdg_face{f.elem_minus, f.face_minus, f.elem_plus, f.face_plus,
                                 f.reversed ? 1 : 0,
                                 f.tag == BoundaryTag::wall ? SWDG_TAG_WALL : SWDG_TAG_INTERIOR});
    const MeshGeometry& g = mesh.geom;
    swdg_mesh_view v{};
    v.n_elem = mesh.n_elements();
    v.degree = mesh.ops.degree;
    v.n_owned = 0;
    v.n_faces = static_cast<int32_t>(faces_.size());
    v.faces = faces_.data();
    v.weights = mesh.ops.weights.data();
    v.deriv = mesh.ops.deriv.data();
    v.deriv_modified = mesh.ops.deriv_modified.data();
    v.deriv_weak = mesh.ops.deriv_weak.data();
    v.vandermonde_inv = mesh.ops.vandermonde_inv.data();
    v.x = g.x.data();
    v.y = g.y.data();
    v.x_xi = g.x_xi.data();
    v.x_eta = g.x_eta.data();
    v.y_xi = g.y_xi.data();
    v.y_eta = g.y_eta.data();
    v.jac = g.jac.data();
    v.b = g.b.data();
    v.face_jsurf = g.face_jsurf.data();
    v.face_nx = g.face_nx.data();
    v.face_ny = g.face_ny.data();
    v.face_a = g.face_a.data();
    swdg_params p{};
    p.g = cfg.phys.g;
    p.h_tol = cfg.phys.h_tol;
    p.h_des = cfg.phys.h_des;
    p.h_ref = cfg.phys.h_ref;
    p.epsilon0 = cfg.visc.epsilon0;
    p.sigma_min = cfg.visc.sigma_min;
    p.sigma_max = cfg.visc.sigma_max;
    p.visc_enabled = cfg.visc.enabled ? 1 : 0;
    p.limiter_enabled = cfg.limiter_enabled ? 1 : 0;
    p.mode = exact ? SWDG_MODE_EXACT : SWDG_MODE_FAST;
    p.scheme = cfg.mode == SchemeMode::standard ? SWDG_SCHEME_STANDARD : SWDG_SCHEME_ES;
    const int rc = swdg_gpu_create(&v, &p, device, &ctx_);
    if (rc != SWDG_OK) raise(rc, swdg_gpu_create_error());
  }
  ~TimeIntegrator() { swdg_gpu_destroy(ctx_); }
  TimeIntegrator(const TimeIntegrator&) = delete;
  TimeIntegrator& operator=(const TimeIntegrator&) = delete;

  // timeloop.hpp:156-170
  bool try_step(State& w, double t, double dt) {
    sync_forcing();
    sync_tracking();
    check(swdg_gpu_upload_state(ctx_, w.h.data(), w.hu.data(), w.hv.data()));
    check(swdg_gpu_try_step(ctx_, t, dt, &info_));
    evaluated();
    if (info_.accepted) check(swdg_gpu_download_state(ctx_, w.h.data(), w.hu.data(), w.hv.data()));
    return info_.accepted != 0;
  }

  // timeloop.hpp:173-190
  void evaluate_rhs(const State& s, double t, Residual& out) {
    sync_forcing();
    out.resize(s.n_elem, s.n1);
    check(swdg_gpu_upload_state(ctx_, s.h.data(), s.hu.data(), s.hv.data()));
    check(swdg_gpu_evaluate_rhs(ctx_, t, out.h.data(), out.hu.data(), out.hv.data()));
    evaluated();
  }

  // timeloop.hpp:192 (const like the reference).  Like the reference's eps_, it
  // is empty until a viscous evaluation has run (compute_viscosity fills it,
  // timeloop.hpp:179) and is read back once per evaluation into a cache.
  const std::vector<double>& last_eps() const {
    if (eps_stale_) {
      eps_.resize(mesh_.n_elements());
      check(swdg_gpu_last_eps(ctx_, eps_.data()));
      eps_stale_ = false;
    }
    return eps_;
  }
  int last_limited_count() const { return info_.n_limited; }
  double last_max_eps() const { return info_.max_eps; }
  double last_min_stage_h() const { return info_.min_stage_h; }
  double worst_limiter_entropy_jump() const {
    double v = 0.0;
    check(swdg_gpu_worst_limiter_entropy_jump(ctx_, &v));
    return v;
  }

  ForcingFn forcing;                   // dg_rhs.hpp:255, evaluated on the host per stage
  bool track_limiter_entropy = false;  // timeloop.hpp:199 (limited_entropy_check on the device)

  // ---- device-resident surface (no reference counterpart): the state stays on
  // the device between steps; see swdg_gpu_driver.hpp
  void upload(const State& w) {
    check(swdg_gpu_upload_state(ctx_, w.h.data(), w.hu.data(), w.hv.data()));
  }
  void download(State& w) const {
    w.resize(mesh_.n_elements(), mesh_.n1());
    check(swdg_gpu_download_state(ctx_, w.h.data(), w.hu.data(), w.hv.data()));
  }
  double compute_dt_device(double cfl) {
    double dt = 0.0;
    check(swdg_gpu_compute_dt(ctx_, cfl, &dt));
    return dt;
  }
  swdg_diagnostics diagnostics_device() {
    swdg_diagnostics d{};
    check(swdg_gpu_diagnostics(ctx_, &d));
    return d;
  }
  // try_step of the device state + the new state's diagnostics and next CFL dt
  swdg_step_report step_device(double t, double dt, double cfl) {
    sync_forcing();
    sync_tracking();
    swdg_step_report r{};
    check(swdg_gpu_step_device(ctx_, t, dt, cfl, &r));
    evaluated();
    info_ = r.info;
    return r;
  }
  void snapshot_async(double* h, double* hu, double* hv) {
    check(swdg_gpu_snapshot_async(ctx_, h, hu, hv));
  }
  void snapshot_wait() { check(swdg_gpu_snapshot_wait(ctx_)); }
  const Mesh& mesh() const { return mesh_; }

 private:
  static void forcing_tramp(void* user, double t, int64_t count, const double* x,
                            const double* y, double* fh, double* fhu, double* fhv) {
    auto* self = static_cast<TimeIntegrator*>(user);
    for (int64_t n = 0; n < count; ++n) {
      const Vec3 f = self->forcing(x[n], y[n], t);
      fh[n] = f.h;
      fhu[n] = f.hu;
      fhv[n] = f.hv;
    }
  }
  // a viscous evaluation refreshed eps on the device (only the ES scheme with
  // viscosity computes it, timeloop.hpp:178)
  void evaluated() {
    if (cfg_.visc.enabled && cfg_.mode == SchemeMode::es) eps_stale_ = true;
  }
  void sync_tracking() {
    if (track_limiter_entropy != tracking_set_) {
      check(swdg_gpu_set_track_limiter_entropy(ctx_, track_limiter_entropy ? 1 : 0));
      tracking_set_ = track_limiter_entropy;
    }
  }
  void sync_forcing() {
    const bool want = static_cast<bool>(forcing);
    if (want != forcing_set_) {
      check(swdg_gpu_set_forcing(ctx_, want ? &forcing_tramp : nullptr, this));
      forcing_set_ = want;
    }
  }
  [[noreturn]] static void raise(int rc, const char* msg) {
    if (rc == SWDG_ERR_ABORT) throw NumericalAbort(msg);
    if (rc == SWDG_ERR_INPUT) throw SwdgError(msg);
    throw std::runtime_error(std::string("swdg_gpu: ") + msg);
  }
  void check(int rc) const {
    if (rc != SWDG_OK) raise(rc, swdg_gpu_last_error(ctx_));
  }

  const Mesh& mesh_;
  RunConfig cfg_;
  std::vector<swdg_face> faces_;
  swdg_gpu* ctx_ = nullptr;
  swdg_step_info info_{};
  mutable std::vector<double> eps_;
  mutable bool eps_stale_ = false;
  bool forcing_set_ = false;
  bool tracking_set_ = false;
};

}  // namespace gpu
}  // namespace swdg
