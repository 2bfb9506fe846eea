// swdg_gpu_driver.hpp — run_simulation (proj/include/swdg/driver.hpp:62-142)
// with the state resident on the B200.  Header-only, next to the reference
// headers: it uses the reference's own scenario catalogue, mesh builders,
// config hash and io writers (scenarios.hpp, config.hpp, io.hpp), so the files
// it writes have the reference's formats (io.hpp:54-74 snapshots, :234-256
// diagnostics, tagged with config_hash config.hpp:216-226).
//
//   swdg::RunResult r = swdg::gpu::run_simulation(cfg, opt);
//
// Differences from driver.hpp, all on the data path only:
//   * the state is uploaded once; each step is one swdg_gpu_step_device call
//     (three stages + the StepDiagnostics reductions + the next compute_dt of
//     the new state, one host synchronisation);
//   * reject-and-halve rolls back on the device (W^n stays until acceptance);
//   * snapshots are asynchronous: the D2H copy runs on a copy stream behind the
//     step that produced the state, the file is written on a host thread while
//     the following steps run;
//   * the host State is materialised only for on_step, snapshots, the abort dump
//     and the final result.
// With opt.exact (the default) the arithmetic is the parity mode: the
// trajectory, the step diagnostics (serial-order sums) and hence every file are
// bitwise the reference's.  opt.exact = false runs the fused fast kernels.
#pragma once

#include <future>
#include <memory>
#include <string>
#include <vector>

#include "swdg/driver.hpp"  // reference: RunConfig, RunResult, StepDiagnostics, io, scenarios
#include "swdg_gpu.hpp"

namespace swdg {
namespace gpu {

// RunOptions (driver.hpp:16-22) with on_step typed on the GPU integrator
struct RunOptions {
  bool write_files = false;
  bool keep_series = true;
  bool track_limiter_entropy = false;
  ForcingFn forcing;
  std::function<void(const StepDiagnostics&, const State&, const gpu::TimeIntegrator&)> on_step;
  bool exact = true;  // SWDG_MODE_EXACT (bitwise) or the fused fast kernels
  int device = 0;
};

namespace detail {

struct PinnedState {
  size_t n = 0;
  double* p = nullptr;
  explicit PinnedState(size_t nodes) : n(nodes) {
    p = static_cast<double*>(swdg_gpu_alloc_pinned(3 * nodes * sizeof(double)));
    if (!p) throw std::runtime_error("swdg_gpu: pinned snapshot buffer allocation failed");
  }
  ~PinnedState() { swdg_gpu_free_pinned(p); }
  PinnedState(const PinnedState&) = delete;
  PinnedState& operator=(const PinnedState&) = delete;
  double* h() { return p; }
  double* hu() { return p + n; }
  double* hv() { return p + 2 * n; }
  State to_state(int n_elem, int n1) const {
    State s;
    s.resize(n_elem, n1);
    std::copy(p, p + n, s.h.begin());
    std::copy(p + n, p + 2 * n, s.hu.begin());
    std::copy(p + 2 * n, p + 3 * n, s.hv.begin());
    return s;
  }
};

}  // namespace detail

inline RunResult run_simulation(const RunConfig& cfg, const RunOptions& opt = {}) {
  const Scenario sc = make_scenario(cfg.scenario);
  Mesh mesh = build_mesh(cfg);
  RunResult out;
  out.state = initial_state(sc, mesh);
  const std::string hash = config_hash(cfg);

  io::DiagnosticsWriter diag;
  if (opt.write_files) {
    diag.open(cfg.out_dir + "/diagnostics.txt", hash);
    if (cfg.dump_mesh) io::dump_mesh(cfg.out_dir + "/mesh.txt", mesh, hash);
  }

  TimeIntegrator integ(mesh, cfg, opt.exact, opt.device);
  integ.forcing = opt.forcing;
  integ.track_limiter_entropy = opt.track_limiter_entropy;

  out.mass_initial = total_mass(out.state, mesh);
  out.entropy_initial = total_entropy(out.state, mesh, cfg.phys);

  std::vector<double> snaps = driver_detail::snapshot_schedule(cfg, sc);
  size_t next_snap = 0;
  const bool any_snap = cfg.snapshot_dt > 0.0 || !sc.snapshot_times.empty();
  if (opt.write_files && any_snap)
    io::write_snapshot(cfg.out_dir + "/snapshot_t" + driver_detail::time_label(0.0) + ".txt",
                       out.state, mesh, 0.0, integ.last_eps(), hash);

  integ.upload(out.state);
  const size_t nn = out.state.h.size();
  std::unique_ptr<detail::PinnedState> snap_buf;
  std::future<void> writer;  // the previous snapshot's file write
  auto flush_writer = [&] {
    if (writer.valid()) writer.get();
  };

  const double t_end = cfg.final_time;
  double t = 0.0;
  const double t_eps = 1e-12 * std::max(1.0, t_end);
  bool have_dt = false;
  double next_dt = 0.0;
  State host;  // materialised on demand
  while (t < t_end - t_eps) {
    double dt = have_dt ? next_dt : integ.compute_dt_device(cfg.cfl);
    double t_event = t_end;
    if (next_snap < snaps.size()) t_event = std::min(t_event, snaps[next_snap]);
    bool hit_event = false;
    if (t + dt >= t_event - t_eps) {
      dt = t_event - t;
      hit_event = true;
    }

    int rejections = 0;
    swdg_step_report rep{};
    while (true) {
      rep = integ.step_device(t, dt, cfg.cfl);
      if (rep.info.accepted) break;
      dt *= 0.5;
      hit_event = false;
      if (++rejections >= 10) {
        if (opt.write_files) {
          flush_writer();
          integ.download(host);
          io::write_snapshot(cfg.out_dir + "/state_dump.txt", host, mesh, t, integ.last_eps(),
                             hash);
        }
        throw NumericalAbort("step rejected 10 times at t=" + std::to_string(t));
      }
    }
    next_dt = rep.next_dt;
    have_dt = true;
    t = hit_event ? t_event : t + dt;
    ++out.steps;

    StepDiagnostics d;
    d.step = out.steps;
    d.t = t;
    d.dt = dt;
    d.mass = rep.diag.mass;
    d.entropy = rep.diag.entropy;
    d.min_h = rep.diag.min_h;
    d.n_limited = integ.last_limited_count();
    d.max_eps = integ.last_max_eps();
    d.min_stage_h = integ.last_min_stage_h();
    d.positivity_dt = rep.diag.positivity_dt;
    diag.append(d);
    if (opt.keep_series) out.series.push_back(d);
    if (opt.on_step) {
      integ.download(host);
      opt.on_step(d, host, integ);
    }

    while (next_snap < snaps.size() && t >= snaps[next_snap] - t_eps) {
      if (opt.write_files) {
        // one snapshot in flight: the previous file is complete before its
        // buffer is reused; this copy overlaps the next steps
        flush_writer();
        if (!snap_buf) snap_buf = std::make_unique<detail::PinnedState>(nn);
        integ.snapshot_async(snap_buf->h(), snap_buf->hu(), snap_buf->hv());
        const std::string path = cfg.out_dir + "/snapshot_t" +
                                 driver_detail::time_label(snaps[next_snap]) + ".txt";
        std::vector<double> eps = integ.last_eps();
        detail::PinnedState* buf = snap_buf.get();
        TimeIntegrator* ip = &integ;
        const int ne = mesh.n_elements(), n1 = mesh.n1();
        const double tw = t;
        writer = std::async(std::launch::async, [=, &mesh] {
          ip->snapshot_wait();
          io::write_snapshot(path, buf->to_state(ne, n1), mesh, tw, eps, hash);
        });
      }
      ++next_snap;
    }
  }
  flush_writer();
  integ.download(out.state);
  out.t = t;
  out.worst_limiter_entropy_jump = integ.worst_limiter_entropy_jump();
  return out;
}

}  // namespace gpu
}  // namespace swdg
