// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (parity checker, never the product).
//
// A C ABI over the UNMODIFIED reference headers (/root/reference/proj/include/swdg),
// compiled with the reference's own flags (proj/CMakeLists.txt:6-8: Release =
// -O3 -DNDEBUG, no -march; we add -ffp-contract=off to pin the no-FMA build,
// SURVEY fact 4).  Built by oracle/Makefile into oracle/_ref/libswdg_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load it.  Nothing here is copied from the reference: every call
// below forwards to the reference's own functions.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "swdg/bench.hpp"
#include "swdg/driver.hpp"
#include "swdg/validate.hpp"
#include "../include/swdg_gpu.h"

using namespace swdg;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const NumericalAbort*>(&e)) return SWDG_ERR_ABORT;
  if (dynamic_cast<const SwdgError*>(&e)) return SWDG_ERR_INPUT;
  return SWDG_ERR_CUDA;  // "other"
}

struct RefMesh {
  Mesh mesh;
};

RunConfig make_cfg(const Mesh& m, const swdg_params* p) {
  RunConfig c;
  c.degree = m.ops.degree;
  c.phys.g = p->g;
  c.phys.h_tol = p->h_tol;
  c.phys.h_des = p->h_des;
  c.phys.h_ref = p->h_ref;
  c.visc.enabled = p->visc_enabled != 0;
  c.visc.epsilon0 = p->epsilon0;
  c.visc.sigma_min = p->sigma_min;
  c.visc.sigma_max = p->sigma_max;
  c.limiter_enabled = p->limiter_enabled != 0;
  c.mode = p->scheme == 1 ? SchemeMode::standard : SchemeMode::es;
  return c;
}

State to_state(const Mesh& m, const double* h, const double* hu, const double* hv) {
  State s;
  s.resize(m.n_elements(), m.n1());
  std::memcpy(s.h.data(), h, sizeof(double) * s.size());
  std::memcpy(s.hu.data(), hu, sizeof(double) * s.size());
  std::memcpy(s.hv.data(), hv, sizeof(double) * s.size());
  return s;
}

void from_state(const State& s, double* h, double* hu, double* hv) {
  std::memcpy(h, s.h.data(), sizeof(double) * s.size());
  std::memcpy(hu, s.hu.data(), sizeof(double) * s.size());
  std::memcpy(hv, s.hv.data(), sizeof(double) * s.size());
}

// Traveling-wave manufactured forcing of validate.hpp:543-556 (crit_convergence).
ForcingFn wave_forcing(const double* f) {
  const double h0 = f[0], amp = f[1], u0 = f[2], v0 = f[3], k = f[4], g = f[5];
  const double omega = k * (u0 + v0);
  return [=](double x, double y, double t) {
    const double hx = amp * k * std::cos(k * (x + y) - omega * t);
    const double h = h0 + amp * std::sin(k * (x + y) - omega * t);
    return Vec3{0.0, g * h * hx, g * h * hx};
  };
}

struct RefInteg {
  const Mesh* mesh;
  RunConfig cfg;
  TimeIntegrator integ;
  RefInteg(const Mesh* m, const RunConfig& c) : mesh(m), cfg(c), integ(*m, c) {}
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_operators(int degree, double* nodes, double* weights, double* d, double* dt, double* dh,
                  double* v, double* vinv) {
  try {
    const Operators1D ops = make_operators(degree);
    const size_t n1 = ops.n1(), m = n1 * n1;
    std::memcpy(nodes, ops.nodes.data(), n1 * sizeof(double));
    std::memcpy(weights, ops.weights.data(), n1 * sizeof(double));
    std::memcpy(d, ops.deriv.data(), m * sizeof(double));
    std::memcpy(dt, ops.deriv_modified.data(), m * sizeof(double));
    std::memcpy(dh, ops.deriv_weak.data(), m * sizeof(double));
    std::memcpy(v, ops.vandermonde.data(), m * sizeof(double));
    std::memcpy(vinv, ops.vandermonde_inv.data(), m * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// kind: 0 cartesian (mesh.hpp:342), 1 curved dam (mesh.hpp:352, extra=dam_fraction),
// 2 wavy (mesh.hpp:370, extra=amp).
void* ref_mesh_build(int kind, int degree, int kx, int ky, double x0, double x1, double y0,
                     double y1, int px, int py, double extra) {
  try {
    auto* r = new RefMesh;
    if (kind == 0)
      r->mesh = build_cartesian_mesh(degree, kx, ky, x0, x1, y0, y1, px != 0, py != 0);
    else if (kind == 1)
      r->mesh = build_curved_dam_mesh(degree, kx, ky, x0, x1, y0, y1, extra);
    else
      r->mesh = build_wavy_mesh(degree, kx, ky, x0, x1, y0, y1, extra, px != 0, py != 0);
    sample_bathymetry(r->mesh, nullptr);
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Bathymetry closures sampled with the reference's sample_bathymetry (mesh.hpp:223).
// 0 none; 1 constant p0; 2 linear p0*x+p1*y+p2; 3 paraboloid p0*(x^2+y^2);
// 4 validate smooth 0.1+0.05 sin2pix sin2piy (validate.hpp:103); 5 step x<p0 ? p1 : p2;
// 6 sine bump p0 + p1*sin(p2*x)*sin(p2*y).
void ref_mesh_bathymetry(void* mh, int kind, const double* p) {
  Mesh& m = static_cast<RefMesh*>(mh)->mesh;
  const double p0 = p ? p[0] : 0, p1 = p ? p[1] : 0, p2 = p ? p[2] : 0;
  std::function<double(double, double)> f;
  switch (kind) {
    case 1: f = [=](double, double) { return p0; }; break;
    case 2: f = [=](double x, double y) { return p0 * x + p1 * y + p2; }; break;
    case 3: f = [=](double x, double y) { return p0 * (x * x + y * y); }; break;
    case 4: f = validate::detail::smooth_bathymetry; break;
    case 5: f = [=](double x, double) { return x < p0 ? p1 : p2; }; break;
    case 6: f = [=](double x, double y) { return p0 + p1 * std::sin(p2 * x) * std::sin(p2 * y); }; break;
    default: break;
  }
  sample_bathymetry(m, f);
}

// Scenario mesh (scenarios.hpp:189) with kx/ky/degree overrides (<=0 keeps default).
void* ref_scenario_mesh(const char* id, int kx, int ky, int degree) {
  try {
    Scenario sc = make_scenario(id);
    RunConfig c = sc.config;
    if (kx > 0) c.kx = kx;
    if (ky > 0) c.ky = ky;
    if (degree > 0) c.degree = degree;
    auto* r = new RefMesh;
    r->mesh = build_mesh(c);
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// initial_state (scenarios.hpp:205): samples the scenario bathymetry into the mesh.
int ref_scenario_initial(const char* id, void* mh, double* h, double* hu, double* hv) {
  try {
    Scenario sc = make_scenario(id);
    const State s = initial_state(sc, static_cast<RefMesh*>(mh)->mesh);
    from_state(s, h, hu, hv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Scenario defaults needed to configure a run: g, h_tol, h_des, h_ref, eps0, smin, smax,
// visc_enabled, limiter_enabled, cfl, final_time, degree.
int ref_scenario_config(const char* id, int degree, double* out) {
  try {
    Scenario sc = make_scenario(id);
    RunConfig c = sc.config;
    if (degree > 0 && degree != c.degree) {
      c.degree = degree;
    }
    out[0] = c.phys.g;
    out[1] = c.phys.h_tol;
    out[2] = c.phys.h_des;
    out[3] = c.phys.h_ref;
    out[4] = c.visc.epsilon0;
    out[5] = c.visc.sigma_min;
    out[6] = c.visc.sigma_max;
    out[7] = c.visc.enabled ? 1.0 : 0.0;
    out[8] = c.limiter_enabled ? 1.0 : 0.0;
    out[9] = c.cfl;
    out[10] = c.final_time;
    out[11] = sc.orbital_period;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_mesh_free(void* mh) { delete static_cast<RefMesh*>(mh); }
int ref_mesh_n_elem(void* mh) { return static_cast<RefMesh*>(mh)->mesh.n_elements(); }
int ref_mesh_degree(void* mh) { return static_cast<RefMesh*>(mh)->mesh.ops.degree; }
int ref_mesh_n_faces(void* mh) {
  return static_cast<int>(static_cast<RefMesh*>(mh)->mesh.topo.faces.size());
}

const double* ref_mesh_array(void* mh, const char* name) {
  Mesh& m = static_cast<RefMesh*>(mh)->mesh;
  const std::string n(name);
  MeshGeometry& g = m.geom;
  if (n == "x") return g.x.data();
  if (n == "y") return g.y.data();
  if (n == "x_xi") return g.x_xi.data();
  if (n == "x_eta") return g.x_eta.data();
  if (n == "y_xi") return g.y_xi.data();
  if (n == "y_eta") return g.y_eta.data();
  if (n == "jac") return g.jac.data();
  if (n == "b") return g.b.data();
  if (n == "b_yeta") return g.b_yeta.data();
  if (n == "b_yxi") return g.b_yxi.data();
  if (n == "b_xeta") return g.b_xeta.data();
  if (n == "b_xxi") return g.b_xxi.data();
  if (n == "face_jsurf") return g.face_jsurf.data();
  if (n == "face_nx") return g.face_nx.data();
  if (n == "face_ny") return g.face_ny.data();
  if (n == "face_a") return g.face_a.data();
  if (n == "nodes") return m.ops.nodes.data();
  if (n == "weights") return m.ops.weights.data();
  if (n == "deriv") return m.ops.deriv.data();
  if (n == "deriv_modified") return m.ops.deriv_modified.data();
  if (n == "deriv_weak") return m.ops.deriv_weak.data();
  if (n == "vandermonde") return m.ops.vandermonde.data();
  if (n == "vandermonde_inv") return m.ops.vandermonde_inv.data();
  return nullptr;
}

// Writes n_faces*6 int32 (elem_minus, face_minus, elem_plus, face_plus, reversed, tag)
// and n_faces*2 doubles (offset_x, offset_y).
void ref_mesh_faces(void* mh, int32_t* out, double* offsets) {
  const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
  for (size_t f = 0; f < m.topo.faces.size(); ++f) {
    const FaceInfo& fi = m.topo.faces[f];
    out[6 * f + 0] = fi.elem_minus;
    out[6 * f + 1] = fi.face_minus;
    out[6 * f + 2] = fi.elem_plus;
    out[6 * f + 3] = fi.face_plus;
    out[6 * f + 4] = fi.reversed ? 1 : 0;
    out[6 * f + 5] = fi.tag == BoundaryTag::wall ? SWDG_TAG_WALL : SWDG_TAG_INTERIOR;
    if (offsets) {
      offsets[2 * f] = fi.offset_x;
      offsets[2 * f + 1] = fi.offset_y;
    }
  }
}

double ref_watertightness_gap(void* mh) {
  return watertightness_gap(static_cast<RefMesh*>(mh)->mesh);
}

// assemble_rhs (dg_rhs.hpp:267), no viscous part; mode 0 = es, 1 = standard.
int ref_assemble_rhs(void* mh, const swdg_params* p, int mode, const double* h,
                     const double* hu, const double* hv, double t, double* rh, double* rhu,
                     double* rhv) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig c = make_cfg(m, p);
    const State s = to_state(m, h, hu, hv);
    RhsOptions opt;
    opt.mode = mode == 0 ? SchemeMode::es : SchemeMode::standard;
    opt.time = t;
    Residual res;
    assemble_rhs(s, m, c.phys, opt, res);
    from_state(res, rh, rhu, rhv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void* ref_integ_create(void* mh, const swdg_params* p, int forcing_kind, const double* fp) {
  try {
    const Mesh* m = &static_cast<RefMesh*>(mh)->mesh;
    auto* r = new RefInteg(m, make_cfg(*m, p));
    if (forcing_kind == 1) r->integ.forcing = wave_forcing(fp);
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_integ_free(void* ih) { delete static_cast<RefInteg*>(ih); }

int ref_integ_try_step(void* ih, double* h, double* hu, double* hv, double t, double dt,
                       swdg_step_info* info) {
  auto* r = static_cast<RefInteg*>(ih);
  try {
    State s = to_state(*r->mesh, h, hu, hv);
    const bool ok = r->integ.try_step(s, t, dt);
    if (ok) from_state(s, h, hu, hv);
    info->accepted = ok ? 1 : 0;
    info->n_limited = r->integ.last_limited_count();
    info->max_eps = r->integ.last_max_eps();
    info->min_stage_h = r->integ.last_min_stage_h();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Same as ref_integ_try_step on a persistent State (no per-call copies): used by
// the timing legs so the measured time is the reference's own try_step.
struct RefRunner {
  RefInteg* integ;
  State s;
};

void* ref_runner_create(void* ih, const double* h, const double* hu, const double* hv) {
  auto* r = static_cast<RefInteg*>(ih);
  return new RefRunner{r, to_state(*r->mesh, h, hu, hv)};
}
int ref_runner_steps(void* rh, int nsteps, double t, double dt) {
  auto* r = static_cast<RefRunner*>(rh);
  try {
    int accepted = 0;
    for (int k = 0; k < nsteps; ++k) accepted += r->integ->integ.try_step(r->s, t + k * dt, dt);
    return accepted;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}
void ref_runner_free(void* rh) { delete static_cast<RefRunner*>(rh); }

int ref_integ_evaluate_rhs(void* ih, const double* h, const double* hu, const double* hv,
                           double t, double* rh, double* rhu, double* rhv) {
  auto* r = static_cast<RefInteg*>(ih);
  try {
    const State s = to_state(*r->mesh, h, hu, hv);
    Residual res;
    r->integ.evaluate_rhs(s, t, res);
    from_state(res, rh, rhu, rhv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_integ_last_eps(void* ih, double* eps) {
  const auto& e = static_cast<RefInteg*>(ih)->integ.last_eps();
  std::memcpy(eps, e.data(), e.size() * sizeof(double));
}

int ref_compute_dt(void* mh, const swdg_params* p, const double* h, const double* hu,
                   const double* hv, double cfl, double* dt) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig c = make_cfg(m, p);
    *dt = compute_dt(to_state(m, h, hu, hv), m, c.phys, cfl);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_diagnostics(void* mh, const swdg_params* p, const double* h, const double* hu,
                    const double* hv, swdg_diagnostics* out) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig c = make_cfg(m, p);
    const State s = to_state(m, h, hu, hv);
    out->mass = total_mass(s, m);
    out->entropy = total_entropy(s, m, c.phys);
    out->min_h = min_height(s);
    out->positivity_dt = min_positivity_dt(s, m, c.phys);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Component entry points for fine-grained parity (viscosity.hpp, limiter.hpp).
int ref_compute_viscosity(void* mh, const swdg_params* p, const double* h, double* eps) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig c = make_cfg(m, p);
    State s;
    s.resize(m.n_elements(), m.n1());
    std::memcpy(s.h.data(), h, sizeof(double) * s.size());
    std::vector<double> e;
    compute_viscosity(s, m, c.visc, e);
    std::memcpy(eps, e.data(), e.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_shock_indicator(int degree, const double* field) {
  const Operators1D ops = make_operators(degree);
  std::vector<double> scratch;
  try {
    return shock_indicator(ops, field, scratch);
  } catch (const std::exception& e) {
    fail(e);
    return std::nan("");
  }
}

int ref_br1_gradients(void* mh, const double* u, const double* v, double* u1, double* u2,
                      double* v1, double* v2) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const size_t n = static_cast<size_t>(m.n_elements()) * m.np();
    std::vector<double> uu(u, u + n), vv(v, v + n);
    GradientField g;
    br1_gradients(uu, vv, m, g);
    std::memcpy(u1, g.u1.data(), n * sizeof(double));
    std::memcpy(u2, g.u2.data(), n * sizeof(double));
    std::memcpy(v1, g.v1.data(), n * sizeof(double));
    std::memcpy(v2, g.v2.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_viscous_lhs(void* mh, const double* h, const double* hu, const double* hv,
                    const double* u1, const double* u2, const double* v1, const double* v2,
                    const double* eps, double* out_hu, double* out_hv) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const size_t n = static_cast<size_t>(m.n_elements()) * m.np();
    const State s = to_state(m, h, hu, hv);
    GradientField g;
    g.u1.assign(u1, u1 + n);
    g.u2.assign(u2, u2 + n);
    g.v1.assign(v1, v1 + n);
    g.v2.assign(v2, v2 + n);
    std::vector<double> e(eps, eps + m.n_elements());
    Residual out;
    viscous_lhs(s, g, e, m, out);
    std::memcpy(out_hu, out.hu.data(), n * sizeof(double));
    std::memcpy(out_hv, out.hv.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// limit_element over all elements (limiter.hpp:43); writes theta per element.
int ref_limit_all(void* mh, const swdg_params* p, double* h, double* hu, double* hv,
                  int zero_dry, double* theta) {
  try {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig c = make_cfg(m, p);
    State s = to_state(m, h, hu, hv);
    for (int e = 0; e < m.n_elements(); ++e)
      theta[e] = limit_element(s, m, e, c.phys, zero_dry != 0).theta;
    from_state(s, h, hu, hv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_simulation (driver.hpp:62) on a scenario with mesh/time overrides; writes the
// final state (caller sizes it from ref_scenario_mesh) and the step count.
int ref_run_simulation(const char* id, int kx, int ky, int degree, double final_time,
                       double cfl, double* h, double* hu, double* hv, int64_t* steps,
                       double* t_out) {
  try {
    Scenario sc = make_scenario(id);
    RunConfig c = sc.config;
    if (kx > 0) c.kx = kx;
    if (ky > 0) c.ky = ky;
    if (degree > 0) c.degree = degree;
    if (final_time > 0) c.final_time = final_time;
    if (cfl > 0) c.cfl = cfl;
    RunOptions opt;
    opt.keep_series = false;
    const RunResult r = run_simulation(c, opt);
    from_state(r.state, h, hu, hv);
    *steps = r.steps;
    *t_out = r.t;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// crit_convergence's run (validate.hpp:560-595) on the mesh `mh`: the traveling
// wave h0 + amp sin(k(x+y) - omega t), (u0, v0) as the initial state, the
// reference TimeIntegrator with the manufactured forcing, CFL steps
// min(compute_dt, t_end - t) to t_end, then the J-weighted L2 error of h.
int ref_mms_error(void* mh, const swdg_params* p, double cfl, double t_end, const double* fp,
                  double* err, int64_t* steps) {
  try {
    const Mesh& mesh = static_cast<RefMesh*>(mh)->mesh;
    const RunConfig cfg = make_cfg(mesh, p);
    const double h0 = fp[0], amp = fp[1], u0 = fp[2], v0 = fp[3], k = fp[4];
    const double omega = k * (u0 + v0);
    auto h_exact = [&](double x, double y, double t) {
      return h0 + amp * std::sin(k * (x + y) - omega * t);
    };
    State s;
    s.resize(mesh.n_elements(), mesh.n1());
    for (int n = 0; n < s.size(); ++n) {
      const double h = h_exact(mesh.geom.x[n], mesh.geom.y[n], 0.0);
      s.set(n, {h, h * u0, h * v0});
    }
    TimeIntegrator integ(mesh, cfg);
    integ.forcing = wave_forcing(fp);
    double t = 0.0;
    int64_t n_steps = 0;
    while (t < t_end - 1e-13) {
      double dt = std::min(compute_dt(s, mesh, cfg.phys, cfl), t_end - t);
      if (!integ.try_step(s, t, dt)) throw SwdgError("convergence run: step rejected");
      t += dt;
      ++n_steps;
    }
    double err2 = 0.0;
    const int n1 = mesh.n1();
    for (int e = 0; e < mesh.n_elements(); ++e)
      for (int i = 0; i < n1; ++i)
        for (int j = 0; j < n1; ++j) {
          const int n = mesh.geom.node(e, i, j);
          const double d = s.h[n] - h_exact(mesh.geom.x[n], mesh.geom.y[n], t);
          err2 += d * d * mesh.geom.jac[n] * mesh.ops.weights[i] * mesh.ops.weights[j];
        }
    *err = std::sqrt(err2);
    *steps = n_steps;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's volume kernels of the paper's comparison (bench.hpp:133-157)
// over k elements of host arrays: kind 0 split_volume_element with Dtilde,
// kind 1 standard_volume_element with D (dg_rhs.hpp:23-117); out += the term.
int ref_volume_kernel(int kind, int degree, long k, const double* const* in, double* const* out,
                      double g) {
  try {
    const Operators1D ops = make_operators(degree);
    const int n1 = degree + 1, np = n1 * n1;
    std::vector<double> scratch(6 * np);
    for (long e = 0; e < k; ++e) {
      const long o = e * np;
      if (kind == 0)
        kernels::split_volume_element<double>(
            n1, g, 1e-8, in[0] + o, in[1] + o, in[2] + o, in[3] + o, in[4] + o, in[5] + o,
            in[6] + o, ops.deriv_modified.data(), scratch.data(), scratch.data() + np,
            out[0] + o, out[1] + o, out[2] + o);
      else
        kernels::standard_volume_element<double>(
            n1, g, 1e-8, in[0] + o, in[1] + o, in[2] + o, in[3] + o, in[4] + o, in[5] + o,
            in[6] + o, ops.deriv.data(), scratch.data(), scratch.data() + 3 * np, out[0] + o,
            out[1] + o, out[2] + o);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// bench::count_ops (bench.hpp:160-192): CountReal flux evaluations and flops of
// both volume kernels over k elements -> out[4] = evals_split, evals_std,
// flops_split, flops_std.
int ref_count_ops(int degree, long k, uint64_t* out) {
  try {
    std::uint64_t a, b, c, d;
    bench::count_ops(degree, k, a, b, c, d);
    out[0] = a;
    out[1] = b;
    out[2] = c;
    out[3] = d;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The rough synthetic state of the reference's kernel benchmark
// (bench.hpp:108-121, bench::KernelBuffers::init): std::mt19937(20250810),
// h ~ U(0.5, 2), hu = h U(-1, 1), hv = h U(-1, 1), node-major over k elements.
int ref_bench_rough_state(int degree, long k, double* h, double* hu, double* hv) {
  try {
    bench::KernelBuffers kb;
    kb.init(degree, k);
    std::copy(kb.h.begin(), kb.h.end(), h);
    std::copy(kb.hu.begin(), kb.hu.end(), hu);
    std::copy(kb.hv.begin(), kb.hv.end(), hv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
