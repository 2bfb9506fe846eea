// tests/cpp/shim_drop_in.cpp — the C++ drop-in (include/swdg_gpu.hpp) driven by the
// reference's own driver logic: run_simulation's step loop (driver.hpp:91-138) with
// swdg::gpu::TimeIntegrator substituted for swdg::TimeIntegrator.  Prints the step
// count and the FNV-1a state fingerprint.  Built here (needs the
// reference headers); the binary travels to the GPU box and runs there.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "swdg/driver.hpp"
#include "swdg_gpu.hpp"

using namespace swdg;

static uint64_t fnv(const State& s) {
  uint64_t h = 1469598103934665603ull;
  for (const std::vector<double>* a : {&s.h, &s.hu, &s.hv})
    for (double v : *a) {
      uint64_t w;
      std::memcpy(&w, &v, 8);
      h ^= w;
      h *= 1099511628211ull;
    }
  return h;
}

int main(int argc, char** argv) {
  const std::string id = argc > 1 ? argv[1] : "wetdry_dambreak";
  const int k = argc > 2 ? std::atoi(argv[2]) : 12;
  const double T = argc > 3 ? std::atof(argv[3]) : 0.2;
  const Scenario sc = make_scenario(id);
  RunConfig cfg = sc.config;
  cfg.kx = cfg.ky = k;
  cfg.final_time = T;
  Mesh mesh = build_mesh(cfg);
  State s = initial_state(sc, mesh);
  gpu::TimeIntegrator integ(mesh, cfg, /*exact=*/true);  // <- the one-line swap
  double t = 0.0;
  long steps = 0;
  const double t_eps = 1e-12 * std::max(1.0, T);
  while (t < T - t_eps) {
    double dt = compute_dt(s, mesh, cfg.phys, cfg.cfl);
    bool hit = false;
    if (t + dt >= T - t_eps) {
      dt = T - t;
      hit = true;
    }
    int rej = 0;
    while (!integ.try_step(s, t, dt)) {
      dt *= 0.5;
      hit = false;
      if (++rej >= 10) throw NumericalAbort("step rejected 10 times");
    }
    t = hit ? T : t + dt;
    ++steps;
  }
  std::printf("%s steps=%ld fnv=%016" PRIx64 "\n", id.c_str(), steps, fnv(s));
  return 0;
}
