// tests/cpp/run_driver.cpp — run_simulation three ways on one scenario, writing
// the reference's output files (diagnostics.txt, snapshot_t*.txt) into OUTDIR:
//   built with -DSWDG_DRIVER_REF     : the unmodified reference driver (CPU)
//   built with -DSWDG_DRIVER_PATCHED : the reference driver.hpp with the
//        INTEGRATION.md patch, swdg::gpu::TimeIntegrator swapped in (B200)
//   built with -DSWDG_DRIVER_DEVICE  : swdg::gpu::run_simulation, the
//        device-resident driver of include/swdg_gpu_driver.hpp (B200)
// Usage: run_driver SCENARIO K T OUTDIR [snapshot_dt] [track] [fast]
// Prints the step count, the FNV-1a fingerprint of the final state and the
// worst limiter entropy jump.  Test infrastructure: built here against the
// reference headers, the binaries travel to the GPU box.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#if defined(SWDG_DRIVER_PATCHED) || defined(SWDG_DRIVER_DEVICE)
#include "swdg_gpu.hpp"
#endif
#ifdef SWDG_DRIVER_DEVICE
#include "swdg_gpu_driver.hpp"
#endif
#include "swdg/driver.hpp"  // the patched copy first on the include path for PATCHED

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
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s SCENARIO K T OUTDIR [snapshot_dt] [track] [fast]\n", argv[0]);
    return 2;
  }
  const Scenario sc = make_scenario(argv[1]);
  RunConfig cfg = sc.config;
  cfg.kx = cfg.ky = std::atoi(argv[2]);
  cfg.final_time = std::atof(argv[3]);
  cfg.out_dir = argv[4];
  if (argc > 5) cfg.snapshot_dt = std::atof(argv[5]);
  const bool track = argc > 6 && std::atoi(argv[6]) != 0;
#ifdef SWDG_DRIVER_DEVICE
  gpu::RunOptions opt;
  opt.exact = !(argc > 7 && std::atoi(argv[7]) != 0);
#else
  RunOptions opt;
#endif
  opt.write_files = true;
  opt.track_limiter_entropy = track;
  try {
#ifdef SWDG_DRIVER_DEVICE
    const RunResult r = gpu::run_simulation(cfg, opt);
#else
    const RunResult r = run_simulation(cfg, opt);
#endif
    std::printf("steps=%ld fnv=%016" PRIx64 " t=%.17g worst_jump=%.17g\n", r.steps, fnv(r.state),
                r.t, r.worst_limiter_entropy_jump);
  } catch (const NumericalAbort& e) {
    std::printf("NumericalAbort: %s\n", e.what());
    return 3;
  }
  return 0;
}
