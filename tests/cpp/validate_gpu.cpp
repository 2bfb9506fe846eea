// tests/cpp/validate_gpu.cpp — the reference's acceptance criteria
// (proj/include/swdg/validate.hpp) with the INTEGRATION.md patch applied to
// build-time copies of driver.hpp and validate.hpp: every TimeIntegrator the
// criteria construct (validate.hpp:75, :278, :573, and run_simulation's at
// driver.hpp:75) is swdg::gpu::TimeIntegrator, exact mode, on the B200.
// Built without SWDG_VALIDATE_GPU against the unmodified headers it is the
// reference's own validation (validate_ref), the detail strings to compare with.
// Usage: validate_gpu [criterion ...]; prints one line per criterion and exits
// nonzero if any fails.  Test infrastructure (needs the reference headers to
// build; the binary travels to the GPU box).
#include <cstdio>
#include <string>
#include <vector>

#include <algorithm>

#ifdef SWDG_VALIDATE_GPU
#include "swdg_gpu.hpp"
#endif
// the patched copy (SWDG_INTEGRATOR = gpu::TimeIntegrator) for the GPU build, the
// unmodified reference for validate_ref
#include "swdg/validate.hpp"

int main(int argc, char** argv) {
  std::vector<std::string> want(argv + 1, argv + argc);
  int failed = 0, ran = 0;
  for (const auto& [name, fn] : swdg::validate::registry()) {
    if (!want.empty() && std::find(want.begin(), want.end(), name) == want.end()) continue;
    const swdg::validate::CriterionResult r = fn();
    ++ran;
    if (!r.pass) ++failed;
    std::printf("%s %s: %s\n", r.pass ? "PASS" : "FAIL", name.c_str(), r.detail.c_str());
    std::fflush(stdout);
  }
  std::printf("ran=%d failed=%d\n", ran, failed);
  return failed ? 1 : 0;
}
