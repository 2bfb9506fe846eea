#!/bin/sh
# tests/cpp/patch_reference.sh REF_INC OUT — the drop-in patch of INTEGRATION.md,
# applied to build-time copies of the reference's driver.hpp and validate.hpp in
# OUT/swdg/ (git-ignored build output; the reference tree is never modified).
# Every occurrence of the integrator type in the two files becomes
# SWDG_INTEGRATOR, which defaults to the reference's swdg::TimeIntegrator; a TU
# that includes swdg_gpu.hpp first and defines SWDG_INTEGRATOR=gpu::TimeIntegrator
# gets the reference's run_simulation and validation criteria on the B200.
set -e
REF_INC=$1
OUT=$2
mkdir -p "$OUT/swdg"
for f in driver validate; do
  src="$REF_INC/swdg/$f.hpp"
  dst="$OUT/swdg/$f.hpp"
  {
    echo '#pragma once'
    echo '#ifndef SWDG_INTEGRATOR'
    echo '#define SWDG_INTEGRATOR TimeIntegrator'
    echo '#endif'
    sed -e 's/^#pragma once$//' \
        -e 's/const TimeIntegrator&/const SWDG_INTEGRATOR\&/g' \
        -e 's/^\(  *\)TimeIntegrator integ(mesh, cfg);/\1SWDG_INTEGRATOR integ(mesh, cfg);/' "$src"
  } > "$dst"
done
# the patch must have hit every site: driver.hpp:20 (on_step) and :75 (ctor);
# validate.hpp:75, :278, :573 (ctors) and :659 (on_step lambda)
test "$(grep -c 'SWDG_INTEGRATOR integ(mesh, cfg)' "$OUT/swdg/driver.hpp")" = 1
test "$(grep -c 'const SWDG_INTEGRATOR&' "$OUT/swdg/driver.hpp")" = 1
test "$(grep -c 'SWDG_INTEGRATOR integ(mesh, cfg)' "$OUT/swdg/validate.hpp")" = 3
test "$(grep -c 'const SWDG_INTEGRATOR&' "$OUT/swdg/validate.hpp")" = 1
