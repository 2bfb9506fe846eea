#!/bin/bash
# One ncu --set full capture (source-level, SASS) of the stage kernel per degree,
# on the bench mesh (1000x1000 wavy, 1M elements), one stage-2 launch (-s 1).
#   N="3 7 12" TAG=r02c [K=regex:k_stage] [EXTRA=--viscous] bash tools/ncu_kernels.sh
# Outputs in gpurun_out/$TAG: raw metrics CSV, SASS source CSV, details text.
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
for n in $N; do
  tag=${PFX:-inv}_N$n
  timeout 600 ncu --set full --import-source on --clock-control none -k ${K:-regex:k_stage} \
    -s ${SKIP:-1} -c 1 -o /tmp/ncu_$tag -f \
    python -m paper_1804_02221_b200.profile_stage --degree $n --kx ${KX:-1000} --steps 1 $EXTRA \
    > $O/ncu_$tag.log 2>&1
  ncu -i /tmp/ncu_$tag.ncu-rep --page raw --csv > $O/raw_$tag.csv 2>&1
  ncu -i /tmp/ncu_$tag.ncu-rep --page details > $O/details_$tag.txt 2>&1
  if [ -n "$SRC" ]; then
    ncu -i /tmp/ncu_$tag.ncu-rep --page source --csv --print-source sass > $O/src_$tag.csv 2>&1
  fi
done
