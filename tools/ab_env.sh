#!/bin/bash
# A/B of an environment switch: ENVVAR=name VALS="0 1" DEGS="..." [EXTRA=--viscous] TAG=dir
O=gpurun_out/${TAG}; mkdir -p $O
for n in $DEGS; do for v in $VALS; do
  env $ENVVAR=$v timeout 300 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 3 --time ${REPS:-10} ${EXTRA} 2>&1 | grep "^N=" | sed "s|^|$ENVVAR=$v |"
done; done | tee $O/ab_env.txt
