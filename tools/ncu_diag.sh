#!/bin/bash
# ncu --set full of the step-diagnostics kernel (k_step_diag) at the given degrees
#   N="2 7" TAG=dir bash tools/ncu_diag.sh
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
for n in $N; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_diag -c 1 \
    -o /tmp/ncu_diag_$n -f python bench.py --degree $n --steps 2 --warmup 3 --no-sweep --cpu-budget 1 \
    > $O/ncu_diag_N$n.log 2>&1
  ncu -i /tmp/ncu_diag_$n.ncu-rep --page raw --csv > $O/rawdiag_N$n.csv 2>&1
  ncu -i /tmp/ncu_diag_$n.ncu-rep --page source --csv --print-source sass > $O/srcdiag_N$n.csv 2>&1
done
