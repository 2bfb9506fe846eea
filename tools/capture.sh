#!/bin/bash
# Round-1 profiling pass on one B200 (run through gpurun from the repo root):
#   1. the bench line (N=7 headline) and the N=1..15 sweep
#   2. the ncu launch list of the bench command (per-launch gpu__time_duration)
#   3. one ncu --set full capture of the stage kernel per degree on the bench
#      mesh (1000x1000, 1M elements): DRAM traffic per launch, pipe use, stalls
# Outputs land in gpurun_out/prof_r01/; profiles/summarize_capture.py turns them
# into the committed profiles/r01_* files.
set -x
O=gpurun_out/prof_r01
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_n7.json 2> $O/bench_n7.err
timeout 600 python bench.py --steps 10 --warmup 3 --viscous --no-sweep > $O/bench_n7_visc.json 2> $O/bench_n7_visc.err
timeout 600 python bench.py --steps 5 --warmup 3 --distributed --no-sweep --cpu-budget 1 > $O/bench_n7_dist1.json 2> $O/bench_n7_dist1.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_n7.csv python bench.py --steps 2 --warmup 3 --cpu-budget 1 --no-sweep > /dev/null 2>&1
for n in ${DEGREES:-1 2 3 4 5 6 7 8 9 10 11 12 13 14 15}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stage -s 1 -c 1 \
    -o /tmp/stage_n$n -f python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 1 \
    > $O/ncu_n$n.log 2>&1
  ncu -i /tmp/stage_n$n.ncu-rep --page raw --csv > $O/ncu_n${n}_raw.csv 2>&1
done
for n in ${DEGREES:-1 2 3 4 5 6 7 8 9 10 11 12 13 14 15}; do
  timeout 200 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 3 --time 5 2>&1 | grep "^N="
done > $O/sweep.txt
for n in ${DEGREES_VISC:-2 3 4 5 6 7 8 9 10 11 12 13 14 15}; do
  timeout 300 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 3 --time 5 --viscous 2>&1 | grep "^N="
done > $O/sweep_visc.txt
ls -la $O
