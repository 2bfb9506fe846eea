#!/bin/bash
# End-of-round measurement pass on one B200 (through gpurun, from the repo root):
# GPU tests, the bench lines (headline + sweep, viscous, the distributed path at
# world size 1 inviscid and viscous, the reference arm), the ncu launch list of
# the bench command and the compute-sanitizer pass.  Outputs in gpurun_out/$TAG.
O=gpurun_out/${TAG:-final}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1; tail -1 $O/gputests.txt
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --viscous > $O/bench_visc.json 2> $O/bench_visc.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29513 bench.py --distributed --no-sweep --steps 10 --warmup 3 --cpu-budget 1 \
  > $O/bench_dist1.json 2> $O/bench_dist1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29514 bench.py --distributed --viscous --no-sweep --steps 10 --warmup 3 --cpu-budget 1 \
  > $O/bench_dist1_visc.json 2> $O/bench_dist1_visc.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_n7.csv python bench.py --steps 2 --warmup 3 --cpu-budget 1 --no-sweep \
  > /dev/null 2>&1
[ -n "$SANITIZE" ] && OUT=${TAG:-final}/sanitize.txt bash tools/sanitize.sh > /dev/null 2>&1
for f in $O/bench*.json; do echo "$f $(head -c 300 $f)"; done
