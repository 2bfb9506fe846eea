# compute-sanitizer memcheck / racecheck / synccheck over every stage-kernel family
# (element, node-per-thread incl. its viscous variant, half-line incl. the transposed
# node phase, viscous line pre-kernel, viscous stage, exact mode), the device mesh
# generator, the step reductions (run_steps with reductions: the two-step CUDA graph;
# step_device) on a small mesh; run via gpurun.
o=gpurun_out/${OUT:-sanitize.txt}; : > $o
for tool in memcheck racecheck synccheck; do
  for n in 1 2 3 4 7 8 15; do
    echo "== $tool N=$n" >> $o
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 6 --steps 3 --diag 2>&1 | grep -E "ERROR SUMMARY|Hazard|Error|error" | head -5 >> $o
  done
  for n in 2 3 4 7 12 13 15; do
    echo "== $tool visc N=$n" >> $o
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 6 --steps 3 --diag --viscous 2>&1 | grep -E "ERROR SUMMARY|Hazard|Error|error" | head -5 >> $o
  done
  echo "== $tool exact N=3" >> $o
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m paper_1804_02221_b200.profile_stage --degree 3 --kx 6 --steps 2 --diag --exact --viscous 2>&1 | grep -E "ERROR SUMMARY|Hazard|Error|error" | head -5 >> $o
done
cat $o
