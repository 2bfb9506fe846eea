# A/B stage timing: LIBS="a.so b.so" DEGS="..." VARS="default node" TAG=dir
O=gpurun_out/${TAG}; mkdir -p $O
for n in $DEGS; do for lib in ${LIBS:-paper_1804_02221_b200/_lib/libswdg_gpu.so}; do for v in ${VARS:-default}; do
  SWDG_LIB=$lib SWDG_FAST_VARIANT=$v timeout 200 python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 3 --time ${REPS:-10} ${EXTRA} 2>&1 | grep "^N=" | sed "s|^|$(basename $lib) $v |"
done; done; done | tee $O/ab.txt
