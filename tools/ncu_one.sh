# usage: V=variant N=degree TAG=dir bash scripts/ncu_one.sh
O=gpurun_out/${TAG}; mkdir -p $O
for n in $N; do
SWDG_FAST_VARIANT=$V timeout 300 ncu --set full --import-source on --clock-control none -k regex:${K:-k_stage} -s ${SKIP:-1} -c ${CNT:-1} -o /tmp/r_$n -f python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 1 ${EXTRA} > $O/ncu$n.log 2>&1
ncu -i /tmp/r_$n.ncu-rep --page raw --csv > $O/raw_$n.csv
ncu -i /tmp/r_$n.ncu-rep --page source --csv --print-source sass > $O/src_$n.csv 2>&1
ncu -i /tmp/r_$n.ncu-rep --page details > $O/details_$n.txt 2>&1
done
