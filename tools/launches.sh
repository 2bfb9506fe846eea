# per-kernel launch times of a few device-resident stages: N="2 3" EXTRA=--viscous TAG=dir
O=gpurun_out/${TAG}; mkdir -p $O
for n in $N; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python -m paper_1804_02221_b200.profile_stage --degree $n --kx 1000 --steps 2 $EXTRA 2>/dev/null | grep -v "^==" > $O/launch_$n.csv
python - $O/launch_$n.csv <<'PY'
import csv,sys,collections
rows=list(csv.DictReader(open(sys.argv[1])))
d=collections.defaultdict(list)
for r in rows:
    if r.get('Metric Name')=='gpu__time_duration.sum': d[r['Kernel Name'][:50]].append(float(r['Metric Value']))
for k,v in sorted(d.items(),key=lambda x:-sum(x[1])): print(sys.argv[1].split('_')[-1], f"{k:50s} n={len(v)} avg={sum(v)/len(v):.1f}")
PY
done
