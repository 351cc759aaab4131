# per-launch halo2 times of one bench step under each value of a switch:
#   bash scripts/h2_ab_times.sh TS_H2_PAIR 0 1
V=$1; shift
for X in "$@"; do
env $V=$X timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_halo2 -s 35 -c 35 --csv --log-file gpurun_out/h2_times_$X.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python - $X <<'PY'
import csv, sys
r=list(csv.reader(open(f'gpurun_out/h2_times_{sys.argv[1]}.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]; vi=h.index('Metric Value')
v=[float(x[vi].replace(',',''))/1e3 for x in r[hi+1:]]
print(sys.argv[1], ' '.join(f'{t:.0f}' for t in v), ' total', round(sum(v)))
PY
done
