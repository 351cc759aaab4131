# halo2 per-launch times under several environment settings
for CFG in ${CFGS:-"X=0" "TS_H2_HB=2" "TS_H2_SB=4" "TS_H2_SB=6"}; do
env $CFG timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_halo2 -s 34 -c 34 --csv --log-file gpurun_out/h2e.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python - "$CFG" <<'PY'
import csv, sys
r=list(csv.reader(open('gpurun_out/h2e.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]; vi=h.index('Metric Value')
v=[float(x[vi].replace(',',''))/1e3 for x in r[hi+1:]]
print(sys.argv[1], ' '.join(f'{t:.0f}' for t in v), ' total', round(sum(v)))
PY
done
