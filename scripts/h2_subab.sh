# per-launch halo2 times: default, stacked with one 4-sub-tile buffer, stacked default
for CFG in "X=0" "TS_H2_STACK=1 TS_H2_SUBAB=4,1" "TS_H2_SUBAB=4,1"; do
env $CFG timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_halo2 -s 35 -c 35 --csv --log-file gpurun_out/h2s.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python - "$CFG" <<'PY'
import csv, sys
r=list(csv.reader(open('gpurun_out/h2s.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]; vi=h.index('Metric Value')
v=[float(x[vi].replace(',',''))/1e3 for x in r[hi+1:]]
print(sys.argv[1], ' '.join(f'{t:.0f}' for t in v), ' total', round(sum(v)))
PY
done
