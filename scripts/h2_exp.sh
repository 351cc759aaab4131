# halo2 timing experiments (garbage numerics): 0 normal, 1 weights resident, 2 no halo fill, 3 both
for e in ${EXPS:-0 1 2 3}; do
TS_H2_EXP=$e timeout 100 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:halo2 -s 8 -c 8 --csv --log-file gpurun_out/h2exp_$e.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
echo "exp $e: $(python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/h2exp_$e.csv')))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[hi]
print(' '.join('%.0f'%(float(r[h.index('Metric Value')].replace(',',''))/1000) for r in rows[hi+1:]))
PY
)"
done
