run() {
for E in $1; do
TS_H2_EXP=$E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_halo2 -s 34 -c 34 --csv --log-file gpurun_out/h2exp_$E.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
echo "$2 exp $E: $(python - <<PY
import csv
r=list(csv.reader(open('gpurun_out/h2exp_$E.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]; vi=h.index('Metric Value')
v=[float(x[vi].replace(',',''))/1e3 for x in r[hi+1:]]
print(' '.join(f'{t:.0f}' for t in v), ' total', round(sum(v)))
PY
)"
done
}
run "0 15" tryw
sed -i 's/mbarrier.try_wait.parity.shared::cta.b64 P1/mbarrier.test_wait.parity.shared::cta.b64 P1/' paper_2509_20198_b200/csrc/tc_ptx.cuh
make -C paper_2509_20198_b200/csrc > /dev/null 2>&1 || echo build failed
run "0 15" testw
