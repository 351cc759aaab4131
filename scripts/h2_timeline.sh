# clock64 timeline of CTA 0 of chosen wide-M halo launches (TS_H2_DBG=<launch
# index counted over the process>; 35 halo2 launches per bench step):
# producer chunk completions, MMA hfull/acc waits, epilogue start/end.
for L in ${LAUNCHES:-35 51 67}; do
TS_H2_DBG=$L timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep 2>&1 >/dev/null | grep -A7 h2dbg
done
