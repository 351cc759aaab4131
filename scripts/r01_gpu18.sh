source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0 128 13 141" x
for L in 34; do
TS_H2_EXP=128 TS_H2_DBG=$L timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat 2>&1 >/dev/null | grep -A5 h2dbg
done
