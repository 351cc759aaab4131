for L in 67 68; do
TS_H2_DBG=$L timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep 2>&1 >/dev/null | grep -A7 h2dbg
done
