for E in 15 7; do
TS_H2_EXP=$E TS_H2_DBG=66 timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat 2>&1 >/dev/null | grep -A8 h2dbg
done
