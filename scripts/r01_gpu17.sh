# halo2 timestamps of CTA 0: enc.1 (launch 34 = first halo2 of the 2nd step) and fuse.0 (launch 66)
for L in 34 66 50; do
TS_H2_DBG=$L timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat 2>&1 >/dev/null | grep -A13 h2dbg
done
