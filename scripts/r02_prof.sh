# halo2 wait profile per launch (profiling build), planes off / on
for P in 0 1; do
echo "== TS_PLANES=$P"
TS_PLANES=$P TS_LIB_PATH=build/prof/libts_b200.so timeout 300 python scripts/cnn_once.py 5 2>&1 | grep h2prof | tail -36
done
