# halo2 experiment builds (build/exp_*): CNN time per variant, per-layer launch list
for T in base noepi nocorr mmaonly mmaonly1; do
  if [ $T = base ]; then L=paper_2509_20198_b200/libts_b200.so; else L=build/exp_$T/libts_b200.so; fi
  echo "== $T"; TS_LIB_PATH=$L timeout 300 python scripts/cnn_time.py 5 2>&1 | tail -1
  TS_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/layers_$T.csv python scripts/cnn_once.py 5 > /dev/null 2>&1
  echo "== layers $T"; python scripts/layer_table.py gpurun_out/layers_$T.csv | tail -45 | awk '{printf "%s ", $1} END {print ""}'
done
