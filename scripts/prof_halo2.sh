# full ncu captures of halo2 layers: dec_h.2 (3rd launch) and fuse.0 (7th)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:halo2 -s 2 -c 1 -o gpurun_out/prof_h2_dec3 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > gpurun_out/prof_log.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:halo2 -s 6 -c 1 -o gpurun_out/prof_h2_fuse0 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > gpurun_out/prof_log.txt 2>&1
ls gpurun_out/*.ncu-rep
