# full ncu captures: fuse.0 (largest halo-kernel launch) and enc*.1 (regular kernel)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo -s 6 -c 1 -o gpurun_out/prof_fuse0 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > gpurun_out/prof_log.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'conv_tc_kernel' -c 1 -o gpurun_out/prof_enc1 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > gpurun_out/prof_log.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'conv_tc_kernel' -s 8 -c 1 -o gpurun_out/prof_merge0 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > gpurun_out/prof_log.txt 2>&1
ls gpurun_out/*.ncu-rep
