# full ncu captures of the thin-layer direct conv kernels (enc*.0 and fuse.2)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_direct_kernel -s 1 -c 1 -o gpurun_out/prof_direct48 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'conv_direct_kernel<4>' -c 1 -o gpurun_out/prof_direct4 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
