timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 16 -c 1 -o gpurun_out/prof_tc5 python bench.py --steps 1 --warmup 1 --precision 3 --no-cpu --no-splat > /dev/null 2>&1
ls -la gpurun_out/prof_tc5.ncu-rep
