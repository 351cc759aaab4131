# multi-rank harness check on one GPU: 2 ranks, gloo, both on device 0
TS_BENCH_BACKEND=gloo TS_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-sweep --splat-points 20000000 > gpurun_out/b51.json 2> gpurun_out/b51.err; echo "exit $?"
cat gpurun_out/b51.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['ms_per_step'], d['config']['parallelism'], d['e2e']['value'], d['splat']['value'])"
tail -5 gpurun_out/b51.err
TS_BENCH_BACKEND=gloo TS_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/b51r.json 2>/dev/null; echo "ref exit $?"; head -c 300 gpurun_out/b51r.json
