# planes vs fp32 activations: outputs must be bit-identical
cat > /tmp/cmp.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_20198_b200.refiner import PRECISION_BF16X4, PRECISION_BF16, PRECISION_BF16X3, default_descriptor, device_weights, random_weights
bundle = random_weights(default_descriptor(), seed=3)
g = torch.Generator(device="cuda").manual_seed(5)
B = 70
x = torch.randn((B, 96, 96, 8), generator=g, device="cuda") * 0.1
x[..., 2:] = torch.rand((B, 96, 96, 6), generator=g, device="cuda")
for prec in (PRECISION_BF16X4, PRECISION_BF16, PRECISION_BF16X3):
    w = device_weights(bundle, prec)
    out = torch.empty((B, 64, 64, 4), device="cuda"); nf = torch.zeros(B, dtype=torch.uint8, device="cuda")
    w.run(x, B, out, nf); torch.cuda.synchronize()
    np.save(f"/tmp/out_{os.environ.get('TS_PLANES','1')}_{prec}.npy", out.cpu().numpy())
PY
TS_PLANES=0 python /tmp/cmp.py && TS_PLANES=1 python /tmp/cmp.py && python -c "
import numpy as np
for p in (4,2,3):
  a=np.load(f'/tmp/out_0_{p}.npy'); b=np.load(f'/tmp/out_1_{p}.npy')
  print('mode',p,'bit-identical' if np.array_equal(a,b) else 'DIFF max %g'%np.abs(a-b).max())
"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests32.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests32.log
for V in 0 1; do
TS_PLANES=$V timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench32.json 2> gpurun_out/bench32.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench32.json')); print('planes $V', d['value'], d['stages_ms'])"
done
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" planes
