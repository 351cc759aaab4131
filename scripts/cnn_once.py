"""One warm-up + one profiled CNN refine of 1,024 tiles (for ncu launch
lists: python scripts/cnn_once.py <mode>)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20198_b200 import refiner as R  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B = 1024
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randn((B, 96, 96, 8), generator=g, device="cuda") * 0.1
x[..., 2:] = torch.rand((B, 96, 96, 6), generator=g, device="cuda")
w = R.device_weights(R.random_weights(R.default_descriptor(), seed=3), mode)
out = torch.empty((B, 64, 64, 4), device="cuda")
nf = torch.zeros(B, dtype=torch.uint8, device="cuda")
ws = w.workspace(B)
for _ in range(2):
    w.run(x, B, out, nf, ws)
torch.cuda.synchronize()
