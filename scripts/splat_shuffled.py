"""One shuffled configs[2] bake (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_20198_b200.engine import bake_device, key_grid  # noqa: E402

dev = torch.device("cuda", 0)
xyz, rgb, centers, per = bench.splat_inputs(200_000_000, dev)
P = len(centers)
perm = torch.randperm(len(xyz), device=dev)
xyz, rgb = xyz[perm], rgb[perm]
del perm
prior = torch.zeros((P, 64, 64), device=dev)
prior_rgb = torch.zeros((P, 64, 64, 3), device=dev)
cz = torch.full((P,), 50.0, dtype=torch.float64, device=dev)
grid = key_grid(centers)
for _ in range(2):
    bake_device(xyz, rgb, centers, prior, cz, cz, prior_rgb, grid)
torch.cuda.synchronize()
