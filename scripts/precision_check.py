"""Refine error vs the golden reference output for every precision mode."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20198_b200 import refiner as R
from paper_2509_20198_b200.patches import FaceMap, PatchKey, RawPatch

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "refiner.npz"))
raws = [RawPatch(PatchKey(0, 0, (320.0, 320.0), 100.0), g[f"in_hm_nn{i}"], g[f"in_hm_lin{i}"],
                 g[f"in_rgb_nn{i}"], g[f"in_rgb_lin{i}"],
                 FaceMap(96, np.zeros((96, 96), np.int32)), 25) for i in range(2)]
bundle = R.random_weights(R.default_descriptor(), seed=3)
for mode in range(5):
    res = R.refine_batch(raws, bundle, precision=mode)
    h = np.stack([r.heights_rel for r in res])
    c = np.stack([r.rgb for r in res])
    dh = np.abs(h - g["default_h"])
    print(f"mode {mode}: max|dh| {dh.max():.4g} m  rms {np.sqrt((dh**2).mean()):.3g}  "
          f"max|drgb| {np.abs(c - g['default_rgb']).max():.3g}  "
          f"|h| scale {np.abs(g['default_h']).max():.4g}")
