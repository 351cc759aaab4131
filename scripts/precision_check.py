"""Refine error of every precision mode against the fp32 oracle.

Inputs: the CNN rasters of a real 6 x 6-tile configs[1]-style batch (36
patches, built by the device pipeline) plus the two golden rasters.  The
reference output is the oracle's numpy float32 forward (im2col + sgemm,
refiner.py:330-441) on the same rasters.  Bundles: random He weights (seed
3, which amplify per-layer error through 11 layers) and the same bundle
scaled to a 'smooth' passthrough-like regime (weights x 0.5).

    python scripts/precision_check.py [modes...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refiner as oref  # noqa: E402
from paper_2509_20198_b200 import _device as D  # noqa: E402
from paper_2509_20198_b200 import refiner as R  # noqa: E402
from paper_2509_20198_b200 import synth  # noqa: E402
from paper_2509_20198_b200.lasio import parse_header  # noqa: E402
from paper_2509_20198_b200.pipeline import HeightmapPipeline  # noqa: E402


def rasters():
    side = 6
    tiles = synth.chunked_terrain_tiles(side, side, chunks_per_tile=150)
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    pipe = HeightmapPipeline(R.random_weights(R.default_descriptor(), seed=3), 0)
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in tiles])
    res = pipe.run(tb, centers)
    x = res["cnn_in"].cpu().numpy()
    g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                             "refiner.npz"))
    extra = np.stack([oref.stage_inputs(g[f"in_hm_nn{i}"], g[f"in_hm_lin{i}"],
                                        g[f"in_rgb_nn{i}"], g[f"in_rgb_lin{i}"])
                      .transpose(1, 2, 0) for i in range(2)])
    return np.concatenate([x, extra]).astype(np.float32)


def main():
    modes = [int(m) for m in sys.argv[1:]] or [0, 2, 4, 5]
    x = rasters()
    B = len(x)
    for label, scale in (("He seed 3", 1.0), ("He seed 3 x0.5", 0.5)):
        bundle = R.random_weights(R.default_descriptor(), seed=3)
        if scale != 1.0:
            bundle.tensors = {k: (v * np.float32(scale)).astype(np.float32)
                              for k, v in bundle.tensors.items()}
        layers = oref.text_to_layers(bundle.descriptor.to_text())
        ref = oref.forward(layers, bundle.tensors, x.transpose(0, 3, 1, 2))
        ref = ref[:, :, 16:80, 16:80]
        href = ref[:, 0] * np.float32(480.0)
        print(f"{label}: {B} tiles, |h| max {np.abs(href).max():.3g} m")
        for mode in modes:
            w = R.device_weights(bundle, mode)
            out = torch.empty((B, 64, 64, 4), device="cuda")
            nf = torch.zeros(B, dtype=torch.uint8, device="cuda")
            w.run(torch.from_numpy(x).cuda(), B, out, nf)
            o = out.cpu().numpy()
            dh = np.abs(o[..., 0] - href)
            dc = np.abs(o[..., 1:4] - np.clip(ref[:, 1:4].transpose(0, 2, 3, 1), 0, 1))
            print(f"  mode {mode}: max|dh| {dh.max():.3e} m  rms {np.sqrt((dh ** 2).mean()):.3e}"
                  f"  max|drgb| {dc.max():.3e}  nonfinite {int(nf.sum())}")


if __name__ == "__main__":
    main()
