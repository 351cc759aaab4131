"""CNN refine time per 1,024-tile batch for the given precision modes
(CUDA events, inputs resident, 3 warm-up + 10 timed runs each).

    python scripts/cnn_time.py 4 5
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20198_b200 import refiner as R  # noqa: E402

CROP_GFLOP = 2.283


def main():
    modes = [int(m) for m in sys.argv[1:]] or [4, 5]
    B = 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((B, 96, 96, 8), generator=g, device="cuda") * 0.1
    x[..., 2:] = torch.rand((B, 96, 96, 6), generator=g, device="cuda")
    bundle = R.random_weights(R.default_descriptor(), seed=3)
    for mode in modes:
        w = R.device_weights(bundle, mode)
        out = torch.empty((B, 64, 64, 4), device="cuda")
        nf = torch.zeros(B, dtype=torch.uint8, device="cuda")
        ws = w.workspace(B)
        for _ in range(3):
            w.run(x, B, out, nf, ws)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            w.run(x, B, out, nf, ws)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"mode {mode}: {ms:.3f} ms / {B} tiles  "
              f"{CROP_GFLOP * B / ms:.1f} TFLOP/s alg  "
              f"[{'pair' if os.environ.get('TS_H2_PAIR') == '1' else 'default'}]", flush=True)


if __name__ == "__main__":
    main()
