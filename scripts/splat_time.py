"""configs[2] splat timing alone (grouped and shuffled), as bench.py's
splat line computes it:  python scripts/splat_time.py"""
import json
import os
import sys
import types

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

args = types.SimpleNamespace(splat_points=200_000_000, warmup=3, steps=10)
r = bench.run_splat(args, torch.device("cuda", 0), 1, 0)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"],
                  "shuffled_ms": r["shuffled"]["ms_per_step"]}))
