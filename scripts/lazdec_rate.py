"""Chunk-decode throughput: the realistic golden tile replicated N times
(python scripts/lazdec_rate.py 16 256 1024)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20198_b200 import _device as D  # noqa: E402
from paper_2509_20198_b200.lasio import parse_header  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "fullres_big.npz"))
img = g["laz"].tobytes()
for reps in [int(a) for a in sys.argv[1:]] or [16, 256]:
    imgs = [img] * reps
    descs = np.concatenate([D.tile_desc(parse_header(img))] * reps)
    tb = D.TileBatch(imgs, descs)
    tables = D.ChunkTables(tb)
    fr = D.FullRecords(tb, tables)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fr = D.FullRecords(tb, tables)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    n = fr.n_points
    print(f"{reps} tiles, {tables.total} chunks, {n:,} points: {ms:.1f} ms, "
          f"{n / ms / 1e3:.1f} M points/s, status ok {not fr.status.any()}", flush=True)
