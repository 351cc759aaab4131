"""Where does a bench step's time go?  Kernel busy time vs gaps (host syncs,
launch overhead), plus the e2e copy costs.  Diagnostic only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_20198_b200 import _device as D  # noqa: E402
from paper_2509_20198_b200.lasio import parse_header  # noqa: E402
from paper_2509_20198_b200.pipeline import HeightmapPipeline  # noqa: E402
from paper_2509_20198_b200.refiner import default_descriptor, random_weights  # noqa: E402

torch.cuda.set_device(0)
tiles, own = bench.band_tiles(0, 1)
images = [t.data for t in tiles]
descs = np.concatenate([D.tile_desc(parse_header(b)) for b in images])
centers = D.upload(np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in own]))
cell_range = HeightmapPipeline.cell_range((0.0, 0.0), (32 * 640.0, 32 * 640.0))
pipe = HeightmapPipeline(random_weights(default_descriptor(), seed=3), 3)
tb = D.TileBatch(images, descs)
P = len(centers)


def step():
    t0 = time.perf_counter()
    tables, cp, idx = pipe.overview(tb, cell_range)
    t1 = time.perf_counter()
    g, t, o, cnn_in = pipe.patches(idx, centers)
    t2 = time.perf_counter()
    out, nf = pipe.refine(cnn_in, P)
    t3 = time.perf_counter()
    return out, (t1 - t0, t2 - t1, t3 - t2)


for _ in range(3):
    step()
torch.cuda.synchronize()
host = []
for _ in range(5):
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    out, h = step()
    e.record()
    torch.cuda.synchronize()
    host.append((s.elapsed_time(e),) + tuple(1e3 * x for x in h))
print("device ms, host ms (overview, patches, refine):")
for r in host:
    print("  %.2f | %.2f %.2f %.2f" % r)

from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
busy = sum(e.device_time for e in ev) / 1e3
print(f"kernel busy ms {busy:.2f} over {len(ev)} device events")
tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=18)
print(tab[:6000])

host_bytes = tb.bytes.cpu().pin_memory()
out_host = torch.empty((P, 64, 64, 4), dtype=torch.float32).pin_memory()
for _ in range(3):
    torch.cuda.synchronize()
    a, b, c, d = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    a.record()
    tb.bytes.copy_(host_bytes, non_blocking=True)
    b.record()
    out, _h = step()
    c.record()
    out_host.copy_(out, non_blocking=True)
    d.record()
    torch.cuda.synchronize()
    print("e2e: h2d %.2f step %.2f d2h %.2f ms" % (a.elapsed_time(b), b.elapsed_time(c),
                                                c.elapsed_time(d)))
