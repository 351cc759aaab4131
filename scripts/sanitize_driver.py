"""Small workloads of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): FP16X3 refine (wide-M halo kernel,
promoted epilogue, 1x1 merges), Delaunay (shared-memory and global-memory
patches), raster, bake (grouped + binned), LAZ chunk decode, render."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20198_b200 import _device as D  # noqa: E402
from paper_2509_20198_b200 import synth  # noqa: E402
from paper_2509_20198_b200.engine import bake_device, bin_points, key_grid  # noqa: E402
from paper_2509_20198_b200.lasio import parse_header  # noqa: E402
from paper_2509_20198_b200.pipeline import HeightmapPipeline  # noqa: E402
from paper_2509_20198_b200.refiner import default_descriptor, random_weights  # noqa: E402

what = sys.argv[1:] or ["refine", "geometry", "bake", "lazdec", "render"]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "refine" in what or "geometry" in what:
    tiles = synth.chunked_terrain_tiles(3, 2, chunks_per_tile=150)
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    pipe = HeightmapPipeline(random_weights(default_descriptor(), seed=3))
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in tiles])
    res = pipe.run(tb, centers)
    torch.cuda.synchronize()
    print("pipeline", res["out"].shape, int(res["status"].sum()))
if "geometry" in what:
    from paper_2509_20198_b200.patches import triangulate
    rng = np.random.default_rng(1)
    xys = [rng.uniform(-0.9, 0.9, (n, 2)) for n in (30, 500)]
    x = np.linspace(-0.9, 0.9, 370)
    xys.append(np.stack([x, 0.9 - 1.7 * x ** 2], 1))     # cavity overflow -> global
    off = np.concatenate([[0], np.cumsum([len(a) for a in xys])]).astype(np.int64)
    g = dict(n=len(xys), xy=D.upload(np.concatenate(xys)), h=D.upload(np.zeros(off[-1])),
             off=torch.from_numpy(off).cuda())
    t = triangulate(g)
    torch.cuda.synchronize()
    print("delaunay", t["status"].cpu().numpy())
if "bake" in what:
    dev = torch.device("cuda", 0)
    centers = np.stack(np.meshgrid(np.arange(4) * 640.0 + 320.0,
                                   np.arange(4) * 640.0 + 320.0), -1).reshape(-1, 2)
    rng = np.random.default_rng(2)
    m = 1 << 20
    xyz = D.upload(np.stack([rng.uniform(0, 2560, m), rng.uniform(0, 2560, m),
                             rng.uniform(0, 50, m)], 1))
    rgb = D.upload(rng.random((m, 3)).astype(np.float32))
    P = len(centers)
    prior = torch.zeros((P, 64, 64), device=dev)
    prior_rgb = torch.zeros((P, 64, 64, 3), device=dev)
    cz = torch.zeros(P, dtype=torch.float64, device=dev)
    h, _c = bake_device(xyz, rgb, centers, prior, cz, cz, prior_rgb)   # shuffled: binned
    torch.cuda.synchronize()
    print("bake", float(h.mean()))
if "lazdec" in what:
    g = np.load(os.path.join(root, "tests", "golden", "fullres.npz"))
    imgs = [g[f"file{k}"].tobytes() for k in range(4)]
    for k in range(4):
        tb = D.TileBatch([imgs[k]], D.tile_desc(parse_header(imgs[k])))
        fr = D.FullRecords(tb, D.ChunkTables(tb))
        torch.cuda.synchronize()
        print("lazdec", k, int(fr.status.sum()))
if "render" in what:
    from paper_2509_20198_b200.geometry import fit_overview
    from paper_2509_20198_b200.patches import PatchKey
    from paper_2509_20198_b200.refiner import RefinedPatch
    from paper_2509_20198_b200.render import (Framebuffer, rasterize_heightmaps,
                                              rasterize_points, resolve)
    cam = fit_overview((0, 0, 0), (640, 640, 20), (96, 96))
    fb = Framebuffer(96, 96)
    p = RefinedPatch(key=PatchKey(0, 0, (320.0, 320.0), 5.0),
                     heights_rel=np.zeros((64, 64), np.float32), rgb=None, provenance="refined")
    rasterize_heightmaps([p], cam, fb)
    rasterize_points(np.random.default_rng(3).uniform(0, 640, (1000, 3)), None, cam, fb)
    print("render", resolve(fb).shape)
