"""Batched, device-resident heightmap path (the benchmark's unit of work).

tile images in HBM --ts_chunk_counts/decode--> chunk tables
  --ts_extract_chunk_points--> chunk points (xyz f64, rgb f32, 640 m cells)
  --ts_index_build--> stable cell order (ChunkPointIndex)
  --ts_gather_count/fill--> patch-space points per patch (CSR)
  --ts_triangulate--> Delaunay triangles per patch
  --ts_raster--> B x 96 x 96 x 8 CNN input (+ re-centred c_z)
  --ts_refine--> B x 64 x 64 x 4 refined heights/rgb.

This is ``ScoutEngine.load_overview`` + the interpolate/refine tasks
(engine.py:157-175, 246-266) collapsed into one batched pass.  Three small
device->host reads size intermediate buffers (chunk total, cell grid,
gathered point total); everything else stays on the stream.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .patches import DeviceIndex, RASTER_RES, OUTPUT_RES, raster, triangulate
from .refiner import PRECISION_FP16X3, WeightBundle, device_weights


class HeightmapPipeline:
    def __init__(self, weights: WeightBundle, precision: int = PRECISION_FP16X3):
        self.weights = device_weights(weights, precision)
        self._ws = None
        self._ws_batch = 0

    def _workspace(self, batch):
        if self._ws is None or self._ws_batch < batch:
            self._ws = self.weights.workspace(batch)
            self._ws_batch = batch
        return self._ws

    @staticmethod
    def cell_range(bbox_min, bbox_max):
        """Inclusive 640 m cell range of a dataset bbox (plus one cell)."""
        lo = np.floor(np.asarray(bbox_min[:2], np.float64) / 640.0) - 1
        hi = np.floor(np.asarray(bbox_max[:2], np.float64) / 640.0) + 1
        return (int(lo[0]), int(lo[1]), int(hi[0]), int(hi[1]))

    def overview(self, tb: D.TileBatch, cell_range=None):
        """Chunk tables + chunk points + index (load_overview)."""
        tables = D.ChunkTables(tb)
        cp = D.ChunkPoints(tb, tables, records=False)
        idx = DeviceIndex(cp.xyz[:max(cp.n, 1)], cp.rgb, cp.cells[:max(cp.n, 1)],
                          cell_range)
        return tables, cp, idx

    def overview_staged(self, st, cell_range=None):
        """load_overview from files: ``lasio.reader.StagedChunkPoints``
        (tables decoded from the table bytes, first records from 64-byte
        windows of the reference's 4 KiB-aligned preads)."""
        cp = D.ChunkPoints(st.tb, st, records=False)
        D.raise_item_status(cp.status.cpu().numpy(), "chunk points")
        idx = DeviceIndex(cp.xyz[:max(cp.n, 1)], cp.rgb, cp.cells[:max(cp.n, 1)],
                          cell_range)
        return st, cp, idx

    def patches(self, idx: DeviceIndex, centers):
        """Gather + triangulate + rasterise every patch -> CNN input."""
        g = idx.gather(centers)
        t = triangulate(g)
        P = g["n"]
        cnn_in = D.empty((P, RASTER_RES, RASTER_RES, 8), torch.float32)
        o = raster(g, t, recenter=True, cnn_in=cnn_in)
        return g, t, o, cnn_in

    def refine(self, cnn_in, P):
        out = D.empty((P, OUTPUT_RES, OUTPUT_RES, 4), torch.float32)
        nonfinite = torch.zeros(P, dtype=torch.uint8, device=out.device)
        self.weights.run(cnn_in, P, out, nonfinite, self._workspace(P))
        return out, nonfinite

    def run(self, tb: D.TileBatch, centers, cell_range=None):
        """centers: (P, 2) patch centres (numpy, or a device tensor to keep
        host->device copies out of the step)."""
        tables, cp, idx = self.overview(tb, cell_range)
        g, t, o, cnn_in = self.patches(idx, centers)
        out, nonfinite = self.refine(cnn_in, g["n"])
        return dict(out=out, cz=o["cz"], status=o["status"],
                    tri_status=t["status"], tile_status=tables.status,
                    nonfinite=nonfinite, n_points=cp.n,
                    n_gathered=len(g["h"]), cnn_in=cnn_in, g=g, t=t)
