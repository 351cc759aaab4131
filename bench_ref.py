"""The reference arm of bench.py: the UNMODIFIED reference package
(`terrascout`, pip-installed into baseline/_ref from /root/reference/pkg)
timed through its own public API on the host cores.

Workload = a bounded sample of BASELINE.json configs[1] (the same seeded
stub-body LAZ corpus bench.py's GPU arm runs, written to a temp directory
so the reference reads real files):

  per step  read_chunk_points + positions + colors + ChunkPointIndex for
            every tile of an 8 x 8 corner (reader.py:239-283, the chunk
            table re-decoded each step), reconstruct_patch for the sample
            patches on a fork pool of all host cores (patches.py:408-412),
            refine_batch of the sample (refiner.py:475-528, OpenBLAS on all
            cores).

`configs0()` runs configs[0] as BASELINE.md specifies: ScoutEngine
.load_overview + run_until_idle (engine.py:157-175, 362-379) over the 8 x 8
corpus with batch_max = 64 and the random seed-3 bundle.

Falls back to the oracle/ port (kind "port") when baseline/_ref is absent.
"""

from __future__ import annotations

import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "baseline", "_ref")

_G = {}  # fork-inherited state of the reconstruct workers


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "terrascout"))


def _reconstruct(key):
    from terrascout.patches import reconstruct_patch
    return reconstruct_patch(key, _G["index"])


class RefArm:
    def __init__(self, tiles_side: int = 8, sample: int = 32,
                 chunks_per_tile: int = 150):
        if REF not in sys.path:
            sys.path.insert(0, REF)
        import terrascout  # noqa: F401  (the installed reference)
        from terrascout.lasio import scan_tile
        from terrascout.refiner import default_descriptor, random_weights

        from paper_2509_20198_b200 import synth  # corpus generator only
        self.tmp = tempfile.TemporaryDirectory(prefix="ts_ref_")
        tiles = synth.chunked_terrain_tiles(tiles_side, tiles_side,
                                            chunks_per_tile=chunks_per_tile)
        self.paths = []
        for i, t in enumerate(tiles):
            p = os.path.join(self.tmp.name, f"tile_{i:04d}.laz")
            with open(p, "wb") as fp:
                fp.write(t.data)
            self.paths.append(p)
        self.scan_tile = scan_tile
        self.centers = [(t.x0 + 320.0, t.y0 + 320.0) for t in tiles][:sample]
        self.sample = len(self.centers)
        self.weights = random_weights(default_descriptor(), seed=3)
        self.cores = len(os.sched_getaffinity(0))
        self.module = terrascout.__file__

    def step(self) -> float:
        """One timed pass over the sample; returns seconds."""
        import multiprocessing as mp

        from terrascout.lasio import colors, positions, read_chunk_points
        from terrascout.patches import ChunkPointIndex, PatchKey
        from terrascout.refiner import refine_batch
        t0 = time.perf_counter()
        index = ChunkPointIndex()
        for i, p in enumerate(self.paths):
            tile = self.scan_tile(p, i)          # chunk table decoded again
            rec = read_chunk_points(tile)
            index.add_points(positions(rec, tile.header),
                             colors(rec, tile.header))
        keys = [PatchKey(int(cx // 640), int(cy // 640), (cx, cy), 0.0)
                for cx, cy in self.centers]
        _G["index"] = index
        # fork after the index exists: workers inherit it, nothing pickled
        with mp.get_context("fork").Pool(self.cores) as pool:
            raws = pool.map(_reconstruct, keys, chunksize=1)
        refine_batch(raws, self.weights)
        return time.perf_counter() - t0

    def configs0(self) -> dict:
        """configs[0]: the full reference engine over the 8 x 8 corpus."""
        from terrascout.engine import Dataset, EngineConfig, ScoutEngine
        t0 = time.perf_counter()
        ds = Dataset.scan(self.paths)
        eng = ScoutEngine(ds, EngineConfig(batch_max=64), self.weights)
        eng.load_overview()
        tasks = eng.run_until_idle()
        dt = time.perf_counter() - t0
        n = len(eng.refined)
        return {"workload": "configs[0]: 8x8 tiles, ScoutEngine.load_overview"
                            " + run_until_idle (batch_max 64, random seed-3 "
                            "bundle), reference engine as shipped",
                "value": round(n / dt, 3), "unit": "heightmaps/s",
                "seconds": round(dt, 2), "refined": n, "tasks": tasks}

    def close(self):
        self.tmp.cleanup()
