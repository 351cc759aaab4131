"""Country-scale streaming driver (BASELINE.json configs[3]).

A cols x rows patch grid (configs[3]: 1,000 x 1,000 = 1 M tiles) is too large
to hold as tile images, so it is streamed through ``HeightmapPipeline`` in
rectangular blocks of tiles:

  * each rank owns a contiguous band of grid rows (``parallel.band_for``);
  * each block = up to ``block x block`` owned tiles plus a one-tile halo
    ring (clipped to the grid): chunk points of neighbouring tiles reach
    480 m into a patch's padded square, so every patch of the block sees
    exactly the points it would see in one whole-grid run (the streamed
    result equals the unsharded run bit for bit, tests/test_gpu_country.py);
  * refined tiles land in one device array per rank, in row-major order of
    the rank's band; ``gather`` is the only collective (NCCL to rank 0,
    ``parallel.gather_tiles``).

Tile images are synthesised on the host (this is the data source, not the
measured path): a pool of distinct stub-body LAZ tiles generated once
(``synth.grid_tiles``) is re-used with every chunk's first record moved to
the virtual tile's footprint (x, y integers shifted by whole tiles), so the
chunk tables, record formats and per-tile point counts are those of real
tiles.  A producer thread concatenates block i+1's pool images straight into
pinned memory (one numpy call) while the GPU runs block i; the upload runs
on a copy stream and the record moves are applied on the device
(``TilePool.move_records``, byte-for-byte what ``images_for`` does on the
host).
"""

from __future__ import annotations

import queue
import threading

import numpy as np
import torch

from . import _device as D
from . import synth
from .lasio import parse_header
from .parallel import band_for
from .pipeline import HeightmapPipeline

TILE = 640.0


class TilePool:
    """Distinct stub-body tiles whose records are re-placed per virtual tile."""

    def __init__(self, side: int = 16, chunks_per_tile: int = 150,
                 points_per_chunk: int = 50_000, seed: int = 1):
        tiles = synth.grid_tiles((0, side), (0, side),
                                 chunks_per_tile=chunks_per_tile,
                                 points_per_chunk=points_per_chunk,
                                 record_seed=seed)
        self.n = len(tiles)
        self.images = [np.frombuffer(t.data, np.uint8) for t in tiles]
        self.sizes = np.array([len(t.data) for t in tiles], np.int64)
        # the images again, each zero-padded to 16 bytes, as views of one
        # array (the block buffers are their concatenation)
        self.aligned = (self.sizes + 15) // 16 * 16
        flat = np.zeros(int(self.aligned.sum()), np.uint8)
        o = np.concatenate([[0], np.cumsum(self.aligned)[:-1]])
        for i, im in enumerate(self.images):
            flat[o[i]:o[i] + len(im)] = im
        self.padded = [flat[o[i]:o[i] + self.aligned[i]] for i in range(self.n)]
        self._rec_off_dev = {}
        self.pos = np.array([[round(t.x0 / TILE), round(t.y0 / TILE)]
                             for t in tiles], np.int64)
        self.rec_off = np.stack([t.chunk_offsets for t in tiles]).astype(np.int64)
        self.desc = np.concatenate([D.tile_desc(parse_header(t.data))
                                    for t in tiles])
        sx, sy = self.desc["scale"][0, 0], self.desc["scale"][0, 1]
        self.step = (int(round(TILE / sx)), int(round(TILE / sy)))

    def pick(self, cx: np.ndarray, cy: np.ndarray) -> np.ndarray:
        return (cx * 7919 + cy * 104729) % self.n

    def stage(self, cx: np.ndarray, cy: np.ndarray, pin: bool = True):
        """Block staging for the streaming driver: the chosen pool images
        concatenated into a pinned buffer (records NOT yet moved), the
        descriptors, and a pinned int64 (4, n) array (pool tile, image
        offset, x and y shift in record units) for ``move_records``."""
        k = self.pick(cx, cy)
        al = self.aligned[k]
        offs = np.zeros(len(k), np.int64)
        offs[1:] = np.cumsum(al)[:-1]
        total = int(al.sum())
        pinned = torch.empty(total + D.TileBatch.PAD, dtype=torch.uint8, pin_memory=pin)
        host = pinned.numpy()
        np.concatenate([self.padded[i] for i in k], out=host[:total])
        host[total:] = 0
        meta = torch.empty((4, len(k)), dtype=torch.int64, pin_memory=pin)
        m = meta.numpy()
        m[0], m[1] = k, offs
        m[2] = (cx - self.pos[k, 0]) * self.step[0]
        m[3] = (cy - self.pos[k, 1]) * self.step[1]
        descs = self.desc[k].copy()
        descs["file_offset"] = offs
        descs["file_size"] = self.sizes[k]
        return pinned, descs, meta

    def move_records(self, d_bytes: torch.Tensor, meta: torch.Tensor) -> None:
        """On the device: every chunk's first record of tile i moves by
        (meta[2, i], meta[3, i]) record units in x and y (little-endian int32
        at record bytes 0 and 4, wrapping like the host path)."""
        dev = d_bytes.device
        ro = self._rec_off_dev.get(dev)
        if ro is None:
            ro = self._rec_off_dev[dev] = torch.from_numpy(self.rec_off).to(dev)
        nch = ro.shape[1]
        idx = (meta[1][:, None] + ro[meta[0]]).reshape(-1)
        for axis, shift in ((0, meta[2]), (4, meta[3])):
            j = idx + axis
            v = torch.zeros_like(j)
            for t in range(4):
                v |= d_bytes[j + t].to(torch.int64) << (8 * t)
            v = (v + shift.repeat_interleave(nch)) & 0xFFFFFFFF
            for t in range(4):
                d_bytes[j + t] = ((v >> (8 * t)) & 0xFF).to(torch.uint8)

    def images_for(self, cx: np.ndarray, cy: np.ndarray):
        """Host image buffer (16-byte aligned tiles) + descriptors."""
        k = self.pick(cx, cy)
        sizes = self.sizes[k]
        aligned = (sizes + 15) // 16 * 16
        offs = np.zeros(len(k), np.int64)
        offs[1:] = np.cumsum(aligned)[:-1]
        buf = np.zeros(int(aligned.sum()) + D.TileBatch.PAD, np.uint8)
        for i, kk in enumerate(k):
            buf[offs[i]:offs[i] + sizes[i]] = self.images[kk]
        # move every first record's x, y by whole tiles (exact integers)
        pos = offs[:, None] + self.rec_off[k]
        four = np.arange(4)
        for axis, d in ((0, (cx - self.pos[k, 0]) * self.step[0]),
                        (4, (cy - self.pos[k, 1]) * self.step[1])):
            idx = (pos + axis)[..., None] + four
            v = buf[idx].view("<i4")[..., 0].astype(np.int64) + d[:, None]
            buf[idx] = v.astype("<i4")[..., None].view(np.uint8).reshape(idx.shape)
        descs = self.desc[k].copy()
        descs["file_offset"] = offs
        descs["file_size"] = sizes
        return buf, descs


class CountryRun:
    """Stream a rank's band of the grid through the pipeline in blocks."""

    def __init__(self, pipe: HeightmapPipeline, pool: TilePool, cols: int,
                 rows: int, block: int = 64, rank: int = 0, world: int = 1):
        self.pipe, self.pool = pipe, pool
        self.cols, self.rows = cols, rows
        self.band = band_for(rank, world, rows)
        b = self.band
        self.blocks = [(c0, min(c0 + block, cols), r0, min(r0 + block, b.row1))
                       for r0 in range(b.row0, b.row1, block)
                       for c0 in range(0, cols, block)]
        self.n_owned = cols * b.own_rows
        self.dev = D.device()
        self.out = torch.empty((self.n_owned, 64, 64, 4), dtype=torch.float32,
                               device=self.dev)
        self.cz = torch.empty((self.n_owned,), dtype=torch.float64, device=self.dev)
        self.status = torch.empty((self.n_owned,), dtype=torch.int32, device=self.dev)

    def _host_block(self, blk):
        c0, c1, r0, r1 = blk
        h0, h1 = max(0, r0 - 1), min(self.rows, r1 + 1)
        g0, g1 = max(0, c0 - 1), min(self.cols, c1 + 1)
        cy, cx = np.meshgrid(np.arange(h0, h1), np.arange(g0, g1), indexing="ij")
        pinned, descs, meta = self.pool.stage(cx.ravel(), cy.ravel())
        oy, ox = np.meshgrid(np.arange(r0, r1), np.arange(c0, c1), indexing="ij")
        centers = np.stack([ox.ravel() * TILE + TILE / 2,
                            oy.ravel() * TILE + TILE / 2], 1)
        cr = HeightmapPipeline.cell_range((g0 * TILE, h0 * TILE),
                                          (g1 * TILE, h1 * TILE))
        return blk, pinned, descs, meta, centers, cr

    def run(self, on_block=None):
        """Process every block; returns host-side block count.  on_block(i)
        is called after block i is queued on the device (timing hooks)."""
        q: queue.Queue = queue.Queue(maxsize=2)

        def produce():
            for blk in self.blocks:
                q.put(self._host_block(blk))
            q.put(None)

        th = threading.Thread(target=produce, daemon=True)
        th.start()
        stream = torch.cuda.current_stream()
        copy_s = torch.cuda.Stream(device=self.dev)
        i = 0
        while True:
            item = q.get()
            if item is None:
                break
            (c0, c1, r0, r1), pinned, descs, meta, centers, cr = item
            # allocated on the copy stream (written there first); the
            # record_stream below keeps them from being reused there until
            # the compute stream is done with them
            with torch.cuda.stream(copy_s):
                d_bytes = torch.empty(pinned.shape, dtype=torch.uint8, device=self.dev)
                d_meta = torch.empty(meta.shape, dtype=torch.int64, device=self.dev)
                d_bytes.copy_(pinned, non_blocking=True)
                d_meta.copy_(meta, non_blocking=True)
            stream.wait_stream(copy_s)
            d_bytes.record_stream(stream)
            d_meta.record_stream(stream)
            self.pool.move_records(d_bytes, d_meta)
            tb = D.TileBatch.from_device(d_bytes, descs)
            res = self.pipe.run(tb, centers, cr)
            # owned tiles of the block -> row-major slots of the band
            n = (r1 - r0) * (c1 - c0)
            rr = torch.arange(r0, r1, device=self.dev).repeat_interleave(c1 - c0)
            cc = torch.arange(c0, c1, device=self.dev).repeat(r1 - r0)
            slot = (rr - self.band.row0) * self.cols + cc
            self.out.index_copy_(0, slot, res["out"][:n])
            self.cz.index_copy_(0, slot, res["cz"][:n])
            self.status.index_copy_(0, slot, res["status"][:n])
            if on_block is not None:
                on_block(i)
            i += 1
        th.join()
        return i

    def gather(self, dst: int = 0):
        """The one collective: every rank's tiles to dst (parallel.py)."""
        from .parallel import gather_tiles
        return gather_tiles(self.out, dst)
