"""Generate golden vectors by running the REAL reference (build container).

Run (in the container that has /root/reference):
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

It imports the unmodified reference package ``terrascout`` and records its
outputs on seeded inputs into small ``.npz`` fixtures next to this script.
The GPU box has no reference tree, so these fixtures are how the oracle
(``oracle/``) and, through it, the CUDA path are pinned to the reference.
"""

from __future__ import annotations

import hashlib
import io
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from terrascout import synth as rsynth  # noqa: E402
from terrascout.engine import bake_fullres  # noqa: E402
from terrascout.lasio import (colors, positions, read_chunk_points,  # noqa
                              scan_tile, write_laz, write_las)
from terrascout.patches import (ChunkPointIndex, PatchKey,  # noqa: E402
                                PatchSpacePoints, gather_and_normalize,
                                interpolate_patch, reconstruct_patch)
from scipy.spatial import Delaunay  # noqa: E402
from terrascout.patches import FaceMap, RawPatch  # noqa: E402
from terrascout.refiner import (ConvLayer, RefinedPatch,  # noqa
                                Upsample2, ArchDescriptor,
                                WeightBundle, conv2d, default_descriptor,
                                identity_descriptor, random_weights,
                                refine_batch, save_weights)


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


# ------------------------------------------------------------ chunk points

def gold_chunk_points(tmp):
    """Real reference-written LAZ/LAS files + read_chunk_points outputs."""
    terrain = rsynth.FractalTerrain(seed=77)
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    offsets = [(0.0, 0.0, 0.0), (712000.0, 4.1e6, -123.45)]
    for i in range(8):
        fmt = i % 4
        off = offsets[i % 2]
        n = int(rng.integers(400, 1500))
        rec = rsynth.sample_tile_records(terrain, 640.0 * i, 0.0, 640.0, n,
                                         fmt, rng, offset=off)
        path = os.path.join(tmp, f"g{i}.laz")
        if i == 5:
            sizes = [100, 300, n - 400]
            write_laz(path, rec, fmt, offset=off, chunk_sizes=sizes)
        elif i == 7:
            path = path.replace(".laz", ".las")
            write_las(path, rec, fmt, offset=off)
        else:
            write_laz(path, rec, fmt, offset=off,
                      chunk_size=int(rng.integers(60, 200)))
        cases.append(path)
    for k, path in enumerate(cases):
        tile = scan_tile(path, k)
        stride = 137 if path.endswith(".las") else 50_000
        cp = read_chunk_points(tile, las_stride=stride)
        out[f"file{k}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
        out[f"stride{k}"] = np.array(stride)
        out[f"rec{k}"] = np.frombuffer(cp.tobytes(), np.uint8)
        out[f"fmt{k}"] = np.array(tile.header.point_record_format)
        out[f"xyz{k}"] = positions(cp, tile.header)
        c = colors(cp, tile.header)
        if c is not None:
            out[f"rgb{k}"] = c
    # an 8-bit colour batch exercises the /255 branch (records.py:81-85)
    rec = rsynth.sample_tile_records(terrain, 0.0, 0.0, 640.0, 300, 2, rng)
    for ch in ("red", "green", "blue"):
        rec[ch] = rec[ch] >> 8
    path = os.path.join(tmp, "c8.laz")
    write_laz(path, rec, 2, chunk_size=10)
    tile = scan_tile(path, 0)
    cp = read_chunk_points(tile)
    k = len(cases)
    out[f"file{k}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    out[f"stride{k}"] = np.array(50_000)
    out[f"rec{k}"] = np.frombuffer(cp.tobytes(), np.uint8)
    out[f"fmt{k}"] = np.array(2)
    out[f"xyz{k}"] = positions(cp, tile.header)
    out[f"rgb{k}"] = colors(cp, tile.header)
    out["n_files"] = np.array(k + 1)
    _save("chunk_points.npz", **out)


# ------------------------------------------------------- index + Algorithm 1

def _stub_corpus(n_cols, n_rows, seed_rec=1):
    from paper_2509_20198_b200 import synth
    return synth.chunked_terrain_tiles(n_cols, n_rows, record_seed=seed_rec)


def gold_reconstruct(tmp):
    """CA13-like patches through the reference index + reconstruct_patch."""
    tiles = _stub_corpus(4, 4)
    index = ChunkPointIndex()
    out = {}
    for t, st in enumerate(tiles):
        path = os.path.join(tmp, f"s{t}.laz")
        open(path, "wb").write(st.data)
        tile = scan_tile(path, t)
        rec = read_chunk_points(tile)
        xyz = positions(rec, tile.header)
        rgb = colors(rec, tile.header)
        index.add_points(xyz, rgb)
        out[f"tile{t}"] = np.frombuffer(st.data, np.uint8)
    out["n_tiles"] = np.array(len(tiles))
    keys = [(i, j) for j in range(4) for i in range(4)]
    for p, (i, j) in enumerate(keys):
        key = PatchKey(i, j, (i * 640.0 + 320.0, j * 640.0 + 320.0))
        pts = gather_and_normalize(key, index)
        raw = reconstruct_patch(key, index)
        out[f"xy{p}"] = pts.xy
        out[f"h{p}"] = pts.h
        out[f"prgb{p}"] = pts.rgb
        out[f"cz_in{p}"] = np.array(pts.c_z)
        out[f"hm_nn{p}"] = raw.hm_nn
        out[f"hm_lin{p}"] = raw.hm_lin
        out[f"rgb_nn{p}"] = raw.rgb_nn
        out[f"rgb_lin{p}"] = raw.rgb_lin
        out[f"face{p}"] = raw.face_map.cells
        out[f"cz{p}"] = np.array(raw.key.c_z)
        corners = np.array([[-1., -1.], [1., -1.], [-1., 1.], [1., 1.]])
        out[f"simp{p}"] = Delaunay(np.vstack([pts.xy, corners])).simplices
    out["keys"] = np.array(keys)
    _save("reconstruct.npz", **out)


def gold_interpolate():
    """Random patch-space inputs + the edge cases of test_patches.py."""
    out = {}
    cases = []
    rng = np.random.default_rng(5150)
    for trial in range(6):
        n = int(rng.integers(3, 400))
        xy = rng.uniform(-1, 1, (n, 2))
        h = rng.uniform(-0.7, 0.7, n)
        rgb = rng.random((n, 3)).astype(np.float32) if trial % 2 else None
        cases.append((xy, h, rgb))
    # single point, centroid triangle, collinear, NN tie, grid-aligned point
    cases.append((np.array([[0.3, -0.2]]), np.array([0.17]), None))
    cases.append((np.array([[-0.5, -0.5], [0.5, -0.5], [0.0, 0.5]]),
                  np.array([0.0, 0.0, 1.0]), None))
    cases.append((np.stack([np.linspace(-0.7, 0.7, 5), np.zeros(5)], 1),
                  np.linspace(0, 1, 5), None))
    cases.append((np.array([[1.0, 0.0], [-1.0, 0.0]]), np.array([1., 2.]),
                  None))
    cell = -1.0 + (40 + 0.5) * (2.0 / 96)
    cases.append((np.array([[cell, cell], [0.9, 0.9], [-0.8, 0.6]]),
                  np.array([0.25, 0.0, -0.1]), None))
    for k, (xy, h, rgb) in enumerate(cases):
        pts = PatchSpacePoints(xy=xy, h=h, rgb=rgb, c_z=12.5)
        raw = interpolate_patch(pts)
        key = PatchKey(1, 2, (960.0, 1600.0))
        raw_k = interpolate_patch(pts, key=key)
        out[f"xy{k}"] = xy
        out[f"h{k}"] = h
        if rgb is not None:
            out[f"rgb{k}"] = rgb
            out[f"rgb_nn{k}"] = raw.rgb_nn
            out[f"rgb_lin{k}"] = raw.rgb_lin
        out[f"hm_nn{k}"] = raw.hm_nn
        out[f"hm_lin{k}"] = raw.hm_lin
        out[f"face{k}"] = raw.face_map.cells
        out[f"khm_lin{k}"] = raw_k.hm_lin
        out[f"khm_nn{k}"] = raw_k.hm_nn
        out[f"kcz{k}"] = np.array(raw_k.key.c_z)
        if len(xy) >= 1:
            corners = np.array([[-1., -1.], [1., -1.], [-1., 1.], [1., 1.]])
            out[f"simp{k}"] = Delaunay(np.vstack([xy, corners])).simplices
    out["n_cases"] = np.array(len(cases))
    _save("interpolate.npz", **out)


# ----------------------------------------------------------------- refiner

def small_descriptor():
    def enc(c_in):
        return [ConvLayer(c_in, 4, 3, 2, 1, "lrelu"),
                ConvLayer(4, 8, 3, 2, 1, "lrelu"),
                ConvLayer(8, 8, 3, 2, 1, "lrelu")]

    def dec():
        return [Upsample2(), ConvLayer(8, 8, 3, 1, 1, "lrelu"),
                Upsample2(), ConvLayer(8, 8, 3, 1, 1, "lrelu"),
                Upsample2(), ConvLayer(8, 8, 3, 1, 1, "lrelu")]
    stages = {"enc_hm_nn": enc(1), "enc_hm_lin": enc(1),
              "enc_rgb_nn": enc(3), "enc_rgb_lin": enc(3),
              "merge": [ConvLayer(32, 16, 1, 1, 0, "lrelu"),
                        ConvLayer(16, 8, 1, 1, 0, "lrelu")],
              "dec_height": dec(), "dec_color": dec(),
              "fuse": [ConvLayer(24, 8, 3, 1, 1, "lrelu"),
                       ConvLayer(8, 4, 3, 1, 1, "linear")]}
    d = ArchDescriptor(identity=False, stages=stages)
    d.declared_params = d.parameter_count()
    return d


def _make_raw(rng, with_rgb=True, cz=100.0):
    return RawPatch(
        key=PatchKey(0, 0, (320.0, 320.0), cz),
        hm_nn=rng.normal(0, 0.1, (96, 96)).astype(np.float32),
        hm_lin=rng.normal(0, 0.1, (96, 96)).astype(np.float32),
        rgb_nn=rng.random((96, 96, 3)).astype(np.float32)
        if with_rgb else None,
        rgb_lin=rng.random((96, 96, 3)).astype(np.float32)
        if with_rgb else None,
        face_map=FaceMap(96, np.zeros((96, 96), np.int32)),
        chunk_point_count=25)


def gold_refiner(tmp):
    out = {}
    rng = np.random.default_rng(12)
    raws = [_make_raw(rng), _make_raw(rng)]
    nc = _make_raw(rng, with_rgb=False)
    for name, desc, seed in (("small", small_descriptor(), 8),
                             ("default", default_descriptor(), 3)):
        bundle = random_weights(desc, seed=seed)
        path = os.path.join(tmp, f"{name}.lswb")
        save_weights(path, bundle)
        blob = open(path, "rb").read()
        out[f"{name}_sha"] = np.frombuffer(
            hashlib.sha256(blob).digest(), np.uint8)
        if name == "small":
            out["small_lswb"] = np.frombuffer(blob, np.uint8)
        res = refine_batch(raws, bundle)
        out[f"{name}_h"] = np.stack([r.heights_rel for r in res])
        out[f"{name}_rgb"] = np.stack([r.rgb for r in res])
        res_nc = refine_batch([nc], bundle)[0]
        out[f"{name}_nc_h"] = res_nc.heights_rel
        out[f"{name}_desc"] = np.frombuffer(
            desc.to_text().encode(), np.uint8)
    for i, r in enumerate(raws):
        out[f"in_hm_nn{i}"], out[f"in_hm_lin{i}"] = r.hm_nn, r.hm_lin
        out[f"in_rgb_nn{i}"], out[f"in_rgb_lin{i}"] = r.rgb_nn, r.rgb_lin
    out["nc_hm_nn"], out["nc_hm_lin"] = nc.hm_nn, nc.hm_lin
    ident = refine_batch(raws, WeightBundle(1, {}, identity_descriptor()))
    out["ident_h"] = np.stack([r.heights_rel for r in ident])
    out["ident_rgb"] = np.stack([r.rgb for r in ident])
    # conv2d: random small configurations (test_acceptance.py:257-301)
    crng = np.random.default_rng(99)
    for c in range(40):
        ci, co = int(crng.integers(1, 5)), int(crng.integers(1, 5))
        k = int(crng.choice([1, 3, 5]))
        st, pd = int(crng.choice([1, 2])), int(crng.choice([0, 1, 2]))
        hh, ww = int(crng.integers(k, 11)), int(crng.integers(k, 11))
        x = crng.normal(size=(ci, hh, ww)).astype(np.float32)
        w = crng.normal(size=(co, ci, k, k)).astype(np.float32)
        b = crng.normal(size=co).astype(np.float32)
        out[f"cx{c}"], out[f"cw{c}"], out[f"cb{c}"] = x, w, b
        out[f"cs{c}"] = np.array([st, pd])
        out[f"cy{c}"] = conv2d(x, w, b, stride=st, padding=pd)
    out["n_conv"] = np.array(40)
    _save("refiner.npz", **out)


# -------------------------------------------------------------------- bake

def gold_bake():
    out = {}
    terrain = rsynth.FractalTerrain(seed=11)
    rng = np.random.default_rng(3)
    keys, bases, pts_all, rgb_all = [], [], [], []
    for p, (i, j) in enumerate([(0, 0), (1, 0), (0, 1), (5, 3)]):
        x0, y0 = i * 640.0, j * 640.0
        rec = rsynth.sample_tile_records(terrain, x0, y0, 640.0, 3000, 2,
                                         rng)
        hdr = type("H", (), {"scale": (0.01,) * 3, "offset": (0.0,) * 3,
                             "color_channels_present": True})
        xyz = positions(rec, hdr)
        rgb = colors(rec, hdr)
        if p == 3:      # half-covered patch keeps prior texels
            keep = xyz[:, 0] < x0 + 320.0
            xyz, rgb = xyz[keep], rgb[keep]
        key = PatchKey(i, j, (x0 + 320.0, y0 + 320.0), c_z=50.0 + p)
        base = RefinedPatch(
            key=PatchKey(i, j, key.center, c_z=40.0 + p),
            heights_rel=rng.normal(0, 3, (64, 64)).astype(np.float32),
            rgb=rng.random((64, 64, 3)).astype(np.float32),
            provenance="refined")
        keys.append(key)
        bases.append(base)
        pts_all.append(xyz)
        rgb_all.append(rgb)
    xyz = np.concatenate(pts_all)
    rgb = np.concatenate(rgb_all)
    baked = bake_fullres(xyz, rgb, bases, keys)
    out["xyz"], out["rgb"] = xyz, rgb
    out["centers"] = np.array([k.center for k in keys])
    out["key_cz"] = np.array([k.c_z for k in keys])
    out["base_cz"] = np.array([b.key.c_z for b in bases])
    out["base_h"] = np.stack([b.heights_rel for b in bases])
    out["base_rgb"] = np.stack([b.rgb for b in bases])
    out["out_h"] = np.stack([b.heights_rel for b in baked])
    out["out_rgb"] = np.stack([b.rgb for b in baked])
    nocol = bake_fullres(xyz, None, [RefinedPatch(b.key, b.heights_rel, None,
                                                  "refined") for b in bases],
                         keys)
    out["out_h_nocol"] = np.stack([b.heights_rel for b in nocol])
    _save("bake.npz", **out)


def gold_wire():
    """server.wire_heightmap on a stand-in engine holding RefinedPatches."""
    import threading
    from terrascout.server import wire_heightmap
    rng = np.random.default_rng(2024)
    ties = ((np.arange(64 * 64 * 3) % 255 + 0.5) / 255).astype(np.float32)
    out = {}
    for name, colour in (("rgb", True), ("nocol", False)):
        eng = type("E", (), {})()
        eng.lock = threading.Lock()
        eng.refined, eng.patches = {}, {}
        recs, hs, rgbs, czs, ijs, stages = [], [], [], [], [], []
        for p, (i, j) in enumerate([(0, 0), (7, 3), (-2, 5)]):
            h = rng.normal(0, 40, (64, 64)).astype(np.float32)
            if colour:
                rgb = rng.uniform(-0.2, 1.2, (64, 64, 3)).astype(np.float32)
                if p == 2:
                    rgb = ties.reshape(64, 64, 3)      # x.5 products: half-even
            else:
                rgb = None
            cz = 100.0 + 1234.56789 * p
            stage = [3, 4, 2][p]
            eng.refined[(i, j)] = RefinedPatch(
                key=PatchKey(i, j, (i * 640.0 + 320, j * 640.0 + 320), cz),
                heights_rel=h, rgb=rgb, provenance="refined")
            eng.patches[(i, j)] = type("P", (), {"stage": stage})()
            recs.append(np.frombuffer(wire_heightmap(eng, i, j), np.uint8))
            hs.append(h)
            rgbs.append(rgb if colour else np.zeros((64, 64, 3), np.float32))
            czs.append(cz)
            ijs.append((i, j))
            stages.append(stage)
        out[f"{name}_wire"] = np.concatenate(recs)
        out[f"{name}_h"] = np.stack(hs)
        out[f"{name}_rgb"] = np.stack(rgbs)
        out[f"{name}_cz"] = np.array(czs)
        out[f"{name}_ij"] = np.array(ijs, np.int32)
        out[f"{name}_stage"] = np.array(stages, np.uint8)
    _save("wire.npz", **out)


# ------------------------------------------------------ full chunk decode

def gold_fullres(tmp):
    """Reference-compressed LAZ files (write_laz encodes every point with the
    reference's POINT10 / GPSTIME11 / RGB12 v2 encoders) and their
    load_tile_fullres records (reader.py:286-364), formats 0-3, covering the
    item coders' branches: varying returns / classes / user data / point
    source ids (changed_values), two interleaved GPS sequences with jumps,
    repeats and exact duplicates (the four-sequence GPS state), grey and
    8-bit colours (RGB byte masks), fixed and variable chunking."""
    from terrascout.lasio import load_tile_fullres
    terrain = rsynth.FractalTerrain(seed=31)
    rng = np.random.default_rng(31)
    out = {}
    k = 0
    for i in range(8):
        fmt = i % 4
        n = int(rng.integers(1500, 4000))
        rec = rsynth.sample_tile_records(terrain, 640.0 * i, 640.0, 640.0, n,
                                         fmt, rng)
        if i >= 4:
            # branchy content: per-point return/class/user/source changes
            n_ret = rng.integers(1, 4, n)
            ret = np.minimum(n_ret, rng.integers(1, 4, n))
            rec["bitfield"] = (ret | (n_ret << 3) |
                               (rng.integers(0, 2, n) << 6)).astype(np.uint8)
            rec["classification"] = rng.choice([1, 2, 3, 6, 9], n).astype(np.uint8)
            rec["user_data"] = rng.choice([0, 0, 0, 7], n).astype(np.uint8)
            rec["point_source_id"] = rng.choice([7, 7, 7, 8, 300], n).astype(np.uint16)
        if fmt in (1, 3) and i >= 4:
            # two flight lines interleaved in blocks, repeats and jumps
            t = np.where((np.arange(n) // 37) % 2 == 0,
                         1.0e5 + np.arange(n) * 1e-3,
                         3.7e5 + np.arange(n) * 7e-4)
            t[::11] = t[np.maximum(np.arange(0, n, 11) - 1, 0)]
            t[5::97] += rng.uniform(1e3, 1e5, len(t[5::97]))
            rec["gps_time"] = t.view(np.uint64)
        if fmt in (2, 3) and i >= 4:
            grey = rng.random(n) < 0.3
            for ch in ("green", "blue"):
                rec[ch] = np.where(grey, rec["red"], rec[ch])
            if i == 6:
                for ch in ("red", "green", "blue"):
                    rec[ch] = rec[ch] >> 8
        path = os.path.join(tmp, f"full{i}.laz")
        if i == 5:
            write_laz(path, rec, fmt, chunk_sizes=[400, 1, 999, n - 1400])
        else:
            write_laz(path, rec, fmt, chunk_size=int(rng.integers(500, 2500)))
        tile = scan_tile(path, i)
        full = load_tile_fullres(tile, max_workers=1)
        assert full.tobytes() == rec.tobytes()
        out[f"file{k}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
        out[f"rec{k}"] = np.frombuffer(full.tobytes(), np.uint8)
        out[f"fmt{k}"] = np.array(fmt)
        k += 1
    out["n_files"] = np.array(k)
    _save("fullres.npz", **out)


def gold_fullres_big(tmp):
    """One realistic tile for decode throughput: 4 chunks x 50,000 format-2
    points (the reference's chunk size), compressed by the reference; the
    expected records are pinned by their SHA-256 (5.2 MB raw)."""
    from terrascout.lasio import load_tile_fullres
    terrain = rsynth.FractalTerrain(seed=11)
    rng = np.random.default_rng(12)
    rec = rsynth.sample_tile_records(terrain, 0.0, 0.0, 640.0, 200_000, 2, rng)
    path = os.path.join(tmp, "big.laz")
    write_laz(path, rec, 2, chunk_size=50_000)
    full = load_tile_fullres(scan_tile(path, 0), max_workers=1)
    assert full.tobytes() == rec.tobytes()
    _save("fullres_big.npz", laz=np.frombuffer(open(path, "rb").read(), np.uint8),
          sha256=np.frombuffer(hashlib.sha256(full.tobytes()).digest(), np.uint8),
          n=np.array(len(full)))


def gold_fullres_models(tmp):
    """A chunk that creates hundreds of adaptive models: every point a new
    classification, user-data and bitfield byte (items.py:156-164 create one
    256-symbol model per previous value), format 3."""
    from terrascout.lasio import load_tile_fullres
    terrain = rsynth.FractalTerrain(seed=5)
    rng = np.random.default_rng(5)
    n = 3000
    rec = rsynth.sample_tile_records(terrain, 0.0, 0.0, 640.0, n, 3, rng)
    rec["classification"] = rng.integers(0, 256, n).astype(np.uint8)
    rec["user_data"] = rng.integers(0, 256, n).astype(np.uint8)
    rec["bitfield"] = rng.integers(0, 256, n).astype(np.uint8)
    path = os.path.join(tmp, "models.laz")
    write_laz(path, rec, 3, chunk_size=n)
    full = load_tile_fullres(scan_tile(path, 0), max_workers=1)
    assert full.tobytes() == rec.tobytes()
    _save("fullres_models.npz", laz=np.frombuffer(open(path, "rb").read(), np.uint8),
          rec=np.frombuffer(full.tobytes(), np.uint8))


def gold_render(tmp):
    """Framebuffers of the reference renderer (render.py:55-239, geometry.py
    projection / depth keys): random points (with and without colour) and
    refined heightmaps (coloured and shaded) under a top-down, an oblique
    and a close-up camera, plus resolve()."""
    from terrascout.geometry import CameraState, fit_overview
    from terrascout.patches import PatchKey
    from terrascout.refiner import RefinedPatch
    from terrascout.render import (Framebuffer, rasterize_heightmaps,
                                   rasterize_points, resolve)
    rng = np.random.default_rng(2024)
    cams = {
        "top": fit_overview((0, 0, 0), (1280, 1280, 120), (128, 96)),
        "oblique": CameraState.from_yaw_pitch((-300.0, -250.0, 420.0),
                                              np.deg2rad(40), np.deg2rad(-35),
                                              np.deg2rad(55), (160, 120)),
        "close": CameraState.from_yaw_pitch((300.0, 280.0, 95.0),
                                            np.deg2rad(15), np.deg2rad(-60),
                                            np.deg2rad(70), (200, 150),
                                            near=0.5, far=5000.0),
    }
    out = {}
    pts = np.stack([rng.uniform(-100, 1400, 30000), rng.uniform(-100, 1400, 30000),
                    rng.uniform(0, 140, 30000)], 1)
    rgb = rng.random((30000, 3)).astype(np.float32)
    out["pts"] = pts
    out["rgb"] = rgb
    patches = []
    for j in range(2):
        for i in range(2):
            c_z = float(40 + 10 * i + 5 * j)
            xs = (np.arange(64) + 0.5) * 10.0
            h = (20 * np.sin(xs[None, :] / 90.0 + i) * np.cos(xs[:, None] / 70.0 + j)
                 + rng.normal(0, 0.5, (64, 64))).astype(np.float32)
            col = rng.random((64, 64, 3)).astype(np.float32) if (i + j) % 2 == 0 else None
            key = PatchKey(i, j, (640.0 * i + 320.0, 640.0 * j + 320.0), c_z)
            patches.append(RefinedPatch(key=key, heights_rel=h, rgb=col, provenance="refined"))
            out[f"hm{2 * j + i}"] = h
            out[f"cz{2 * j + i}"] = np.array(c_z)
            out[f"key{2 * j + i}"] = np.array([i, j, 640.0 * i + 320.0, 640.0 * j + 320.0])
            if col is not None:
                out[f"col{2 * j + i}"] = col
    for name, cam in cams.items():
        out[f"cam_{name}"] = np.concatenate([cam.position, cam.direction,
                                             [cam.fov_y, cam.viewport[0], cam.viewport[1],
                                              cam.near, cam.far]])
        w, h = cam.viewport
        fb = Framebuffer(w, h)
        rasterize_points(pts, rgb, cam, fb)
        out[f"fb_pts_{name}"] = fb.cells.copy()
        fb = Framebuffer(w, h)
        rasterize_points(pts[:5000], None, cam, fb)
        out[f"fb_grey_{name}"] = fb.cells.copy()
        fb = Framebuffer(w, h)
        rasterize_heightmaps(patches, cam, fb)
        out[f"fb_hm_{name}"] = fb.cells.copy()
        rasterize_points(pts, rgb, cam, fb)
        out[f"fb_both_{name}"] = fb.cells.copy()
        out[f"img_{name}"] = resolve(fb)
    _save("render.npz", **out)


def gold_engine(tmp):
    """The reference ScoutEngine end to end on a 3 x 3 corpus of real
    (reference-compressed) LAZ tiles, like tests/conftest.py small_dataset:
    (A) overview camera, random seed-3 bundle, batch_max 64 -- configs[0]'s
    driver; (B) the close-up of test_baked_patches_survive_eviction with
    the identity bundle -- tile loads (full chunk decode), bakes, eviction.
    Records priorities, task counts, stages, ready events and every refined
    patch."""
    import glob

    from terrascout.engine import Dataset, EngineConfig, ScoutEngine, Stage
    from terrascout.geometry import CameraState
    from terrascout.synth import FractalTerrain, generate_corpus
    d = os.path.join(tmp, "engine_corpus")
    generate_corpus(d, n_tiles=9, points_per_tile=4000, seed=11, point_format=2,
                    chunk_size=250, terrain=FractalTerrain(seed=11))
    paths = sorted(glob.glob(os.path.join(d, "*.laz")))
    out = {"n_files": np.array(len(paths))}
    for k, pth in enumerate(paths):
        out[f"file{k}"] = np.frombuffer(open(pth, "rb").read(), np.uint8)
        out[f"name{k}"] = np.array(os.path.basename(pth))

    def record(tag, eng, n_tasks, pre_prio):
        pids = sorted(eng.patches)
        out[f"{tag}_pids"] = np.array(pids, np.int64)
        out[f"{tag}_prio"] = np.array([pre_prio[p] for p in pids])
        out[f"{tag}_stage"] = np.array([int(eng.patches[p].stage) for p in pids])
        out[f"{tag}_nodata"] = np.array([eng.patches[p].no_data for p in pids])
        out[f"{tag}_tasks"] = np.array(n_tasks)
        out[f"{tag}_events"] = np.array([(i, j, int(s)) for (i, j), s in eng.ready_events],
                                        np.int64).reshape(-1, 3)
        for p in pids:
            r = eng.refined.get(p)
            if r is not None:
                out[f"{tag}_h_{p[0]}_{p[1]}"] = r.heights_rel
                out[f"{tag}_prov_{p[0]}_{p[1]}"] = np.array(r.provenance)
                if r.rgb is not None:
                    out[f"{tag}_rgb_{p[0]}_{p[1]}"] = r.rgb
        out[f"{tag}_tile_state"] = np.array([int(eng.tiles[t].state) for t in sorted(eng.tiles)])
        out[f"{tag}_tile_wanted"] = np.array([eng.tiles[t].wanted for t in sorted(eng.tiles)])

    ds = Dataset.scan(paths)
    eng = ScoutEngine(ds, EngineConfig(batch_max=64), random_weights(default_descriptor(), seed=3))
    eng.load_overview()
    prio = {p: s.priority for p, s in eng.patches.items()}
    n = eng.run_until_idle()
    record("A", eng, n, prio)

    ds = Dataset.scan(paths)
    eng = ScoutEngine(ds)
    eng.load_overview()
    t = ds.tiles[4]
    cx = (t.header.bbox_min[0] + t.header.bbox_max[0]) / 2
    cy = (t.header.bbox_min[1] + t.header.bbox_max[1]) / 2
    cam = CameraState(position=np.array([cx, cy, 100.0]), direction=np.array([0.0, 0.3, -0.95]),
                      fov_y=np.deg2rad(60), viewport=(800, 600), near=0.5, far=10000.0)
    out["B_cam"] = np.concatenate([cam.position, cam.direction,
                                   [cam.fov_y, 800, 600, 0.5, 10000.0]])
    eng.update_viewpoint(cam)
    prio = {p: s.priority for p, s in eng.patches.items()}
    out["B_tile_prio"] = np.array([eng.tiles[t].priority for t in sorted(eng.tiles)])
    n = eng.run_until_idle()
    assert any(s.stage == Stage.FULLRES_BAKED for s in eng.patches.values())
    record("B", eng, n, prio)
    _save("engine.npz", **out)


if __name__ == "__main__":
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        if len(sys.argv) > 1:  # only the named fixtures
            for name in sys.argv[1:]:
                f = globals()[f"gold_{name}"]
                f(tmp) if f.__code__.co_argcount else f()
            sys.exit(0)
        gold_fullres(tmp)
        gold_fullres_big(tmp)
        gold_fullres_models(tmp)
        gold_render(tmp)
        gold_engine(tmp)
        gold_chunk_points(tmp)
        gold_reconstruct(tmp)
        gold_interpolate()
        gold_refiner(tmp)
        gold_bake()
        gold_wire()
