"""The CPU oracle reproduces the reference's own outputs (golden vectors).

CPU-only.  Fixtures come from ``tests/golden/make_golden.py`` run against
the unmodified reference.  Passing here is what makes the oracle a valid
checker for the CUDA path in the ``-m gpu`` tests.
"""

import hashlib

import numpy as np

from oracle import bake as obake
from oracle import laz as olaz
from oracle import patches as opatch
from oracle import refiner as oref


def test_chunk_points_bit_exact(golden):
    g = golden("chunk_points.npz")
    for k in range(int(g["n_files"])):
        img = g[f"file{k}"].tobytes()
        rec = olaz.chunk_points(img, las_stride=int(g[f"stride{k}"]))
        assert rec.tobytes() == g[f"rec{k}"].tobytes(), k
        h = olaz.header_fields(img)
        xyz = olaz.positions(rec, h["scale"], h["offset"])
        assert np.array_equal(xyz, g[f"xyz{k}"]), k
        if f"rgb{k}" in g:
            assert np.array_equal(olaz.colors(rec), g[f"rgb{k}"]), k


def test_index_gather_and_reconstruct(golden):
    g = golden("reconstruct.npz")
    index = opatch.Index()
    for t in range(int(g["n_tiles"])):
        img = g[f"tile{t}"].tobytes()
        rec = olaz.chunk_points(img)
        h = olaz.header_fields(img)
        index.add(olaz.positions(rec, h["scale"], h["offset"]),
                  olaz.colors(rec))
    for p, (i, j) in enumerate(g["keys"]):
        center = (i * 640.0 + 320.0, j * 640.0 + 320.0)
        xy, hh, rgb, cz = opatch.gather(center, index)
        assert np.array_equal(xy, g[f"xy{p}"])
        assert np.array_equal(hh, g[f"h{p}"])
        assert np.array_equal(rgb, g[f"prgb{p}"])
        assert cz == float(g[f"cz_in{p}"])
        out = opatch.interpolate(xy, hh, rgb, cz, key_center=center,
                                 flood=(p < 2))
        for name in ("hm_nn", "hm_lin", "rgb_nn", "rgb_lin"):
            assert np.array_equal(out[name], g[f"{name}{p}"]), (p, name)
        assert np.array_equal(out["face"], g[f"face{p}"]), p
        assert out["c_z"] == float(g[f"cz{p}"])


def test_interpolate_cases(golden):
    g = golden("interpolate.npz")
    for k in range(int(g["n_cases"])):
        xy, hh = g[f"xy{k}"], g[f"h{k}"]
        rgb = g[f"rgb{k}"] if f"rgb{k}" in g else None
        out = opatch.interpolate(xy, hh, rgb, 12.5, flood=(k % 3 == 0))
        assert np.array_equal(out["hm_nn"], g[f"hm_nn{k}"]), k
        assert np.array_equal(out["hm_lin"], g[f"hm_lin{k}"]), k
        assert np.array_equal(out["face"], g[f"face{k}"]), k
        if rgb is not None:
            assert np.array_equal(out["rgb_lin"], g[f"rgb_lin{k}"]), k
        outk = opatch.interpolate(xy, hh, rgb, 12.5, key_center=(960., 1600.))
        assert np.array_equal(outk["hm_lin"], g[f"khm_lin{k}"]), k
        assert outk["c_z"] == float(g[f"kcz{k}"]), k


def test_refiner_weights_and_outputs(golden):
    g = golden("refiner.npz")
    # LSWB container + He init reproduce the reference byte for byte
    blob = g["small_lswb"].tobytes()
    tensors, text = oref.read_lswb(blob)
    assert text == g["small_desc"].tobytes().decode()
    layers = oref.text_to_layers(text)
    mine = oref.random_tensors(layers, seed=8)
    for k, v in tensors.items():
        assert np.array_equal(mine[k], v), k
    inputs = np.stack([oref.stage_inputs(g[f"in_hm_nn{i}"], g[f"in_hm_lin{i}"],
                                         g[f"in_rgb_nn{i}"],
                                         g[f"in_rgb_lin{i}"])
                       for i in range(2)])
    hm_lin = [g[f"in_hm_lin{i}"] for i in range(2)]
    rgb_lin = [g[f"in_rgb_lin{i}"] for i in range(2)]
    for name, seed in (("small", 8), ("default", 3)):
        layers = oref.text_to_layers(g[f"{name}_desc"].tobytes().decode())
        t = oref.random_tensors(layers, seed=seed)
        res = oref.refine(layers, t, inputs, hm_lin, rgb_lin)
        h = np.stack([r[0] for r in res])
        c = np.stack([r[1] for r in res])
        # same algorithm, different BLAS blocking: fp32 rounding only
        assert np.abs(h - g[f"{name}_h"]).max() < 1e-3, name
        assert np.abs(c - g[f"{name}_rgb"]).max() < 1e-5, name
    ident = oref.refine(None, None, inputs, hm_lin, rgb_lin)
    assert np.array_equal(np.stack([r[0] for r in ident]), g["ident_h"])
    assert np.array_equal(np.stack([r[1] for r in ident]), g["ident_rgb"])


def test_default_bundle_hash(golden):
    """random_weights(default_descriptor(), 3) -> identical LSWB bytes."""
    g = golden("refiner.npz")
    text = g["default_desc"].tobytes().decode()
    layers = oref.text_to_layers(text)
    from paper_2509_20198_b200.refiner import lswb_bytes
    blob = lswb_bytes(oref.random_tensors(layers, seed=3), text)
    assert hashlib.sha256(blob).digest() == g["default_sha"].tobytes()


def test_conv_cases(golden):
    g = golden("refiner.npz")
    for c in range(int(g["n_conv"])):
        st, pd = g[f"cs{c}"]
        y = oref.conv(g[f"cx{c}"][None], g[f"cw{c}"], g[f"cb{c}"], int(st),
                      int(pd))[0]
        assert np.abs(y - g[f"cy{c}"]).max() < 1e-5, c


def test_bake(golden):
    g = golden("bake.npz")
    for p in range(len(g["centers"])):
        h, c = obake.bake_one(g["xyz"], g["rgb"], g["base_h"][p],
                              float(g["base_cz"][p]), g["base_rgb"][p],
                              g["centers"][p], float(g["key_cz"][p]))
        assert np.array_equal(h, g["out_h"][p]), p
        assert np.array_equal(c, g["out_rgb"][p]), p
        h2, _ = obake.bake_one(g["xyz"], None, g["base_h"][p],
                               float(g["base_cz"][p]), None,
                               g["centers"][p], float(g["key_cz"][p]))
        assert np.array_equal(h2, g["out_h_nocol"][p]), p


def test_wire_records(golden):
    """oracle.wire vs the reference's server.wire_heightmap bytes (colour,
    clipping, half-to-even ties, negative grid indices, colourless)."""
    from oracle import wire as owire
    g = golden("wire.npz")
    for name, colour in (("rgb", True), ("nocol", False)):
        recs = b"".join(
            owire.wire_record(int(g[f"{name}_ij"][p][0]), int(g[f"{name}_ij"][p][1]),
                              float(g[f"{name}_cz"][p]), int(g[f"{name}_stage"][p]),
                              g[f"{name}_h"][p], g[f"{name}_rgb"][p] if colour else None)
            for p in range(len(g[f"{name}_cz"])))
        assert recs == g[f"{name}_wire"].tobytes(), name


def test_oracle_full_chunk_decode_matches_reference(golden):
    """oracle.lazdec restates decode_chunk + the POINT10 / GPSTIME11 /
    RGB12 v2 item decoders: bit-exact with the reference's
    load_tile_fullres on reference-compressed files (formats 0-3)."""
    from oracle import lazdec
    g = golden("fullres.npz")
    for k in range(int(g["n_files"])):
        rec = lazdec.load_fullres(g[f"file{k}"].tobytes())
        assert rec.tobytes() == g[f"rec{k}"].tobytes(), k


def _render_scene(g):
    from oracle import render as orender
    patches = []
    for k in range(4):
        key = g[f"key{k}"]
        patches.append((g[f"hm{k}"], g[f"col{k}"] if f"col{k}" in g else None,
                        (float(key[2]), float(key[3])), float(g[f"cz{k}"])))
    return orender, patches


def test_oracle_render_matches_reference(golden):
    """oracle.render restates render.py / geometry.py projection with the
    same numpy expressions: framebuffers bit-identical to the reference."""
    g = golden("render.npz")
    orender, patches = _render_scene(g)
    for name in ("top", "oblique", "close"):
        cam = orender.Camera(g[f"cam_{name}"])
        w, h = cam.viewport
        fb = orender.new_fb(w, h)
        orender.rasterize_points(g["pts"], g["rgb"], cam, fb)
        assert np.array_equal(fb, g[f"fb_pts_{name}"]), name
        fb = orender.new_fb(w, h)
        orender.rasterize_points(g["pts"][:5000], None, cam, fb)
        assert np.array_equal(fb, g[f"fb_grey_{name}"]), name
        fb = orender.new_fb(w, h)
        orender.rasterize_heightmaps(patches, cam, fb)
        assert np.array_equal(fb, g[f"fb_hm_{name}"]), name
        orender.rasterize_points(g["pts"], g["rgb"], cam, fb)
        assert np.array_equal(fb, g[f"fb_both_{name}"]), name
        assert np.array_equal(orender.resolve(fb), g[f"img_{name}"]), name
