"""configs[1] at full size on the GPU (needs a B200).

The whole 32 x 32-tile batch goes through the device pipeline in the bench's
precision mode (FP16X3, fp32-class tensor cores); size-independent
properties are checked on every patch (status, finiteness, re-centring
identity) and a seeded sample of patches is checked against the oracle with
the stated tolerances (raster 1e-6 patch units, c_z 1e-3 m, refined heights
2e-3 m max on random He weights -- the fp32 bar).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import laz as olaz  # noqa: E402
from oracle import patches as opatch  # noqa: E402
from oracle import refiner as oref  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_configs1_full_batch_properties_and_sample_parity():
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.lasio import parse_header
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    from paper_2509_20198_b200.refiner import (PRECISION_FP16X3,
                                               default_descriptor,
                                               random_weights)
    side = 32
    tiles = synth.chunked_terrain_tiles(side, side, chunks_per_tile=150)
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    bundle = random_weights(default_descriptor(), seed=3)
    pipe = HeightmapPipeline(bundle, PRECISION_FP16X3)
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in tiles])
    res = pipe.run(tb, centers)
    torch.cuda.synchronize()
    P = len(centers)
    assert P == 1024
    assert not res["status"].cpu().numpy().any()
    assert not res["tri_status"].cpu().numpy().any()
    assert not res["nonfinite"].cpu().numpy().any()
    out = res["out"].cpu().numpy()
    assert np.isfinite(out).all()
    assert ((out[..., 1:] >= 0) & (out[..., 1:] <= 1)).all()
    cnn_in = res["cnn_in"].cpu().numpy()
    # re-centring: hm_lin at cell [48, 48] is exactly 0 after _finish
    assert (cnn_in[:, 48, 48, 1] == 0).all()

    index = opatch.Index()
    for t in tiles:
        r = olaz.chunk_points(t.data)
        hf = olaz.header_fields(t.data)
        index.add(olaz.positions(r, hf["scale"], hf["offset"]),
                  olaz.colors(r))
    layers = oref.text_to_layers(bundle.descriptor.to_text())
    tensors = oref.random_tensors(layers, seed=3)
    sample = np.random.default_rng(7).choice(P, 6, replace=False)
    for p in sample:
        want = opatch.reconstruct(tuple(centers[p]), index)
        assert np.array_equal(cnn_in[p, :, :, 0], want["hm_nn"]), p
        assert np.abs(cnn_in[p, :, :, 1] - want["hm_lin"]).max() <= 1e-6, p
        assert abs(float(res["cz"][p].item()) - want["c_z"]) <= 1e-3, p
        ref = oref.refine(layers, tensors, oref.stage_inputs(
            want["hm_nn"], want["hm_lin"], want["rgb_nn"],
            want["rgb_lin"])[None], [want["hm_lin"]], [want["rgb_lin"]])[0]
        assert np.abs(out[p, :, :, 0] - ref[0]).max() <= 2e-3, p
        assert np.abs(out[p, :, :, 1:4] - ref[1]).max() <= 1e-4, p


def test_tensor_core_refine_batch_invariance_at_scale():
    """Each tile's result is independent of its position in a large batch
    (different M-tile boundaries, halo splits and N-tile interleavings)."""
    from paper_2509_20198_b200.refiner import (PRECISION_FP16X3,
                                               default_descriptor,
                                               device_weights,
                                               random_weights)
    bundle = random_weights(default_descriptor(), seed=3)
    w = device_weights(bundle, PRECISION_FP16X3)
    g = torch.Generator(device="cuda").manual_seed(5)
    B = 37
    x = torch.randn((B, 96, 96, 8), generator=g, device="cuda") * 0.1
    x[..., 2:] = torch.rand((B, 96, 96, 6), generator=g, device="cuda")
    out = torch.empty((B, 64, 64, 4), device="cuda")
    nf = torch.zeros(B, dtype=torch.uint8, device="cuda")
    w.run(x, B, out, nf)
    for i in (0, 17, 36):
        o1 = torch.empty((1, 64, 64, 4), device="cuda")
        n1 = torch.zeros(1, dtype=torch.uint8, device="cuda")
        w.run(x[i:i + 1].contiguous(), 1, o1, n1)
        assert torch.equal(o1[0], out[i]), i


@pytest.mark.parametrize("precision", [0, 5])
def test_colourless_tiles_through_the_pipeline(precision):
    """Point format 0 (no RGB): the CNN sees zero colour channels
    (refiner.py:458-468) and heights still match the oracle."""
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.lasio import parse_header
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    from paper_2509_20198_b200.refiner import default_descriptor, random_weights
    tiles = synth.chunked_terrain_tiles(3, 3, chunks_per_tile=150, point_format=0)
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    bundle = random_weights(default_descriptor(), seed=3)
    pipe = HeightmapPipeline(bundle, precision)
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in tiles])
    res = pipe.run(tb, centers)
    out = res["out"].cpu().numpy()
    cnn_in = res["cnn_in"].cpu().numpy()
    assert (cnn_in[..., 2:] == 0).all()
    index = opatch.Index()
    for t in tiles:
        r = olaz.chunk_points(t.data)
        hf = olaz.header_fields(t.data)
        assert olaz.colors(r) is None
        index.add(olaz.positions(r, hf["scale"], hf["offset"]), None)
    layers = oref.text_to_layers(bundle.descriptor.to_text())
    tensors = oref.random_tensors(layers, seed=3)
    tol = 2e-3
    for p in (0, 4, 8):
        want = opatch.reconstruct(tuple(centers[p]), index)
        assert want["rgb_nn"] is None
        ref = oref.refine(layers, tensors, oref.stage_inputs(
            want["hm_nn"], want["hm_lin"], None, None)[None], [want["hm_lin"]],
            [None], has_rgb=False)[0]
        assert np.abs(out[p, :, :, 0] - ref[0]).max() <= tol, p
