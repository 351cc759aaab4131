"""configs[2] at full scale (needs a B200): 200 M points into 4,096
heightmaps, grouped by patch and shuffled.

Size-independent properties on the whole batch: the fixed-point sums make
the result independent of point order (grouped == shuffled, bit for bit)
and covered texels change while uncovered ones keep the prior.  A seeded
sample of patches is checked against the oracle's bincount bake
(engine.py:416-456) on that patch's points: heights within 1e-6 m, rgb
within 1e-6.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_configs2_full_scale_grouped_shuffled_and_sampled_oracle():
    import bench
    from oracle import bake as obake
    from paper_2509_20198_b200._lib import lib
    from paper_2509_20198_b200.engine import bake_device, key_grid
    dev = torch.device("cuda", 0)
    xyz, rgb, centers, per = bench.splat_inputs(200_000_000, dev)
    P, M = len(centers), len(xyz)
    assert P == 4096 and M >= 199_000_000
    g = torch.Generator(device=dev).manual_seed(9)
    prior = torch.rand((P, 64, 64), generator=g, device=dev) * 10
    prior_rgb = torch.rand((P, 64, 64, 3), generator=g, device=dev)
    base_cz = torch.full((P,), 50.0, dtype=torch.float64, device=dev)
    key_cz = torch.full((P,), 47.5, dtype=torch.float64, device=dev)
    grid = key_grid(centers)
    accum = torch.empty(int(lib().ts_bake_workspace(P)), dtype=torch.uint8, device=dev)
    h1, c1 = bake_device(xyz, rgb, centers, prior, base_cz, key_cz, prior_rgb, grid, accum)
    h1, c1 = h1.clone(), c1.clone()
    rng = np.random.default_rng(4)
    sample = rng.choice(P, 6, replace=False)
    # a patch's window also catches neighbours' points rounded onto its
    # edge: hand the oracle the points of the 3 x 3 patch neighbourhood
    side = int(round(P ** 0.5))
    pts = {}
    for p in sample:
        nb = [q for q in (p + dy * side + dx for dy in (-1, 0, 1) for dx in (-1, 0, 1))
              if 0 <= q < P]
        pts[int(p)] = (np.concatenate([xyz[q * per:(q + 1) * per].cpu().numpy() for q in nb]),
                       np.concatenate([rgb[q * per:(q + 1) * per].cpu().numpy() for q in nb]))
    perm = torch.randperm(M, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
    xs, rs = xyz[perm], rgb[perm]
    del xyz, rgb, perm
    h2, c2 = bake_device(xs, rs, centers, prior, base_cz, key_cz, prior_rgb, grid, accum)
    torch.cuda.synchronize()
    assert torch.equal(h1, h2) and torch.equal(c1, c2)
    # every texel is covered at ~12 points per texel
    assert (h1.cpu().numpy() != (prior.double() + 50.0 - 47.5).float().cpu().numpy()).mean() > 0.99
    hh, cc = h1.cpu().numpy(), c1.cpu().numpy()
    pr, prc = prior.cpu().numpy(), prior_rgb.cpu().numpy()
    for p, (px, pc) in pts.items():
        want_h, want_c = obake.bake_one(px, pc, pr[p], 50.0, prc[p],
                                        tuple(centers[p]), 47.5)
        assert np.abs(hh[p] - want_h).max() <= 1e-6, p
        assert np.abs(cc[p] - want_c).max() <= 1e-6, p
