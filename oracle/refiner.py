"""Oracle: descriptor-driven refiner CNN in numpy float32.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``pkg/src/terrascout/refiner.py``: the topology of ``_Forward.run``
(``:430-441``), ``_conv_batched`` as im2col + float32 matmul (``:330-380``),
leaky ReLU / nearest up2 (``:391-396``), ``refine_batch`` crop, non-finite
fallback and colour clamp (``:475-528``), He-init ``random_weights``
(``:314-327``) and the LSWB container (``:258-311``).
"""

from __future__ import annotations

import struct

import numpy as np

STAGES = ("enc_hm_nn", "enc_hm_lin", "enc_rgb_nn", "enc_rgb_lin",
          "merge", "dec_height", "dec_color", "fuse")
CROP = 16


def default_layers():
    """Stage -> list of ("conv", ci, co, k, s, p, act) / ("up2",)."""
    def enc(ci):
        return [("conv", ci, 48, 3, 2, 1, "lrelu"),
                ("conv", 48, 96, 3, 2, 1, "lrelu"),
                ("conv", 96, 192, 3, 2, 1, "lrelu")]

    def dec():
        return [("up2",), ("conv", 320, 96, 3, 1, 1, "lrelu"),
                ("up2",), ("conv", 96, 64, 3, 1, 1, "lrelu"),
                ("up2",), ("conv", 64, 32, 3, 1, 1, "lrelu")]
    return {"enc_hm_nn": enc(1), "enc_hm_lin": enc(1),
            "enc_rgb_nn": enc(3), "enc_rgb_lin": enc(3),
            "merge": [("conv", 768, 768, 1, 1, 0, "lrelu"),
                      ("conv", 768, 320, 1, 1, 0, "lrelu")],
            "dec_height": dec(), "dec_color": dec(),
            "fuse": [("conv", 72, 64, 3, 1, 1, "lrelu"),
                     ("conv", 64, 32, 3, 1, 1, "lrelu"),
                     ("conv", 32, 4, 3, 1, 1, "linear")]}


def layers_to_text(layers) -> str:
    n = sum(l[2] * l[1] * l[3] ** 2 + l[2] for st in layers.values()
            for l in st if l[0] == "conv")
    out = ["arch 1", f"params {n}"]
    for s in STAGES:
        out.append(f"stage {s}")
        for l in layers[s]:
            out.append("up2" if l[0] == "up2" else
                       "conv " + " ".join(str(v) for v in l[1:]))
    return "\n".join(out) + "\n"


def text_to_layers(text: str):
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()
             and not ln.startswith("#")]
    if len(lines) > 1 and lines[1] == "identity":
        return None
    layers, cur = {}, None
    for ln in lines[1:]:
        p = ln.split()
        if p[0] == "stage":
            cur = layers.setdefault(p[1], [])
        elif p[0] == "up2":
            cur.append(("up2",))
        elif p[0] == "conv":
            cur.append(("conv", int(p[1]), int(p[2]), int(p[3]), int(p[4]),
                        int(p[5]), p[6]))
    return layers


def random_tensors(layers, seed=0):
    rng = np.random.default_rng(seed)
    t = {}
    for s in STAGES:
        for li, l in enumerate(layers[s]):
            if l[0] != "conv":
                continue
            _, ci, co, k = l[:4]
            # shape order of tensor_shapes(): weight then bias per layer
            t[f"{s}.{li}.weight"] = rng.normal(
                0, np.sqrt(2.0 / (ci * k * k)), (co, ci, k, k)).astype(
                np.float32)
            t[f"{s}.{li}.bias"] = np.zeros(co, np.float32)
    return t


def read_lswb(blob: bytes):
    """(tensors, descriptor_text); refiner.py:275-311 without validation."""
    assert blob[:4] == b"LSWB"
    _ver, n = struct.unpack_from("<II", blob, 4)
    off, tensors = 12, {}
    for _ in range(n):
        ln, = struct.unpack_from("<H", blob, off)
        name = blob[off + 2:off + 2 + ln].decode()
        off += 2 + ln
        rank = blob[off]
        dims = struct.unpack_from(f"<{rank}I", blob, off + 1)
        off += 1 + 4 * rank
        cnt = int(np.prod(dims)) if rank else 1
        tensors[name] = np.frombuffer(blob, "<f4", cnt, off).reshape(
            dims).copy()
        off += 4 * cnt
    dl, = struct.unpack_from("<I", blob, off)
    return tensors, blob[off + 4:off + 4 + dl].decode()


def conv(x, w, b, stride=1, pad=0):
    """B,C,H,W float32 cross-correlation via im2col + float32 matmul."""
    bsz, ci, hh, ww = x.shape
    co, _, kh, kw = w.shape
    if pad:
        x = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    ho = (hh + 2 * pad - kh) // stride + 1
    wo = (ww + 2 * pad - kw) // stride + 1
    wm = w.reshape(co, -1)
    out = np.empty((bsz, co, ho * wo), np.float32)
    for s in range(bsz):
        cols = np.empty((ci, kh, kw, ho, wo), np.float32)
        for dy in range(kh):
            for dx in range(kw):
                cols[:, dy, dx] = x[s, :, dy:dy + stride * ho:stride,
                                    dx:dx + stride * wo:stride]
        out[s] = wm @ cols.reshape(ci * kh * kw, ho * wo) + b[:, None]
    return out.reshape(bsz, co, ho, wo)


def forward(layers, tensors, inputs):
    """inputs: B x 8 x 96 x 96 float32 -> B x 4 x 96 x 96."""
    def stage(name, x):
        for li, l in enumerate(layers[name]):
            if l[0] == "up2":
                x = x.repeat(2, axis=2).repeat(2, axis=3)
                continue
            x = conv(x, tensors[f"{name}.{li}.weight"],
                     tensors[f"{name}.{li}.bias"], l[4], l[5])
            if l[6] == "lrelu":
                x = np.where(x >= 0, x, np.float32(0.01) * x)
        return x
    feats = [stage("enc_hm_nn", inputs[:, 0:1]),
             stage("enc_hm_lin", inputs[:, 1:2]),
             stage("enc_rgb_nn", inputs[:, 2:5]),
             stage("enc_rgb_lin", inputs[:, 5:8])]
    merged = stage("merge", np.concatenate(feats, axis=1))
    return stage("fuse", np.concatenate(
        [inputs, stage("dec_height", merged), stage("dec_color", merged)],
        axis=1))


def stage_inputs(hm_nn, hm_lin, rgb_nn, rgb_lin):
    """_staging_copy (refiner.py:458-468) for one patch."""
    x = np.zeros((8, 96, 96), np.float32)
    x[0], x[1] = hm_nn, hm_lin
    if rgb_nn is not None:
        x[2:5] = rgb_nn.transpose(2, 0, 1)
        x[5:8] = rgb_lin.transpose(2, 0, 1)
    return x


def refine(layers, tensors, batch, hm_lin, rgb_lin, has_rgb=True):
    """refine_batch numerics: list of (heights_rel, rgb|None, refined?)."""
    c = slice(CROP, CROP + 64)
    out = []
    if layers is None:                       # identity bundle
        for i in range(len(batch)):
            rgb = None if not has_rgb else np.clip(rgb_lin[i][c, c], 0, 1)
            out.append(((hm_lin[i][c, c] * np.float32(480.0)).astype(
                np.float32), rgb, True))
        return out
    fused = forward(layers, tensors, batch)
    for i in range(len(batch)):
        cr = fused[i][:, c, c]
        if not np.isfinite(cr).all():
            rgb = rgb_lin[i][c, c] if has_rgb else None
            out.append(((hm_lin[i][c, c] * np.float32(480.0)).astype(
                np.float32), rgb, False))
            continue
        rgb = np.clip(cr[1:4].transpose(1, 2, 0), 0.0, 1.0) if has_rgb \
            else None
        out.append(((cr[0] * np.float32(480.0)).astype(np.float32), rgb,
                    True))
    return out
