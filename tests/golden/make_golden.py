"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container only (it imports ``fasthog`` from the read-only
reference checkout, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes ``tests/golden/lut_sha256.json`` and ``tests/golden/golden.npz``.
Both are committed; tests pin the oracle (and through it the CUDA path)
against them without needing the reference at run time.  Inputs are seeded
so every case can be regenerated bit-for-bit from the recipe below.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, REF)

import fasthog as fh  # noqa: E402  (the reference)

from paper_1703_06256_b200 import synth  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def image_cases():
    """(name, planes, bins) small seeded images covering gray/RGB/odd sizes."""
    rng = np.random.default_rng(20260101)
    cases = [
        ("gray45x37", rng.integers(0, 256, (1, 37, 45), dtype=np.uint8), 9),
        ("rgb48x40", rng.integers(0, 256, (3, 40, 48), dtype=np.uint8), 9),
        ("gray133x77", rng.integers(0, 256, (1, 77, 133), dtype=np.uint8), 8),
        ("rgb3x3", rng.integers(0, 256, (3, 3, 3), dtype=np.uint8), 4),
        ("gray300x200_b18", rng.integers(0, 256, (1, 200, 300), dtype=np.uint8), 18),
    ]
    # identical channels (tie rule) and a blurred config-like frame
    p = rng.integers(0, 256, (1, 50, 70), dtype=np.uint8)
    cases.append(("rgbtie70x50", np.concatenate([p, p, p]), 9))
    cfg = synth.CONFIGS["c2"]
    cases.append(("c2frame0_crop", synth.make_frame(cfg, 0)[:, :160, :200].copy(), 8))
    return cases


def main():
    out = {}
    lut_hash = {}
    for n in range(fh.gradient.MIN_BINS, fh.gradient.MAX_BINS + 1):
        lut_hash[str(n)] = sha(fh.build_lut(n).table.astype("<i2"))
    with open(os.path.join(HERE, "lut_sha256.json"), "w") as f:
        json.dump(lut_hash, f, indent=1, sort_keys=True)
    for n in (8, 9):
        out[f"lut{n}"] = fh.build_lut(n).table.astype(np.int8)

    geoms = {
        "g16b2": fh.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=9),
        "g16x24": fh.DescriptorGeometry(16, 24, 8, block=2, block_stride=1, bins=9),
    }
    for name, planes, bins in image_cases():
        img = fh.Image(planes)
        lut = fh.build_lut(bins)
        bm = fh.gradient_map(img, lut)
        st = fh.build_integral_stack(bm)
        out[f"{name}/image"] = planes
        out[f"{name}/bins"] = np.array(bins)
        out[f"{name}/binmap"] = bm.cells
        if st.planes.size <= 200_000:
            out[f"{name}/planes"] = st.planes
        out[f"{name}/planes_sha"] = np.array(sha(st.planes))
        H, W = bm.height, bm.width
        for gname, g0 in geoms.items():
            if g0.bins != bins or g0.window_w > W or g0.window_h > H:
                continue
            for norm in ("none", "l1", "l2"):
                g = fh.DescriptorGeometry(g0.window_w, g0.window_h, g0.cell, g0.block,
                                          g0.block_stride, g0.bins, norm)
                for stride in (1, 3, 8):
                    key = f"{name}/{gname}/{norm}/s{stride}"
                    oxs, oys = fh.window_origins(W, H, g, stride)
                    cache = fh.CellHistogramCache(st, g, oxs, oys)
                    descs = np.stack([d for _, _, d in fh.scan_descriptors(st, g, stride)])
                    if norm == "none":
                        out[f"{key}/grid"] = cache.grid
                    if descs.size <= 60_000:
                        out[f"{key}/descs"] = descs
                    out[f"{key}/descs_sha"] = np.array(sha(descs))
            # scores through scan() with seeded weights
            g = g0
            wrng = np.random.default_rng(77)
            model = fh.LinearModel(g, wrng.normal(size=fh.descriptor_length(g)), 0.125)
            for stride in (2, 4):
                dets = fh.scan(st, model, stride, float("-inf"))
                out[f"{name}/{gname}/scan_s{stride}/xy"] = np.array(
                    [(d.x, d.y) for d in dets], dtype=np.int64)
                out[f"{name}/{gname}/scan_s{stride}/score"] = np.array(
                    [d.score for d in dets], dtype=np.float64)
                out[f"{name}/{gname}/weights"] = model.weights
        # block=1 BASELINE-style geometry on the larger images (cell 8, 16x32 window)
        if W >= 64 and H >= 64:
            for norm in ("none", "l2"):
                g = fh.DescriptorGeometry(16, 32, 8, block=1, block_stride=1, bins=bins,
                                          normalization=norm)
                for stride in (4, 8):
                    key = f"{name}/b1_{norm}/s{stride}"
                    oxs, oys = fh.window_origins(W, H, g, stride)
                    cache = fh.CellHistogramCache(st, g, oxs, oys)
                    if norm == "none":
                        out[f"{key}/grid"] = cache.grid
                    wrng = np.random.default_rng(99)
                    model = fh.LinearModel(g, wrng.normal(0, 0.01, fh.descriptor_length(g)), 0.0)
                    dets = fh.scan(st, model, stride, float("-inf"))
                    out[f"{key}/score"] = np.array([d.score for d in dets])
                    out[f"{key}/weights"] = model.weights

    # config c1 at full size: hashes of every stage and the score map
    cfg = synth.CONFIGS["c1"]
    frame = synth.make_frame(cfg, 0)
    w, bias = synth.make_weights(cfg)
    g = fh.DescriptorGeometry(64, 128, 8, block=1, block_stride=1, bins=cfg.bins)
    bm = fh.gradient_map(fh.Image(frame), fh.build_lut(cfg.bins))
    st = fh.build_integral_stack(bm)
    oxs, oys = fh.window_origins(cfg.width, cfg.height, g, cfg.stride)
    cache = fh.CellHistogramCache(st, g, oxs, oys)
    dets = fh.scan(st, fh.LinearModel(g, w, bias), cfg.stride, float("-inf"))
    out["c1/frame_sha"] = np.array(sha(frame))
    out["c1/binmap_sha"] = np.array(sha(bm.cells))
    out["c1/planes_sha"] = np.array(sha(st.planes))
    out["c1/grid_sha"] = np.array(sha(cache.grid))
    out["c1/scores"] = np.array([d.score for d in dets]).reshape(len(oys), len(oxs))

    # bilinear resize (detector.py:202-221) and the pyramid level loop
    rng = np.random.default_rng(4242)
    src = rng.integers(0, 256, (3, 83, 97), dtype=np.uint8)
    out["resize/src"] = src
    for (nw, nh) in ((80, 69), (40, 33), (97, 83), (13, 7), (96, 82)):
        out[f"resize/{nw}x{nh}"] = fh.detector._resize_bilinear(fh.Image(src), nw, nh).planes
    big = synth.make_frame(synth.CONFIGS["c5"], 0)[:, :540, :960].copy()
    out["resize_big/src_sha"] = np.array(sha(big))
    for (nw, nh) in ((800, 450), (666, 375), (555, 312)):
        out[f"resize_big/{nw}x{nh}_sha"] = np.array(
            sha(fh.detector._resize_bilinear(fh.Image(big), nw, nh).planes))

    g = fh.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=9)
    pimg = np.random.default_rng(515).integers(0, 256, (1, 61, 83), dtype=np.uint8)
    model = fh.LinearModel(g, np.random.default_rng(516).normal(size=36), -0.5)
    dets = fh.pyramid_scan(fh.Image(pimg), model, 1.3, 4, float("-inf"))
    out["pyramid/image"] = pimg
    out["pyramid/weights"] = model.weights
    out["pyramid/boxes"] = np.array([(d.x, d.y, d.w, d.h) for d in dets], dtype=np.int64)
    out["pyramid/score"] = np.array([d.score for d in dets])
    out["pyramid/scale"] = np.array([d.scale for d in dets])

    # threshold + greedy NMS (detector.py:145-153, 285-299) on the pyramid hits
    for thr in (0.0, 1.5):
        hits = fh.pyramid_scan(fh.Image(pimg), model, 1.3, 4, thr)
        out[f"pyramid_thr{thr}/boxes"] = np.array([(d.x, d.y, d.w, d.h) for d in hits],
                                                   dtype=np.int64).reshape(-1, 4)
        out[f"pyramid_thr{thr}/score"] = np.array([d.score for d in hits])
        out[f"pyramid_thr{thr}/scale"] = np.array([d.scale for d in hits])
    pos = {id(d): i for i, d in enumerate(dets)}
    for iou_t in (0.0, 0.3, 0.5, 1.0):
        out[f"nms/pyramid/{iou_t}"] = np.array([pos[id(d)] for d in fh.nms(dets, iou_t)],
                                               dtype=np.int64)
    # random integer boxes with tied scores, tied (y, x) and several scales
    rng = np.random.default_rng(777)
    k = 1500
    rb = np.stack([rng.integers(0, 300, k), rng.integers(0, 200, k),
                   rng.integers(8, 120, k), rng.integers(8, 160, k)], 1)
    rb[k // 2:, :2] = rb[: k - k // 2, :2]  # duplicate origins: ties broken by scale
    rs = np.round(rng.normal(0, 1, k), 1)   # many equal scores
    rc = rng.choice([1.0, 1.2, 1.44], k)
    rdets = [fh.Detection(int(b[0]), int(b[1]), int(b[2]), int(b[3]), float(s_), float(c))
             for b, s_, c in zip(rb, rs, rc)]
    out["nms/random/boxes"] = rb.astype(np.int64)
    out["nms/random/score"] = rs
    out["nms/random/scale"] = rc
    rpos = {id(d): i for i, d in enumerate(rdets)}
    for iou_t in (0.0, 0.2, 0.45, 0.8, 1.0):
        out[f"nms/random/{iou_t}"] = np.array([rpos[id(d)] for d in fh.nms(rdets, iou_t)],
                                              dtype=np.int64)

    # PNM wire format (image_io.py:50-122): decoded planes or the error class
    pnm_cases = {
        "p5": b"P5\n7 5\n255\n" + bytes(range(35)),
        "p6": b"P6 4 3 255\n" + bytes((7 * i) % 256 for i in range(36)),
        "p2_comments": b"P2\n# a comment\n3 2 # trailing\n255\n0 1 2\n\t 253\r254 255\n",
        "p3": b"P3 2 2 255 1 2 3 4 5 6 7 8 9 10 11 12",
        "p5_trailing": b"P5 2 2 255 abcdXYZ",
        "p5_hash_after_maxval": b"P5 2 1 255#xy",
        "p2_underscore_plus": b"P2 2 1 2_55 +7 0_0_1",
        "p2_leading_zeros": b"P2 0002 001 0255 007 255",
        "bad_magic": b"P4\n1 1\n255\n\x00",
        "maxval_16bit": b"P5 1 1 65535 \x00\x00",
        "maxval_zero": b"P5 1 1 0 \x00",
        "truncated_raw": b"P6 2 2 255 " + bytes(11),
        "truncated_ascii": b"P2 2 2 255 1 2 3",
        "nonnumeric": b"P2 2 1 255 12a 3",
        "sample_range": b"P2 1 1 255 256",
        "negative_width": b"P5 -3 1 255 abc",
        "empty": b"",
        "header_only": b"P5",
    }
    for name, blob in pnm_cases.items():
        out[f"pnm/{name}/bytes"] = np.frombuffer(blob, dtype=np.uint8)
        try:
            out[f"pnm/{name}/planes"] = fh.decode_pnm(blob).planes
            out[f"pnm/{name}/error"] = np.array("")
        except Exception as e:  # the reference's typed error
            out[f"pnm/{name}/error"] = np.array(type(e).__name__)
    # descriptor text (cli.py:124-127 _format_value)
    from fasthog import cli as fcli
    vals = np.array([0.0, -0.0, 0.1, 1 / 3, 1e-7, 123456789.123, 2.5e-300, 1e21, 65536.0,
                     0.999999999, 12.0, float("inf"), -float("inf")])
    out["fmt/values"] = vals
    out["fmt/l2"] = np.array(" ".join(fcli._format_value(v, "l2") for v in vals))
    ints = np.array([0, 1, 64, 4096, 33153604], dtype=np.float64)
    out["fmt/ints"] = ints
    out["fmt/none"] = np.array(" ".join(fcli._format_value(v, "none") for v in ints))

    # `fasthog extract` text for a small image (cli.py:130-143), none and l2
    ximg = np.random.default_rng(99).integers(0, 256, (1, 40, 52), dtype=np.uint8)
    out["extract/image"] = ximg
    for norm in ("none", "l2"):
        g = fh.DescriptorGeometry(16, 24, 8, block=2, block_stride=1, bins=9, normalization=norm)
        st = fh.build_integral_stack(fh.gradient_map(fh.Image(ximg), fh.build_lut(9)))
        lines = []
        for x, y, values in fh.scan_descriptors(st, g, 6):
            lines.append(" ".join([str(x), str(y)] + [fcli._format_value(v, norm) for v in values]))
        out[f"extract/{norm}"] = np.frombuffer(("\n".join(lines) + "\n").encode(), dtype=np.uint8)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays; npz size "
          f"{os.path.getsize(os.path.join(HERE, 'golden.npz')) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
