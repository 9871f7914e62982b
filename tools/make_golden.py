#!/usr/bin/env python3
"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports the reference package from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tools/make_golden.py

Outputs go to tests/golden/*.npz and are committed.  They pin the oracle
(`oracle/`) and, through it, the device path.  Nothing in the product or in
the GPU tests reads /root/reference at run time.
"""

from __future__ import annotations

import io
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")
REF_TOOLS = Path("/root/reference/pkg/tools")
OUT = REPO / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))

import fracodec as fc  # noqa: E402  (the reference)
from fracodec.pool import DomainEntry, DomainPool, LEVEL_DOMAIN_SIDES, _grid_entropies  # noqa: E402

from paper_1502_00324_b200 import workloads as W  # noqa: E402


def _entry(tile):
    flat = np.asarray(tile, dtype=np.int64).ravel()
    s1, s2, n = int(flat.sum()), int((flat * flat).sum()), flat.size
    return DomainEntry(0, 0, 0.0, np.asarray(tile, np.uint8), s1 / n, s2 - s1 * s1 / n)


def _pool(level, tiles):
    levels = [() for _ in range(4)]
    levels[level - 1] = tuple(_entry(t) for t in tiles)
    return DomainPool(fc.PoolParams(pool_cap=max(1, len(tiles))), 512, 512, tuple(levels))


def matcher_cases():
    """Random single-range instances in the style of criterion 1
    (test_acceptance.py:83-107), all four levels, both modes."""
    rng = np.random.default_rng(1234)
    rows = []
    for i in range(240):
        mode = fc.BASELINE if i % 2 == 0 else fc.PROPOSED
        level = int(rng.choice([1, 2, 3, 4])) if i >= 200 else int(rng.choice([2, 3, 4]))
        side = (16, 8, 4, 2)[level - 1]
        count = int(rng.integers(1, 33))
        kind = i % 5
        tiles = []
        for _ in range(count):
            if kind == 3:  # dark / bright extremes exercise the clamp
                t = rng.integers(0, 256, (side, side)) // rng.integers(1, 9)
            elif kind == 4 and rng.random() < 0.3:
                t = np.full((side, side), rng.integers(0, 256))
            else:
                t = rng.integers(0, 256, (side, side))
            tiles.append(t.astype(np.uint8))
        if kind == 2:
            tile = np.clip(rng.integers(0, 40, (side, side)) + rng.choice([0, 215]), 0, 255).astype(np.uint8)
        elif kind == 4 and rng.random() < 0.5:
            tile = np.full((side, side), rng.integers(0, 256), dtype=np.uint8)
        else:
            tile = rng.integers(0, 256, (side, side)).astype(np.uint8)
        policy = fc.SPolicy(mode=mode)
        res = fc.best_match(tile, level, _pool(level, tiles), policy)
        rows.append(dict(mode=mode, level=level, tiles=np.stack(tiles), range=tile,
                         expect=(res.error, res.domain_index, res.isometry, res.s_index, res.offset)))
    out = {"n": len(rows)}
    for k, r in enumerate(rows):
        out[f"mode_{k}"] = np.array(1 if r["mode"] == fc.PROPOSED else 0)
        out[f"level_{k}"] = np.array(r["level"])
        out[f"tiles_{k}"] = r["tiles"]
        out[f"range_{k}"] = r["range"]
        out[f"expect_{k}"] = np.array(r["expect"], dtype=np.int64)
    np.savez_compressed(OUT / "matcher_cases.npz", **out)
    print("matcher_cases", len(rows))


def entropy_cases():
    """Window entropies (float64 bits) and pool orders from the reference."""
    out = {}
    imgs = {
        "rand64_11": np.random.default_rng(11).integers(0, 256, (64, 64)).astype(np.uint8),
        "rand64_12": np.random.default_rng(12).integers(0, 256, (64, 64)).astype(np.uint8),
        "fbm96": W.fbm_image(96, 0.5, 3)[:96, :96],
        "checker64": (np.indices((64, 64)).sum(axis=0) % 2 * 255).astype(np.uint8),
        "const64": np.full((64, 64), 77, np.uint8),
        "c1": W.make_image("c1"),
    }
    for name, img in imgs.items():
        out[f"img_{name}"] = img
        for level in (1, 2, 3, 4):
            side = LEVEL_DOMAIN_SIDES[level - 1]
            for stride in (1, 3):
                xs, ys, ent = _grid_entropies(img, side, stride)
                out[f"ent_{name}_{level}_{stride}"] = ent
        for cap in (12, 10**9):
            pool = fc.build_pool(fc.GrayImage(img), fc.PoolParams(pool_cap=cap))
            for level in (1, 2, 3, 4):
                out[f"pool_{name}_{cap}_{level}"] = np.array(pool.coords(level), dtype=np.int64)
                ents = np.array([e.entropy for e in pool.entries(level)])
                out[f"poolent_{name}_{cap}_{level}"] = ents
                if cap == 12:
                    out[f"pooltiles_{name}_{level}"] = np.stack([e.tile for e in pool.entries(level)])
                    out[f"poolmeans_{name}_{level}"] = np.array([e.mean for e in pool.entries(level)])
                    out[f"poolcnorm_{name}_{level}"] = np.array(
                        [e.centered_norm_sq for e in pool.entries(level)])
    out["names"] = np.array(list(imgs))
    np.savez_compressed(OUT / "entropy_cases.npz", **out)
    print("entropy_cases", len(imgs))


def _encode_case(out, tag, image, caps, strides, mode, thresholds):
    pool_cap = max(caps)
    cfg = fc.EncoderConfig(
        pool=fc.PoolParams(pool_cap=pool_cap, strides=strides, level_caps=tuple(caps)),
        policy=fc.SPolicy(mode=mode), thresholds=thresholds)
    t0 = time.perf_counter()
    stream, report = fc.encode(fc.GrayImage(image), cfg)
    t_enc = time.perf_counter() - t0
    data = fc.serialize(stream)
    decoded, deltas = fc.decode_trace(stream)
    out[f"image_{tag}"] = image
    out[f"caps_{tag}"] = np.array(caps, dtype=np.int64)
    out[f"strides_{tag}"] = np.array(strides, dtype=np.int64)
    out[f"mode_{tag}"] = np.array(1 if mode == fc.PROPOSED else 0)
    out[f"thresholds_{tag}"] = np.array(thresholds, dtype=np.float64)
    out[f"bytes_{tag}"] = np.frombuffer(data, dtype=np.uint8)
    out[f"records_{tag}"] = np.array(
        [(r.step, r.offset, r.isometry, r.domain_address, r.s_index) for r in stream.records],
        dtype=np.int64)
    out[f"collage_{tag}"] = np.array(report.collage_ssd, dtype=np.int64)
    out[f"psnr_{tag}"] = np.array(fc.psnr(fc.GrayImage(image), decoded))
    out[f"deltas_{tag}"] = np.array(deltas, dtype=np.int64)
    out[f"decoded_{tag}"] = decoded.pixels
    print(f"  encode {tag}: {image.shape} {mode} records={len(stream.records)} "
          f"psnr={fc.psnr(fc.GrayImage(image), decoded):.3f} {t_enc:.2f}s")


def _tiled_noise(rng, size=64, cell=8, noise=4.0):
    base = rng.integers(30, 226, (size // cell, size // cell)).astype(np.float64)
    img = np.kron(base, np.ones((cell, cell))) + rng.normal(0.0, noise, (size, size))
    return np.clip(img, 0, 255).astype(np.uint8)


def workload_caps(name, img):
    wl = W.WORKLOADS[name]
    caps = []
    for li in range(4):
        side = LEVEL_DOMAIN_SIDES[li]
        xs, ys, ent = _grid_entropies(img, side, wl.strides[li])
        if wl.cap_one[li]:
            caps.append(1)
        elif wl.taus[li] is None:
            caps.append(len(ent))
        else:
            caps.append(max(1, int((ent > wl.taus[li]).sum())))
    return tuple(caps)


def encode_cases():
    out = {}
    tags = []
    rng = np.random.default_rng(1234)
    tn = _tiled_noise(rng)
    for mode in (fc.PROPOSED, fc.BASELINE):
        tag = f"tiled_{mode}"
        _encode_case(out, tag, tn, (16, 16, 16, 16), (8, 4, 2, 2), mode, (8.0, 8.0, 8.0))
        tags.append(tag)
    tn2 = _tiled_noise(np.random.default_rng(99), size=64, cell=4, noise=12.0)
    for mode in (fc.PROPOSED, fc.BASELINE):
        tag = f"tiled4_{mode}"
        _encode_case(out, tag, tn2, (32, 32, 32, 32), (8, 4, 2, 2), mode, (4.0, 4.0, 4.0))
        tags.append(tag)
    noise = np.random.default_rng(1234).integers(0, 256, (64, 64)).astype(np.uint8)
    _encode_case(out, "noise", noise, (8, 8, 8, 8), (8, 4, 2, 2), fc.PROPOSED, (0.1, 0.1, 0.1))
    tags.append("noise")
    _encode_case(out, "flat", np.full((128, 128), 128, np.uint8), (256,) * 4, (8, 4, 2, 2),
                 fc.PROPOSED, (8.0, 8.0, 8.0))
    tags.append("flat")
    dark = np.clip(W.fbm_image(64, 0.5, 5).astype(np.int32) // 3 + np.where(
        np.indices((64, 64))[1] > 31, 170, 0), 0, 255).astype(np.uint8)
    for mode in (fc.PROPOSED, fc.BASELINE):
        tag = f"darkbright_{mode}"
        _encode_case(out, tag, dark, (64, 64, 64, 64), (4, 2, 1, 1), mode, (6.0, 5.0, 4.0))
        tags.append(tag)
    c1 = W.make_image("c1")
    wl = W.WORKLOADS["c1"]
    _encode_case(out, "c1", c1, workload_caps("c1", c1), wl.strides, fc.PROPOSED, wl.thresholds)
    tags.append("c1")
    out["tags"] = np.array(tags)
    np.savez_compressed(OUT / "encode_cases.npz", **out)


def c2_case():
    out = {}
    img = W.make_image("c2")
    wl = W.WORKLOADS["c2"]
    _encode_case(out, "c2", img, workload_caps("c2", img), wl.strides, fc.PROPOSED, wl.thresholds)
    c3 = W.make_image("c3", 1)
    wl3 = W.WORKLOADS["c3"]
    _encode_case(out, "c3_1", c3, workload_caps("c3", c3), wl3.strides, fc.PROPOSED, wl3.thresholds)
    out["tags"] = np.array(["c2", "c3_1"])
    np.savez_compressed(OUT / "encode_c2.npz", **out)


def paper_fixture_case():
    """The reference's own synthetic 'lena' stand-in at DN=256, thresholds 8
    (pkg/test_output.txt:20 records 33.68 dB / payload ratio 9.89)."""
    with tempfile.TemporaryDirectory() as td:
        subprocess.check_call([sys.executable, str(REF_TOOLS / "make_fixtures.py"), "--out", td],
                              stdout=subprocess.DEVNULL)
        lena = fc.load_pgm(Path(td) / "lena.pgm").pixels.copy()
    out = {}
    _encode_case(out, "lena256", lena, (256,) * 4, (8, 4, 2, 2), fc.PROPOSED, (8.0, 8.0, 8.0))
    stream = fc.deserialize(out["bytes_lena256"].tobytes())
    payload = stream.payload_bits()
    out["ratio_lena256"] = np.array(lena.size * 8 / payload)
    out["tags"] = np.array(["lena256"])
    np.savez_compressed(OUT / "encode_lena.npz", **out)
    print(f"  lena ratio {lena.size * 8 / payload:.4f}")


def shist_cases():
    """bench.py:142 s_histogram on small images, with the per-level
    _real_s_matches outputs (errs, slopes) recorded by wrapping it."""
    import fracodec.bench as fb
    out = {}
    rng = np.random.default_rng(77)
    imgs = {
        "const": (np.full((64, 64), 90, dtype=np.uint8), 8, (8, 4, 2, 2)),
        "tiled": (_tiled_noise(rng, size=64, cell=4, noise=10.0), 16, (8, 4, 2, 2)),
        "c1": (W.make_image("c1", 0), 64, (8, 4, 2, 2)),
        "grad": (W.make_image("c2", 3)[:128, :128].copy(), 48, (4, 2, 2, 2)),
    }
    real = fb._real_s_matches
    for tag, (pix, cap, strides) in imgs.items():
        calls = []

        def rec(tiles, basis, norms, _calls=calls):
            e, s = real(tiles, basis, norms)
            _calls.append((tiles.shape[1], e.copy(), s.copy()))
            return e, s

        fb._real_s_matches = rec
        try:
            cfg = fc.EncoderConfig(pool=fc.PoolParams(pool_cap=cap, strides=strides),
                                   policy=fc.SPolicy(mode=fc.PROPOSED))
            h = fc.s_histogram(fc.GrayImage(pix), cfg)
        finally:
            fb._real_s_matches = real
        out[f"{tag}_pixels"] = pix
        out[f"{tag}_cap"] = np.int64(cap)
        out[f"{tag}_strides"] = np.asarray(strides, dtype=np.int64)
        out[f"{tag}_raw"] = h.raw_counts
        out[f"{tag}_clamped"] = h.clamped_counts
        out[f"{tag}_coded"] = np.asarray(h.coded_blocks, dtype=np.int64)
        out[f"{tag}_raw_means"] = np.asarray([np.nan if v is None else v for v in h.raw_means])
        out[f"{tag}_clamped_means"] = np.asarray(
            [np.nan if v is None else v for v in h.clamped_means])
        for i, (n, e, sl) in enumerate(calls):
            out[f"{tag}_call{i}_n"] = np.int64(n)
            out[f"{tag}_call{i}_err"] = e
            out[f"{tag}_call{i}_slope"] = sl
        out[f"{tag}_calls"] = np.int64(len(calls))
        print(f"  shist {tag}: coded {h.coded_blocks}")
    np.savez_compressed(OUT / "shist_cases.npz", **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    which = sys.argv[1:] or ["matcher", "entropy", "encode", "c2", "lena"]
    if "matcher" in which:
        matcher_cases()
    if "entropy" in which:
        entropy_cases()
    if "encode" in which:
        encode_cases()
    if "c2" in which:
        c2_case()
    if "lena" in which:
        paper_fixture_case()
    if "shist" in which:
        shist_cases()
