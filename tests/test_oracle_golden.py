"""Pin the CPU oracle against golden vectors produced by the reference itself
(tools/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden


def test_isometry_maps_match_numpy_rotations():
    # image.py:140-155: 0-3 clockwise rotations, 4-7 rotation then lr-mirror
    t = np.arange(36).reshape(6, 6)
    for iso in range(8):
        r = np.rot90(t, k=-(iso & 3))
        if iso >= 4:
            r = np.flip(r, axis=-1)
        assert np.array_equal(O.apply_isometry(t, iso), r)


def test_decimate_floor_rule():
    t = np.array([[1, 2], [2, 2]], dtype=np.uint8)
    assert O.decimate(t)[0, 0] == 1  # floor(7/4)


def test_matcher_cases_numpy_and_c_scan():
    g = load_golden("matcher_cases.npz")
    for k in range(int(g["n"])):
        mode = "proposed" if int(g[f"mode_{k}"]) else "baseline"
        level = int(g[f"level_{k}"])
        tiles = g[f"tiles_{k}"]
        rt = g[f"range_{k}"]
        expect = tuple(int(v) for v in g[f"expect_{k}"])
        flat = tiles.reshape(len(tiles), -1).astype(np.int64)
        means = flat.sum(axis=1) / flat.shape[1]
        s_set = O.DEFAULT_PROPOSED_SETS[level - 1] if mode == "proposed" else O.DEFAULT_BASELINE_SET
        q = O.candidate_operands(tiles, means, s_set, mode == "baseline")
        r = rt.reshape(1, -1).astype(np.int16)
        rmean = r.astype(np.int64).sum(axis=1) / r.shape[1]
        for fn in (O.scan_candidates, O.scan_candidates_numpy):
            err, idx = fn(r, rmean, q, means, s_set, mode == "baseline")
            e, iso, si = O.decode_index(idx[0], len(s_set))
            off = O.stored_offset(rmean[0], s_set, means, e, si, mode == "baseline")
            assert (int(err[0]), e, iso, si, off) == expect, (k, fn.__name__)
        if k < 40:
            assert O.naive_best_match(rt, tiles, means, s_set, mode) == expect


def test_entropies_bit_exact_and_pool_order():
    g = load_golden("entropy_cases.npz")
    for name in g["names"]:
        img = g[f"img_{name}"]
        for level in (1, 2, 3, 4):
            side = O.LEVEL_DOMAIN_SIDES[level - 1]
            for stride in (1, 3):
                _, _, ent = O.grid_entropies(img, side, stride)
                ref = g[f"ent_{name}_{level}_{stride}"]
                assert ent.tobytes() == ref.tobytes(), (name, level, stride)
            for cap in (12, 10**9):
                pl = O.build_pool_level(img, level, O.DEFAULT_STRIDES[level - 1], cap)
                coords = np.stack([pl.xs, pl.ys], axis=1)
                assert np.array_equal(coords, g[f"pool_{name}_{cap}_{level}"].reshape(-1, 2))
                assert pl.entropy.tobytes() == g[f"poolent_{name}_{cap}_{level}"].tobytes()
                if cap == 12:
                    assert np.array_equal(pl.tiles, g[f"pooltiles_{name}_{level}"])
                    assert pl.means.tobytes() == g[f"poolmeans_{name}_{level}"].tobytes()
                    assert pl.cnorm.tobytes() == g[f"poolcnorm_{name}_{level}"].tobytes()


def _check_encode_case(g, tag):
    img = g[f"image_{tag}"]
    caps = tuple(int(v) for v in g[f"caps_{tag}"])
    strides = tuple(int(v) for v in g[f"strides_{tag}"])
    mode = "proposed" if int(g[f"mode_{tag}"]) else "baseline"
    thr = tuple(float(v) for v in g[f"thresholds_{tag}"])
    enc = O.encode(img, caps, strides, mode, thr)
    assert O.serialize(enc) == g[f"bytes_{tag}"].tobytes(), tag
    assert enc.collage_ssd == int(g[f"collage_{tag}"])
    return enc


@pytest.mark.parametrize("tag", ["tiled_proposed", "tiled_baseline", "tiled4_proposed",
                                 "tiled4_baseline", "noise", "flat", "darkbright_proposed",
                                 "darkbright_baseline", "c1"])
def test_encode_cases_bytes_identical(tag):
    g = load_golden("encode_cases.npz")
    enc = _check_encode_case(g, tag)
    if tag in ("tiled_proposed", "c1", "darkbright_baseline"):
        dec, deltas = O.decode(enc)
        assert np.array_equal(dec, g[f"decoded_{tag}"])
        assert deltas == list(g[f"deltas_{tag}"])


def test_encode_lena_operating_point():
    g = load_golden("encode_lena.npz")
    enc = _check_encode_case(g, "lena256")
    assert abs(float(g["psnr_lena256"]) - 33.68) < 0.01
    assert abs(float(g["ratio_lena256"]) - 9.89) < 0.01
    del enc


@pytest.mark.slow
def test_encode_c2_bytes_identical():
    g = load_golden("encode_c2.npz")
    _check_encode_case(g, "c2")
