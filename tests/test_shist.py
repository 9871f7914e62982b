"""s-histogram analysis (reference bench.py:104-212): oracle pinned to the
reference's own outputs (tests/golden/shist_cases.npz, tools/make_golden.py
shist), then the device search (fc_real_match_level) bit-exact against both."""

import sys

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

TAGS = ("const", "tiled", "c1", "grad")


def _case(g, tag):
    caps = (int(g[f"{tag}_cap"]),) * 4
    strides = tuple(int(s) for s in g[f"{tag}_strides"])
    return g[f"{tag}_pixels"], caps, strides


def _same_means(a, b):
    return all((x is None and np.isnan(y)) or (x is not None and x == y) for x, y in zip(a, b))


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_s_histogram_matches_reference_golden(tag):
    g = load_golden("shist_cases.npz")
    pix, caps, strides = _case(g, tag)
    calls = []
    mod = sys.modules[O.s_histogram.__module__]
    real = mod.real_s_matches

    def rec(tiles, basis, norms, chunk=4096):
        out = real(tiles, basis, norms, chunk)
        calls.append(out)
        return out

    mod.real_s_matches = rec
    try:
        raw, clamped, coded, rm, cm = O.s_histogram(pix, caps, strides)
    finally:
        mod.real_s_matches = real
    assert np.array_equal(raw, g[f"{tag}_raw"])
    assert np.array_equal(clamped, g[f"{tag}_clamped"])
    assert coded == tuple(int(c) for c in g[f"{tag}_coded"])
    assert _same_means(rm, g[f"{tag}_raw_means"]) and _same_means(cm, g[f"{tag}_clamped_means"])
    assert len(calls) == int(g[f"{tag}_calls"])
    for i, (e, s, _) in enumerate(calls):
        assert e.tobytes() == g[f"{tag}_call{i}_err"].tobytes()
        assert s.tobytes() == g[f"{tag}_call{i}_slope"].tobytes()


def test_oracle_real_search_constant_image_slopes_zero():
    pix = np.full((64, 64), 90, dtype=np.uint8)
    raw, _, coded, rm, _ = O.s_histogram(pix, (8, 8, 8, 8))
    assert coded == (16, 0, 0, 0) and rm[0] == 0.0
    zero_bin = int(np.searchsorted(O.S_BIN_EDGES, 0.0, side="right")) - 1
    assert raw[0, zero_bin] == 16


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_device_s_histogram_matches_reference_golden(tag):
    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native
    g = load_golden("shist_cases.npz")
    pix, caps, strides = _case(g, tag)
    ctx = _native.Context(0)
    calls = []
    real = ctx.real_match_level

    def rec(level, origins):
        out = real(level, origins)
        calls.append(out)
        return out

    ctx.real_match_level = rec
    cfg = fc.EncoderConfig(pool=fc.PoolParams(pool_cap=caps[0], strides=strides),
                           policy=fc.SPolicy(mode=fc.PROPOSED))
    h = fc.s_histogram(fc.GrayImage(pix), cfg, context=ctx)
    assert np.array_equal(h.raw_counts, g[f"{tag}_raw"])
    assert np.array_equal(h.clamped_counts, g[f"{tag}_clamped"])
    assert h.coded_blocks == tuple(int(c) for c in g[f"{tag}_coded"])
    assert _same_means(h.raw_means, g[f"{tag}_raw_means"])
    assert len(calls) == int(g[f"{tag}_calls"])
    for i, (e, s, _) in enumerate(calls):
        assert e.tobytes() == g[f"{tag}_call{i}_err"].tobytes()
        assert s.tobytes() == g[f"{tag}_call{i}_slope"].tobytes()
    assert len(fc.shist_rows(h)) == 4 * (len(h.bin_edges) - 1)


@pytest.mark.gpu
@pytest.mark.parametrize("level,cap,stride", [(1, 3000, 4), (2, 5000, 2), (3, 5000, 2), (4, 2000, 1)])
def test_device_real_search_bit_exact_vs_oracle(level, cap, stride):
    """Larger pools (many entry chunks, ragged last block of ranges): errs,
    slopes and the winning flat index e*8 + iso identical to the oracle."""
    from paper_1502_00324_b200 import _native
    from paper_1502_00324_b200 import workloads as W
    pix = W.make_image("c2", 5)[:256, :256].copy()
    strides = [stride] * 4
    caps = [cap] * 4
    ctx = _native.Context(0)
    ctx.set_image(pix)
    ctx.pool_build(np.asarray(strides, np.int32), np.asarray(caps, np.int64),
                   np.zeros(4), np.zeros(4, np.int32))
    pool = O.build_pool_level(pix, level, stride, cap)
    side = O.LEVEL_RANGE_SIDES[level - 1]
    rng = np.random.default_rng(level)
    M = 333  # not a multiple of the 8-range block
    origins = np.stack([rng.integers(0, 256 - side + 1, M), rng.integers(0, 256 - side + 1, M)],
                       axis=1).astype(np.int32)
    e, s, idx = ctx.real_match_level(level, origins)
    tiles = O.gather_tiles(pix, [tuple(o) for o in origins], side)
    oe, os_, oi = O.real_s_matches(tiles, *O.level_basis(pool))
    assert e.tobytes() == oe.tobytes()
    assert s.tobytes() == os_.tobytes()
    assert np.array_equal(idx, oi)
