"""Device parity against the reference's golden vectors and the CPU oracle.

Bar: bit-exact.  Errors are exact integer SSDs, indices/isometries/s and the
8-bit offsets are integers, entropies are float64 bits, streams are bytes.
"""

import numpy as np
import pytest

import oracle as O
import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native
from paper_1502_00324_b200 import workloads as W
from conftest import load_golden, oracle_collage_ssd, oracle_encoding

pytestmark = pytest.mark.gpu

PATHS = ("exact", "tensor", "auto")


@pytest.fixture(scope="module")
def ctx():
    return _native.Context(0)


def test_pool_entropies_and_order_bit_exact(ctx):
    g = load_golden("entropy_cases.npz")
    for name in g["names"]:
        img = fc.GrayImage(g[f"img_{name}"])
        for cap in (12, 10**9):
            pool = fc.build_pool(img, fc.PoolParams(pool_cap=cap), context=ctx)
            for level in (1, 2, 3, 4):
                ref = g[f"pool_{name}_{cap}_{level}"].reshape(-1, 2)
                assert np.array_equal(pool.coords_array(level), ref), (name, cap, level)
                ents, tiles, means, cnorm = ctx.pool_entries(level, pool.size(level),
                                                             fc.pool.LEVEL_RANGE_SIDES[level - 1])
                assert ents.tobytes() == g[f"poolent_{name}_{cap}_{level}"].tobytes()
                if cap == 12:
                    assert np.array_equal(tiles, g[f"pooltiles_{name}_{level}"])
                    assert means.tobytes() == g[f"poolmeans_{name}_{level}"].tobytes()
                    assert cnorm.tobytes() == g[f"poolcnorm_{name}_{level}"].tobytes()


def test_pool_all_window_entropies_bit_exact(ctx):
    """Every window's entropy (cap = all) at stride 1 and 3 equals numpy's bits."""
    g = load_golden("entropy_cases.npz")
    for name in g["names"]:
        img = g[f"img_{name}"]
        for stride in (1, 3):
            pool = fc.build_pool(fc.GrayImage(img), fc.PoolParams(pool_cap=10**9, strides=(stride,) * 4),
                                 context=ctx)
            for level in (1, 2, 3, 4):
                ref = g[f"ent_{name}_{level}_{stride}"]
                ents, _, _, _ = ctx.pool_entries(level, pool.size(level), 2, want=("entropy",))
                order = np.argsort(-ref, kind="stable")
                assert ents.tobytes() == ref[order].tobytes(), (name, stride, level)


def test_entropy_constant_windows(ctx):
    """Constant windows at every level (a 16x16 window's count reaches 256) in
    patches of every value class mod 4 -- and the windows sliding into and out
    of them -- keep numpy's entropy bits (oracle LUT sums)."""
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, (96, 96)).astype(np.uint8)
    for k, v in enumerate((0, 1, 2, 3, 127, 254, 255, 64)):
        y, x = (k // 4) * 40 + 4, (k % 4) * 22 + 2
        img[y:y + 20, x:x + 20] = v  # 25 constant 16x16 windows per patch
    for stride in (1, 2):
        pool = fc.build_pool(fc.GrayImage(img), fc.PoolParams(pool_cap=10**9, strides=(stride,) * 4),
                             context=ctx)
        for level in (1, 2, 3, 4):
            _, _, ref = O.grid_entropies(img, O.LEVEL_DOMAIN_SIDES[level - 1], stride)
            ents, _, _, _ = ctx.pool_entries(level, pool.size(level), 2, want=("entropy",))
            order = np.argsort(-ref, kind="stable")
            assert ents.tobytes() == ref[order].tobytes(), (stride, level)
    flat = np.full((64, 64), 7, np.uint8)
    pool = fc.build_pool(fc.GrayImage(flat), fc.PoolParams(pool_cap=10**9), context=ctx)
    ents, _, _, _ = ctx.pool_entries(2, pool.size(2), 2, want=("entropy",))
    assert (ents == 0.0).all()


def test_pool_threshold_rank_order_bit_exact(ctx):
    """Threshold pools (device compaction + rank sort) keep {ent > tau} in the
    reference's stable descending order, ties by raster index."""
    g = load_golden("entropy_cases.npz")
    checked = 0
    for name in g["names"]:
        img = g[f"img_{name}"]
        h, w = img.shape
        for stride in (1, 3):
            taus, expect = [], []
            for level in (1, 2, 3, 4):
                ref = g[f"ent_{name}_{level}_{stride}"]
                D = fc.pool.LEVEL_DOMAIN_SIDES[level - 1]
                nx = (w - D) // stride + 1
                tau = float(np.median(ref))
                if not (ref > tau).any():
                    tau = float(np.min(ref)) - 1.0
                order = np.argsort(-ref, kind="stable")
                keep = order[ref[order] > tau]
                expect.append(np.stack([(keep % nx) * stride, (keep // nx) * stride], axis=1))
                taus.append(tau)
            pool = fc.build_pool(fc.GrayImage(img), fc.PoolParams(
                pool_cap=10**9, strides=(stride,) * 4, entropy_thresholds=tuple(taus)), context=ctx)
            for level in (1, 2, 3, 4):
                got = pool.coords_array(level).astype(np.int64)
                assert np.array_equal(got, expect[level - 1]), (name, stride, level)
                checked += 1
    assert checked > 0


def test_pool_threshold_large_set_matches_cap_order(ctx):
    """> 131072 survivors take the two-pass radix path; order equals the cap sort."""
    rng = np.random.default_rng(7)
    img = fc.GrayImage(rng.integers(0, 256, (640, 640)).astype(np.uint8))
    a = fc.build_pool(img, fc.PoolParams(pool_cap=10**9), context=ctx)
    ref = {lv: a.coords_array(lv).copy() for lv in (1, 2, 3, 4)}
    b = fc.build_pool(img, fc.PoolParams(pool_cap=10**9, entropy_thresholds=(-1.0,) * 4), context=ctx)
    for lv in (1, 2, 3, 4):
        assert np.array_equal(b.coords_array(lv), ref[lv]), lv


def test_pool_config_error(ctx):
    with pytest.raises(fc.PoolConfigError):
        fc.build_pool(fc.GrayImage.full(16, 16, 0), fc.PoolParams(pool_cap=4), context=ctx)


@pytest.mark.parametrize("path", PATHS)
def test_matcher_golden_cases(path):
    g = load_golden("matcher_cases.npz")
    checked = 0
    for k in range(int(g["n"])):
        mode = fc.PROPOSED if int(g[f"mode_{k}"]) else fc.BASELINE
        level = int(g[f"level_{k}"])
        if path == "tensor" and level == 4:
            continue
        pool = fc.DomainPool.from_tiles({level: g[f"tiles_{k}"]})
        res = fc.best_match(g[f"range_{k}"], level, pool, fc.SPolicy(mode=mode), path=path)
        got = (res.error, res.domain_index, res.isometry, res.s_index, res.offset)
        assert got == tuple(int(v) for v in g[f"expect_{k}"]), (k, mode, level)
        checked += 1
    assert checked >= 80


def test_empty_pool_raises():
    pool = fc.DomainPool.from_tiles({2: [np.zeros((8, 8), np.uint8)]})
    with pytest.raises(fc.EmptyPoolError):
        fc.best_match(np.zeros((16, 16), np.uint8), 1, pool, fc.SPolicy())


def test_constant_range_tie_breaks_to_first_flat_domain():
    rng = np.random.default_rng(1234)
    tiles = [rng.integers(0, 256, (16, 16)).astype(np.uint8) for _ in range(2)]
    tiles += [np.full((16, 16), 100, np.uint8), rng.integers(0, 256, (16, 16)).astype(np.uint8),
              np.full((16, 16), 30, np.uint8)]
    pool = fc.DomainPool.from_tiles({1: tiles})
    for path in PATHS:
        res = fc.best_match(np.full((16, 16), 77, np.uint8), 1, pool, fc.SPolicy(), path=path)
        assert (res.error, res.domain_index, res.isometry, res.s_index, res.offset) == (0, 2, 0, 0, 77)


def test_scan_candidates_dropin_reference_layout(ctx):
    rng = np.random.default_rng(7)
    for mode in ("proposed", "baseline"):
        for level in (2, 3, 4):
            side = O.LEVEL_RANGE_SIDES[level - 1]
            tiles = rng.integers(0, 256, (13, side, side)).astype(np.uint8)
            means = tiles.reshape(13, -1).astype(np.int64).sum(axis=1) / (side * side)
            s_set = O.DEFAULT_PROPOSED_SETS[level - 1] if mode == "proposed" else O.DEFAULT_BASELINE_SET
            q = O.candidate_operands(tiles, means, s_set, mode == "baseline")
            r = rng.integers(0, 256, (37, side * side)).astype(np.int16)
            rm = r.astype(np.int64).sum(axis=1) / (side * side)
            e_ref, i_ref = O.scan_candidates(r, rm, q, means, s_set, mode == "baseline")
            e_dev, i_dev = ctx.scan_candidates(r, rm, q, means, s_set, mode == "baseline")
            assert np.array_equal(e_ref, e_dev) and np.array_equal(i_ref, i_dev)


def _encode_golden(g, tag, path, taus=None, driver=None):
    img = g[f"image_{tag}"]
    caps = tuple(int(v) for v in g[f"caps_{tag}"])
    strides = tuple(int(v) for v in g[f"strides_{tag}"])
    mode = fc.PROPOSED if int(g[f"mode_{tag}"]) else fc.BASELINE
    thr = tuple(float(v) for v in g[f"thresholds_{tag}"])
    params = fc.PoolParams(pool_cap=max(caps), strides=strides, level_caps=caps,
                           entropy_thresholds=taus)
    cfg = fc.EncoderConfig(pool=params, policy=fc.SPolicy(mode=mode), thresholds=thr, path=path)
    return (driver or fc.encode)(fc.GrayImage(img), cfg)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("tag", ["tiled_proposed", "tiled_baseline", "tiled4_proposed",
                                 "tiled4_baseline", "noise", "flat", "darkbright_proposed",
                                 "darkbright_baseline", "c1"])
def test_encode_bytes_identical(tag, path):
    g = load_golden("encode_cases.npz")
    stream, report = _encode_golden(g, tag, path)
    assert fc.serialize(stream) == g[f"bytes_{tag}"].tobytes()
    assert report.collage_ssd == int(g[f"collage_{tag}"])
    dec = fc.decode(stream)
    p, ref = fc.psnr(fc.GrayImage(g[f"image_{tag}"]), dec), float(g[f"psnr_{tag}"])
    assert p == ref or abs(p - ref) < 0.01


@pytest.mark.parametrize("path", PATHS)
def test_encode_lena_operating_point(path):
    g = load_golden("encode_lena.npz")
    stream, report = _encode_golden(g, "lena256", path)
    assert fc.serialize(stream) == g["bytes_lena256"].tobytes()
    assert abs(report.comp_ratio_payload - 9.89) < 0.01


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("tag", ["c2", "c3_1"])
def test_encode_c2_c3_bytes_identical(tag, path):
    g = load_golden("encode_c2.npz")
    stream, report = _encode_golden(g, tag, path)
    assert fc.serialize(stream) == g[f"bytes_{tag}"].tobytes()
    assert report.collage_ssd == int(g[f"collage_{tag}"])


def test_entropy_threshold_compaction_equals_caps():
    """Device threshold compaction (keep ent > tau) == reference caps #{ent > tau}."""
    g = load_golden("encode_c2.npz")
    wl = W.WORKLOADS["c2"]
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    stream, _ = _encode_golden(g, "c2", "auto", taus=taus)
    assert fc.serialize(stream) == g["bytes_c2"].tobytes()


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("tag", ["tiled4_proposed", "tiled_baseline", "noise", "c1"])
def test_levelwise_driver_bytes_identical(tag, path):
    """The host-driven level seam (fc_match_level) gives the same stream as fc_encode."""
    from paper_1502_00324_b200.codec import encode_levelwise

    g = load_golden("encode_cases.npz")
    stream, report = _encode_golden(g, tag, path, driver=encode_levelwise)
    assert fc.serialize(stream) == g[f"bytes_{tag}"].tobytes()
    assert report.collage_ssd == int(g[f"collage_{tag}"])


def test_encode_records_layout_and_stats():
    """fc_encode records: steps tile the image; per-level stats are consistent."""
    g = load_golden("encode_c2.npz")
    stream, report = _encode_golden(g, "c2", "auto")
    rec = stream.records.array
    side = np.array([0, 16, 8, 4, 2])[rec[:, 0]]
    assert int((side * side).sum()) == report.width * report.height
    assert sum(report.step_blocks) == rec.shape[0]
    for ls in report.level_stats:
        assert ls["comparisons"] == ls["ranges"] * ls["columns"] * 8
        assert ls["scan_ms"] > 0


@pytest.mark.parametrize("graph", [0, 1])
def test_encode_graph_and_eager_identical(graph):
    """The CUDA-graph level loop and eager launches give the same stream."""
    g = load_golden("encode_c2.npz")
    ctx = _native.Context(0)
    ctx.set_option("graph", graph)
    img = g["image_c2"]
    caps = tuple(int(v) for v in g["caps_c2"])
    strides = tuple(int(v) for v in g["strides_c2"])
    thr = tuple(float(v) for v in g["thresholds_c2"])
    params = fc.PoolParams(pool_cap=max(caps), strides=strides, level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=thr)
    for _ in range(2):  # the second encode exercises the graph update path
        stream, _ = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        assert fc.serialize(stream) == g["bytes_c2"].tobytes()


def test_graph_reuse_across_images_abab():
    """Alternating images on one context: the cached level-loop graph is only
    replayed when every launch parameter matches, so results never go stale."""
    g = load_golden("encode_cases.npz")
    ctx = _native.Context(0)
    tags = ["noise", "tiled_proposed", "noise", "c1", "tiled_proposed"]
    for tag in tags:
        img = g[f"image_{tag}"]
        caps = tuple(int(v) for v in g[f"caps_{tag}"])
        strides = tuple(int(v) for v in g[f"strides_{tag}"])
        thr = tuple(float(v) for v in g[f"thresholds_{tag}"])
        params = fc.PoolParams(pool_cap=max(caps), strides=strides, level_caps=caps)
        cfg = fc.EncoderConfig(pool=params, thresholds=thr)
        stream, _ = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        assert fc.serialize(stream) == g[f"bytes_{tag}"].tobytes(), tag


def test_encode_rectangular_image_matches_oracle():
    """A 256x128 image (non-square lattice) against the CPU oracle, stream bytes."""
    rng = np.random.default_rng(11)
    y, x = np.mgrid[0:128, 0:256]
    img = np.clip(0.6 * x + 0.3 * y + rng.normal(0, 12, (128, 256)), 0, 255).astype(np.uint8)
    caps = (40, 60, 80, 100)
    enc = O.encode(img, caps, strides=(2, 2, 2, 2), thresholds=(6.0, 6.0, 6.0))
    params = fc.PoolParams(pool_cap=max(caps), strides=(2, 2, 2, 2), level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=(6.0, 6.0, 6.0))
    stream, _ = fc.encode(fc.GrayImage(img), cfg)
    assert fc.serialize(stream) == O.serialize(enc)


def test_encode_empty_pool_level_raises():
    """fc_encode raises EmptyPoolError when ranges reach a level with no pool."""
    ctx = _native.Context(0)
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (64, 64)).astype(np.uint8)
    ctx.set_image(img)
    ctx.pool_build((1, 1, 1, 1), (8, 8, 8, 8), (0.0,) * 4, (0,) * 4)
    ctx.pool_set_level(2, np.zeros((0, 8, 8), dtype=np.uint8))
    s_sets = tuple(fc.SPolicy().s_set(level) for level in (1, 2, 3, 4))
    with pytest.raises(fc.EmptyPoolError):
        ctx.encode((0.0, 0.0, 0.0), False, s_sets)  # threshold 0: every range splits


@pytest.mark.parametrize("world", [2, 3, 8])
def test_range_sharded_slabs_concatenate_to_the_full_encode(world):
    """Range sharding: the per-rank slabs of top-level slots,
    encoded against the replicated pool, concatenate in rank order into the
    full depth-first record list, so the gathered stream is byte-identical."""
    g = load_golden("encode_c2.npz")
    img = g["image_c2"]
    caps = tuple(int(v) for v in g["caps_c2"])
    strides = tuple(int(v) for v in g["strides_c2"])
    thr = tuple(float(v) for v in g["thresholds_c2"])
    params = fc.PoolParams(pool_cap=max(caps), strides=strides, level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=thr)
    ctx = _native.Context(0)
    full, _ = fc.encode(fc.GrayImage(img), cfg, context=ctx)
    parts = []
    for rank in range(world):
        rec, _, stats = fc.encode_shard(fc.GrayImage(img), cfg, rank, world, context=ctx)
        assert rec.dtype == np.int32 and rec.shape[1] == 6
        parts.append(rec)
    allrec = np.concatenate(parts)
    assert np.array_equal(allrec[:, :5], np.asarray(full.records.array))
    # world 1 without an initialised process group: the same stream
    stream, report = fc.encode_distributed(fc.GrayImage(img), cfg, context=ctx)
    assert fc.serialize(stream) == g["bytes_c2"].tobytes()
    assert report.collage_ssd == int(g["collage_c2"])
    # the full encode is unaffected afterwards (slab reset)
    again, _ = fc.encode(fc.GrayImage(img), cfg, context=ctx)
    assert fc.serialize(again) == g["bytes_c2"].tobytes()


@pytest.mark.parametrize("tag", ["c2", "c3_1"])
@pytest.mark.parametrize("tolerance", [0, 2])
def test_device_decoder_matches_reference_decoder(tag, tolerance):
    """fc_decode (one launch per collage pass) reproduces the reference
    decoder's image and per-pass deltas bit for bit (oracle restatement of
    codec.py:319-363), including the early stop."""
    g = load_golden("encode_c2.npz")
    stream = fc.deserialize(g[f"bytes_{tag}"].tobytes())
    want, wd = O.decode(oracle_encoding(stream), 15, tolerance)
    got, gd = fc.decode_trace(stream, 15, tolerance)
    assert gd == wd
    assert np.array_equal(got.pixels, want)


@pytest.mark.parametrize("tag", ["tiled_baseline", "darkbright_baseline", "noise", "flat",
                                 "tiled_proposed", "c1"])
def test_device_decoder_golden_cases(tag):
    """Both modes and edge streams of the golden set: the device decode equals
    the image and per-pass deltas the REFERENCE decoder recorded, and the
    PSNR it recorded."""
    g = load_golden("encode_cases.npz")
    stream = fc.deserialize(g[f"bytes_{tag}"].tobytes())
    got, deltas = fc.decode_trace(stream)
    assert np.array_equal(got.pixels, g[f"decoded_{tag}"])
    assert deltas == list(g[f"deltas_{tag}"])
    p, ref = fc.psnr(fc.GrayImage(g[f"image_{tag}"]), got), float(g[f"psnr_{tag}"])
    assert p == ref or abs(p - ref) < 0.01


@pytest.mark.parametrize("name", ["c4"])
def test_full_size_encode_properties(name):
    """BASELINE-size encode (c4: 2048^2, three levels, ~100k-column pools per
    level) checked through size-independent properties, since the CPU oracle
    cannot run the whole encode in a test:
    * one collage pass applied to the ORIGINAL image reproduces the reported
      collage SSD (the reference's test_codec.py:77-86 property);
    * a random sample of leaves, re-matched by the oracle's C scan against the
      device pool, gives the same (error, domain, isometry, s, offset)."""
    wl = W.WORKLOADS[name]
    img = wl.image(0)
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    caps = tuple(1 if one else 2**31 - 1 for one in wl.cap_one)
    params = fc.PoolParams(pool_cap=2**31 - 1, strides=wl.strides, level_caps=caps,
                           entropy_thresholds=taus)
    cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
    ctx = _native.Context(0)
    stream, report = fc.encode(fc.GrayImage(img), cfg, context=ctx)
    # (1) collage pass on the original == the sum of the leaf errors
    assert oracle_collage_ssd(stream, img) == report.collage_ssd
    # (2) sampled leaves against the oracle's exhaustive scan over the device pool
    pool = fc.build_pool(fc.GrayImage(img), params, context=ctx)  # same pool, rebuilt
    lx, ly, lside = fc.leaf_origins(stream)
    leaves = [(rec, int(x), int(y), int(sd)) for rec, x, y, sd in zip(stream.records, lx, ly, lside)]
    rng = np.random.default_rng(7)
    pick = rng.choice(len(leaves), size=min(48, len(leaves)), replace=False)
    by_level = {}
    for i in pick:
        rec, x, y, side = leaves[int(i)]
        by_level.setdefault(rec.step, []).append((rec, x, y, side))
    policy = cfg.policy
    for level, items in sorted(by_level.items()):
        side = fc.pool.LEVEL_RANGE_SIDES[level - 1]
        E = pool.size(level)
        ent, tiles, means, _ = ctx.pool_entries(level, E, side)
        svals = np.asarray(policy.s_set(level), dtype=np.float64)
        q = O.candidate_operands(tiles, means, svals, False)
        ranges = np.stack([img[y:y + side, x:x + side].reshape(-1) for _, x, y, _ in items])
        rmeans = ranges.astype(np.int64).sum(axis=1) / (side * side)
        err, idx = O.scan_candidates(ranges.astype(np.int16), rmeans, q, means, svals, False)
        for (rec, _, _, _), e_, i_, rm in zip(items, err, idx, rmeans):
            e, iso, si = O.decode_index(int(i_), len(svals))
            want = (e, iso, si, O.stored_offset(rm, svals, means, e, si, False))
            assert (rec.domain_address, rec.isometry, rec.s_index, rec.offset) == want
        del q


@pytest.mark.parametrize("option,value", [("tc_span_units", 1), ("overlap", 0),
                                          ("graph", 0)])
def test_kernel_variants_give_identical_streams(option, value):
    """Every execution variant produces the same c2 stream (tc_span_units: the
    round-robin span schedule c5 uses when B exceeds L2, forced at c2 size)."""
    g = load_golden("encode_c2.npz")
    img = g["image_c2"]
    caps = tuple(int(v) for v in g["caps_c2"])
    strides = tuple(int(v) for v in g["strides_c2"])
    thr = tuple(float(v) for v in g["thresholds_c2"])
    params = fc.PoolParams(pool_cap=max(caps), strides=strides, level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=thr, path="tensor")
    ctx = _native.Context(0)
    ctx.set_option(option, value)
    for _ in range(2):
        stream, report = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        assert fc.serialize(stream) == g["bytes_c2"].tobytes()
        assert report.collage_ssd == int(g["collage_c2"])
