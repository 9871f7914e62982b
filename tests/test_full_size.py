"""Device parity at the BASELINE full sizes (c3 batch, c4, c5) against
golden vectors the REFERENCE itself produced (tools/make_golden_full.py,
tests/golden/full_size.json):

* c5 (2048^2, 4,133,089-window level-2 pool, 4.33e12 comparisons): the
  device pool's rank order and float64 entropy bits (sha256 of all 4.13M
  entries), and the records of 64 level-2 ranges drawn with default_rng(5)
  against the reference's own scan_tiles over its own pool;
* c4 (2048^2, three levels, ~100k-entry threshold pools): every level's pool
  (sha256 of order and entropy bits) and the records of the quadtree
  subtrees of 24 sampled top-level blocks;
* c3: the stream bytes (sha256) of 8 of the 64 images.

Bar: bit-exact / byte-identical.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native
from paper_1502_00324_b200 import workloads as W
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FULL = json.load(open(os.path.join(GOLDEN, "full_size.json")))


@pytest.fixture(scope="module")
def ctx():
    return _native.Context(0)


def _pool_hashes(ctx, pool, level):
    xy = pool.coords_array(level).astype(np.int32)
    ent, _, _, _ = ctx.pool_entries(level, pool.size(level), 2, want=("entropy",))
    return {"size": pool.size(level),
            "coords_sha256": hashlib.sha256(np.ascontiguousarray(xy).tobytes()).hexdigest(),
            "entropy_sha256": hashlib.sha256(ent.tobytes()).hexdigest()}


def _encode_records(ctx, name, path="auto"):
    """Full device encode -> (int32 records [n, 6] in depth-first order, pool)."""
    img = W.make_image(name)
    cfg = W.encoder_config(name, path)
    rec, pool, _ = fc.encode_shard(fc.GrayImage(img), cfg, 0, 1, context=ctx)
    return img, rec, pool


def _top_runs(rec, width):
    """Start index of each top-level block's records (depth-first order):
    a block's leaves cover 16 x 16 pixels."""
    side = np.array([0, 16, 8, 4, 2])[rec[:, 0]]
    area = np.cumsum(side.astype(np.int64) ** 2)
    n_top = area[-1] // 256
    ends = np.searchsorted(area, np.arange(1, n_top + 1) * 256) + 1
    return np.concatenate([[0], ends])


def test_c5_pool_order_and_entropy_bits(ctx):
    img = W.make_image("c5")
    pool = fc.build_pool(fc.GrayImage(img), W.encoder_config("c5").pool, context=ctx)
    g = FULL["c5"]
    assert list(pool.sizes) == g["caps"]
    assert _pool_hashes(ctx, pool, 2) == g["pool_l2"]


@pytest.mark.parametrize("path", ["auto", "tensor"])
def test_c5_sampled_ranges_match_reference(ctx, path):
    """64 sampled level-2 ranges of the exhaustive c5 search (4.13M domains x
    8 isometries x 2 s each) equal the reference's scan_tiles result."""
    g = FULL["c5"]
    img, rec, pool = _encode_records(ctx, "c5", path)
    assert rec.shape[0] == 65536 and (rec[:, 0] == 2).all()  # every top block split once
    assert g["l1_unsplit"] == 0
    for x, y, err, dom, iso, si, off in g["sampled_l2"]:
        top = (y // 16) * 128 + x // 16
        child = ((y % 16) // 8) * 2 + (x % 16) // 8
        r = rec[top * 4 + child]
        assert (int(r[5]), int(r[3]), int(r[2]), int(r[4]), int(r[1])) == (err, dom, iso, si, off), (x, y)


def test_c4_pools_and_sampled_subtrees_match_reference(ctx):
    g = FULL["c4"]
    img, rec, pool = _encode_records(ctx, "c4")
    assert list(pool.sizes) == g["caps"]
    for level in (1, 2, 3):
        assert _pool_hashes(ctx, pool, level) == g[f"pool_l{level}"], level
    starts = _top_runs(rec, 2048)
    # origins of every record, rebuilt from the depth-first order
    for blk in g["sampled_tops"]:
        t = blk["top"]
        got = rec[starts[t]:starts[t + 1]]
        want = blk["records"]
        assert got.shape[0] == len(want), t
        for r, (level, _x, _y, err, dom, iso, si, off) in zip(got, want):
            assert (int(r[0]), int(r[5]), int(r[3]), int(r[2]), int(r[4]), int(r[1])) == \
                (level, err, dom, iso, si, off), t


def test_c3_batch_images_bytes_identical(ctx):
    """8 of the 64 c3 images (the batch bench.py times) against the reference."""
    cfg = W.encoder_config("c3")
    for row in FULL["c3"]["images"]:
        img = W.make_image("c3", row["image"])
        stream, report = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        data = fc.serialize(stream)
        assert list(report.pool_sizes) == row["caps"], row["image"]
        assert hashlib.sha256(data).hexdigest() == row["sha256"], row["image"]
        assert report.collage_ssd == row["collage_ssd"]


def test_c3_encode_batch_matches_reference(ctx):
    """encode_batch (images overlapped on several contexts / streams, the c3
    bench path) gives each image's reference stream bytes."""
    cfg = W.encoder_config("c3")
    rows = FULL["c3"]["images"]
    imgs = [fc.GrayImage(W.make_image("c3", row["image"])) for row in rows]
    outs = fc.encode_batch(imgs, cfg, workers=3)
    for row, (stream, report) in zip(rows, outs):
        assert hashlib.sha256(fc.serialize(stream)).hexdigest() == row["sha256"], row["image"]
        assert report.collage_ssd == row["collage_ssd"]


def test_c3_encode_batch_shared_entropy_launch_matches_reference(ctx):
    """encode_batch with a context per image: every image's entropy pass in
    one pair of launches (fc_pool_entropy_batch), then per-context ranking
    and encode; each stream equals the reference's bytes."""
    cfg = W.encoder_config("c3")
    rows = FULL["c3"]["images"]
    imgs = [fc.GrayImage(W.make_image("c3", row["image"])) for row in rows]
    ctxs = [_native.Context(0) for _ in imgs]
    for _ in range(2):  # the contexts' buffers reused by a second batch
        outs = fc.encode_batch(imgs, cfg, contexts=ctxs)
        for row, (stream, report) in zip(rows, outs):
            assert hashlib.sha256(fc.serialize(stream)).hexdigest() == row["sha256"], row["image"]
            assert report.collage_ssd == row["collage_ssd"]
