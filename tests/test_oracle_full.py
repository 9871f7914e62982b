"""Pin the oracle's full-size helpers (banded entropies, base-operand scan)
against the reference's own full-size outputs (tests/golden/full_size.json,
tools/make_golden_full.py).  CPU only; a few host cores for ~1 minute."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_1502_00324_b200 import workloads as W
from conftest import GOLDEN

FULL = json.load(open(os.path.join(GOLDEN, "full_size.json")))


def _hashes(xs, ys, ent):
    xy = np.stack([xs, ys], axis=1).astype(np.int32)
    return {"size": len(xs), "coords_sha256": hashlib.sha256(xy.tobytes()).hexdigest(),
            "entropy_sha256": hashlib.sha256(np.ascontiguousarray(ent).tobytes()).hexdigest()}


@pytest.fixture(scope="module")
def c5_pool():
    img = W.make_image("c5")
    xs, ys, ent = O.pool_order(img, 2, 1, 10**9)
    return img, xs, ys, ent


def test_oracle_c5_pool_matches_reference(c5_pool):
    _, xs, ys, ent = c5_pool
    assert _hashes(xs, ys, ent) == FULL["c5"]["pool_l2"]


def test_oracle_c5_sampled_scan_matches_reference(c5_pool):
    img, xs, ys, _ = c5_pool
    tiles, means, _ = O.pool_tiles(img, 2, xs, ys)
    sv = O.DEFAULT_PROPOSED_SETS[1]
    qb = O.base_operands(tiles, means, sv, False)
    rows = FULL["c5"]["sampled_l2"][::8]  # 8 of the 64 (the GPU test checks all)
    r = np.stack([img[y:y + 8, x:x + 8].reshape(-1) for x, y, *_ in rows]).astype(np.int16)
    rm = r.astype(np.int64).sum(axis=1) / 64
    err, idx = O.scan_candidates_base(r, rm, qb, means, sv, False)
    for row, e_, i_, m_ in zip(rows, err, idx, rm):
        e, iso, si = O.decode_index(int(i_), 2)
        assert [row[0], row[1], int(e_), e, iso, si, O.stored_offset(m_, sv, means, e, si, False)] == row


def test_oracle_c4_pools_and_subtrees_match_reference():
    g = FULL["c4"]
    wl = W.WORKLOADS["c4"]
    img = W.make_image("c4")
    pools = {}
    for level in (1, 2, 3):
        xs, ys, ent = O.pool_order(img, level, wl.strides[level - 1], g["caps"][level - 1])
        assert _hashes(xs, ys, ent) == g[f"pool_l{level}"], level
        tiles, means, _ = O.pool_tiles(img, level, xs, ys)
        sv = O.DEFAULT_PROPOSED_SETS[level - 1]
        pools[level] = (means, O.base_operands(tiles, means, sv, False), sv)

    def walk(level, x, y, out):
        side = O.LEVEL_RANGE_SIDES[level - 1]
        means, qb, sv = pools[level]
        r = img[y:y + side, x:x + side].reshape(1, -1).astype(np.int16)
        rm = r.astype(np.int64).sum(axis=1) / (side * side)
        err, idx = O.scan_candidates_base(r, rm, qb, means, sv, False)
        if int(err[0]) > wl.thresholds[level - 1] ** 2 * side * side:  # codec.py:132-141
            h = side // 2
            for dx, dy in ((0, 0), (h, 0), (0, h), (h, h)):
                walk(level + 1, x + dx, y + dy, out)
            return
        e, iso, si = O.decode_index(int(idx[0]), len(sv))
        out.append([level, x, y, int(err[0]), e, iso, si, O.stored_offset(rm[0], sv, means, e, si, False)])

    for blk in g["sampled_tops"][:6]:
        t = blk["top"]
        out = []
        walk(1, (t % 128) * 16, (t // 128) * 16, out)
        assert out == blk["records"], t


def test_oracle_c3_images_match_reference():
    wl = W.WORKLOADS["c3"]
    for row in FULL["c3"]["images"][:2]:
        img = W.make_image("c3", row["image"])
        enc = O.encode(img, row["caps"], wl.strides, "proposed", wl.thresholds)
        data = O.serialize(enc)
        assert hashlib.sha256(data).hexdigest() == row["sha256"]
        assert enc.collage_ssd == row["collage_ssd"]
