#!/usr/bin/env python3
"""Full-size golden vectors (BASELINE c3 / c4 / c5) from the REFERENCE itself.

Run in the build container only (imports the reference package from
/root/reference/pkg/src, absent on the GPU box):

    python tools/make_golden_full.py [c5] [c4] [c3]

Writes tests/golden/full_size.json (small: hashes and sampled records).

* c5 (2048^2 fBm, level 2 only, L=1, every window kept): sha256 of the
  reference pool's rank-ordered origins and float64 entropies at level 2
  (4,133,089 entries), and the reference's scan_tiles result for 64 level-2
  ranges drawn with default_rng(5) (BASELINE.md section 3 sampled mode).
* c4 (2048^2 fBm+noise, levels 1-3, L=2, p90 entropy caps): per-level pool
  hashes, and the records of the quadtree subtrees of 24 top-level blocks
  drawn with default_rng(5).  A top block's subtree depends only on its own
  errors (codec.py:134-142), so the reference's scan_tiles on the sampled
  blocks level by level, with the reference's split rule (codec.py:132-141),
  gives exactly the records the full encode emits for those blocks.
* c3 (64 x 512^2): sha256 of the serialized FRAK stream, collage SSD and
  record count of the reference's full encode of 8 of the 64 images.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")
OUT = REPO / "tests" / "golden" / "full_size.json"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tools"))

import fracodec as fc  # noqa: E402  (the reference)
from fracodec.codec import _gather_tiles  # noqa: E402
from fracodec.matcher import build_candidate_set, result_from_index, scan_tiles  # noqa: E402
from fracodec.pool import LEVEL_RANGE_SIDES  # noqa: E402

from make_golden import workload_caps  # noqa: E402
from paper_1502_00324_b200 import workloads as W  # noqa: E402

C3_IMAGES = (0, 9, 18, 27, 36, 45, 54, 63)
C4_TOPS = 24
C5_RANGES = 64


def pool_hashes(pool, level):
    entries = pool.entries(level)
    xy = np.array([(e.x, e.y) for e in entries], dtype=np.int32).reshape(-1, 2)
    ent = np.array([e.entropy for e in entries], dtype=np.float64)
    return {"size": len(entries),
            "coords_sha256": hashlib.sha256(xy.tobytes()).hexdigest(),
            "entropy_sha256": hashlib.sha256(ent.tobytes()).hexdigest()}


def ref_pool(name, img):
    wl = W.WORKLOADS[name]
    caps = workload_caps(name, img)
    params = fc.PoolParams(pool_cap=max(caps), strides=wl.strides, level_caps=caps)
    t0 = time.perf_counter()
    pool = fc.build_pool(fc.GrayImage(img), params)
    print(f"  {name}: reference pool {time.perf_counter() - t0:.1f}s caps={caps}", flush=True)
    return caps, pool


def c5():
    img = W.make_image("c5")
    caps, pool = ref_pool("c5", img)
    policy = fc.SPolicy()
    out = {"caps": list(caps), "pool_l2": pool_hashes(pool, 2)}
    # level 1: one domain, threshold 1e-9 -> every top block splits unless its error is 0
    cs1 = build_candidate_set(pool, 1, policy)
    tops = [(x, y) for y in range(0, 2048, 16) for x in range(0, 2048, 16)]
    e1, _, _ = scan_tiles(_gather_tiles(img, tops, 16), cs1)
    out["l1_unsplit"] = int((e1 <= 1e-9 ** 2 * 256).sum())
    t0 = time.perf_counter()
    cs = build_candidate_set(pool, 2, policy)
    t1 = time.perf_counter()
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(65536, C5_RANGES, replace=False))
    origins = [(int(p % 256) * 8, int(p // 256) * 8) for p in pick]
    errs, idxs, rmeans = scan_tiles(_gather_tiles(img, origins, 8), cs)
    t2 = time.perf_counter()
    rows = []
    for (x, y), e, i, rm in zip(origins, errs, idxs, rmeans):
        r = result_from_index(cs, float(rm), int(e), int(i))
        rows.append([x, y, r.error, r.domain_index, r.isometry, r.s_index, r.offset])
    out["sampled_l2"] = rows
    out["sample"] = f"default_rng(5).choice(65536, {C5_RANGES}) of the level-2 ranges (raster)"
    out["ref_seconds"] = {"candidate_set": t1 - t0, "scan": t2 - t1,
                          "comparisons": int(C5_RANGES * cs.q.shape[0])}
    print(f"  c5: candidate set {t1 - t0:.1f}s, scan {t2 - t1:.1f}s", flush=True)
    return out


def c4():
    name = "c4"
    img = W.make_image(name)
    wl = W.WORKLOADS[name]
    caps, pool = ref_pool(name, img)
    policy = fc.SPolicy()
    out = {"caps": list(caps)}
    for level in (1, 2, 3):
        out[f"pool_l{level}"] = pool_hashes(pool, level)
    rng = np.random.default_rng(5)
    n_top = (2048 // 16) ** 2
    tops = np.sort(rng.choice(n_top, C4_TOPS, replace=False))
    css = {}
    blocks = []
    for t in tops:
        x0, y0 = int(t % 128) * 16, int(t // 128) * 16
        recs = []

        def walk(level, x, y):
            cs = css.get(level)
            if cs is None:
                cs = css[level] = build_candidate_set(pool, level, policy)
            side = LEVEL_RANGE_SIDES[level - 1]
            e, i, rm = scan_tiles(_gather_tiles(img, [(x, y)], side), cs)
            if level < 4 and int(e[0]) > wl.thresholds[level - 1] ** 2 * side * side:
                h = side // 2
                for dx, dy in ((0, 0), (h, 0), (0, h), (h, h)):
                    walk(level + 1, x + dx, y + dy)
                return
            r = result_from_index(cs, float(rm[0]), int(e[0]), int(i[0]))
            recs.append([level, x, y, r.error, r.domain_index, r.isometry, r.s_index, r.offset])

        walk(1, x0, y0)
        blocks.append({"top": int(t), "records": recs})
    out["sampled_tops"] = blocks
    out["sample"] = f"default_rng(5).choice({n_top}, {C4_TOPS}) top-level 16x16 blocks (raster)"
    return out


def c3():
    wl = W.WORKLOADS["c3"]
    rows = []
    for idx in C3_IMAGES:
        img = W.make_image("c3", idx)
        caps = workload_caps("c3", img)
        cfg = fc.EncoderConfig(pool=fc.PoolParams(pool_cap=max(caps), strides=wl.strides,
                                                  level_caps=caps), thresholds=wl.thresholds)
        t0 = time.perf_counter()
        stream, report = fc.encode(fc.GrayImage(img), cfg)
        data = fc.serialize(stream)
        rows.append({"image": idx, "caps": list(caps), "sha256": hashlib.sha256(data).hexdigest(),
                     "bytes": len(data), "collage_ssd": int(report.collage_ssd),
                     "records": len(stream.records)})
        print(f"  c3 image {idx}: {time.perf_counter() - t0:.1f}s records={len(stream.records)}",
              flush=True)
    return {"images": rows}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c5", "c4", "c3"]
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data["generator"] = "tools/make_golden_full.py (reference fracodec imported in place)"
    for name, fn in (("c5", c5), ("c4", c4), ("c3", c3)):
        if name in which:
            data[name] = fn()
            OUT.write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", OUT)
