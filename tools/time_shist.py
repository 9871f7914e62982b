#!/usr/bin/env python3
"""Time the s-histogram analysis (fc_real_match_level) on a workload, with the
oracle's numpy search (the reference's algorithm, bench.py:117-139) on a range
sample of level 1 for the CPU rate.  Usage: python tools/time_shist.py [c2]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = W.WORKLOADS[name]
img = wl.image(0)
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
stats = {}
real = ctx.real_match_level


def rec(level, origins):
    out = real(level, origins)
    st = ctx.stats()
    stats[level] = (st.comparisons, st.scan_ms)
    return out


ctx.real_match_level = rec
for it in range(4):
    t0 = time.perf_counter()
    h = fc.s_histogram(fc.GrayImage(img), cfg, context=ctx)
    wall = time.perf_counter() - t0
    cmp_total = sum(c for c, _ in stats.values())
    dev_ms = sum(ms for _, ms in stats.values())
    print(f"{name} it{it}: wall {wall * 1e3:.2f} ms, search device {dev_ms:.3f} ms, "
          f"{cmp_total:.4g} comparisons -> {cmp_total / (dev_ms * 1e-3):.4g} cmp/s; coded {h.coded_blocks}",
          flush=True)
for lv, (c, ms) in sorted(stats.items()):
    print(f"  level {lv}: {c:.4g} comparisons in {ms:.3f} ms -> {c / (ms * 1e-3):.4g} cmp/s")

# CPU: the oracle's numpy search on a seeded sample of level-1 ranges
lv = 1
kc = O.level_caps_for_threshold(img, wl.strides, [t if t is not None else None for t in taus])
pool = O.build_pool_level(img, lv, wl.strides[lv - 1], kc[lv - 1])
basis = O.level_basis(pool)
rng = np.random.default_rng(5)
tops = [(x, y) for y in range(0, img.shape[0], 16) for x in range(0, img.shape[1], 16)]
sample = [tops[i] for i in rng.choice(len(tops), 32, replace=False)]
tiles = O.gather_tiles(img, sample, 16)
t0 = time.perf_counter()
O.real_s_matches(tiles, *basis)
dt = time.perf_counter() - t0
c = len(sample) * len(pool.xs) * 8
print(f"oracle numpy level 1: {c:.4g} comparisons in {dt:.3f} s -> {c / dt:.4g} cmp/s "
      f"(32 sampled ranges, {len(pool.xs)} entries, numpy threads {os.cpu_count()})")
