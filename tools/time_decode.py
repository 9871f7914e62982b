#!/usr/bin/env python3
"""Time the device decoder (fc.decode_trace: 15 collage passes from a
constant-128 image, codec.py:339-363) on a workload's encoded stream, with
the oracle's numpy decoder on the same stream as the CPU figure and the
bit-identity check.  Usage: python tools/time_decode.py [c2 c4 c5 ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402
from conftest import oracle_encoding  # noqa: E402

reps = int(os.environ.get("FC_DECODE_REPS", "5"))
ctx = _native.Context(0)
for name in sys.argv[1:] or ["c2"]:
    img = W.make_image(name)
    stream, _ = fc.encode(fc.GrayImage(img), W.encoder_config(name), context=ctx)
    fc.decode_trace(stream, context=ctx)  # warm-up
    walls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out, deltas = fc.decode_trace(stream, context=ctx)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    t0 = time.perf_counter()
    ref, ref_deltas = O.decode(oracle_encoding(stream), 15, 0)
    cpu = time.perf_counter() - t0
    same = np.array_equal(out.pixels, ref) and list(deltas) == list(ref_deltas)
    px = img.size * len(deltas)
    print(f"{name}: {len(stream.records)} leaves, {len(deltas)} passes; device decode {wall * 1e3:.2f} ms "
          f"({px / wall / 1e6:.1f} Mpixel-passes/s, host records in, image out); oracle numpy "
          f"{cpu * 1e3:.0f} ms ({cpu / wall:.0f}x); bit-identical: {same}", flush=True)
