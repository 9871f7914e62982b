"""Line-level host cost of fc.encode after the native call (development tool)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, codec, workloads as W  # noqa: E402
from paper_1502_00324_b200.pool import build_pool  # noqa: E402
from paper_1502_00324_b200.stream import CompressedStream, RecordTable, header_bytes  # noqa: E402

wl = W.WORKLOADS["c2"]
img = fc.GrayImage(wl.image(0))
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
for _ in range(5):
    fc.encode(img, cfg, context=ctx)
T = {}


def tick(name, t0):
    T[name] = T.get(name, 0.0) + time.perf_counter() - t0
    return time.perf_counter()


N = 50
for _ in range(N):
    t = time.perf_counter()
    pool = build_pool(img, cfg.pool, context=ctx)
    t = tick("build_pool", t)
    s_sets = tuple(cfg.policy.s_set(level) for level in (1, 2, 3, 4))
    rec = ctx.encode(cfg.thresholds, False, s_sets, codec.PATHS[cfg.path], capacity=img.width * img.height // 4)
    t = tick("ctx.encode", t)
    stats = [ctx.encode_level_stats(level) for level in (1, 2, 3, 4)]
    t = tick("level_stats", t)
    records = RecordTable(rec[:, :5].astype(np.int64))
    t = tick("RecordTable", t)
    pools = tuple(pool.coords(level) for level in (1, 2, 3, 4))
    t = tick("pool.coords", t)
    stream = CompressedStream(width=img.width, height=img.height, mode=cfg.policy.mode,
                              strides=pool.params.strides, s_sets=s_sets, pools=pools, records=records)
    t = tick("CompressedStream", t)
    payload = stream.payload_bits()
    t = tick("payload_bits", t)
    head = header_bytes(stream)
    t = tick("header_bytes", t)
    sb = tuple(int(v) for v in np.bincount(rec[:, 0], minlength=5)[1:5])
    ssd = int(rec[:, 5].astype(np.int64).sum())
    t = tick("misc", t)
    data = fc.serialize(stream)
    t = tick("serialize", t)
for k, v in T.items():
    print(f"{k:18s} {1e3 * v / N:7.3f} ms")
t = time.perf_counter()
for _ in range(N):
    fc.encode(img, cfg, context=ctx)
print("fc.encode total", 1e3 * (time.perf_counter() - t) / N, "ms")
