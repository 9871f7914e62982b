"""Wall-clock breakdown of fc.encode's host phases on c2 (development tool):
the same calls codec.encode makes, timed one by one."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, codec, workloads as W  # noqa: E402
from paper_1502_00324_b200.pool import build_pool  # noqa: E402
from paper_1502_00324_b200.stream import CompressedStream, RecordTable  # noqa: E402

wl = W.WORKLOADS["c2"]
img = fc.GrayImage(wl.image(0))
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
d = torch.from_numpy(img.pixels.copy()).cuda()
for _ in range(10):
    fc.encode(img, cfg, context=ctx, device_image=d)
T = {}


def tick(name, t0):
    t1 = time.perf_counter()
    T[name] = T.get(name, 0.0) + t1 - t0
    return t1


N = 200
for _ in range(N):
    t = time.perf_counter()
    ctx.set_image_device(int(d.data_ptr()), img.width, img.height)
    t = tick("set_image", t)
    pool = build_pool(img, cfg.pool, context=ctx, device_image=d)
    t = tick("build_pool(+set_image)", t)
    s_sets = tuple(cfg.policy.s_set(level) for level in (1, 2, 3, 4))
    t = tick("s_sets", t)
    rec = ctx.encode(cfg.thresholds, False, s_sets, codec.PATHS[cfg.path], capacity=img.width * img.height // 4)
    t = tick("ctx.encode", t)
    stats = [ctx.encode_level_stats(level) for level in (1, 2, 3, 4)]
    t = tick("level_stats", t)
    records = RecordTable._trusted(rec[:, :5])
    t = tick("RecordTable", t)
    pools = pool.all_coords()
    t = tick("pool.all_coords", t)
    stream = CompressedStream(width=img.width, height=img.height, mode=cfg.policy.mode,
                              strides=pool.params.strides, s_sets=s_sets, pools=pools, records=records)
    t = tick("CompressedStream", t)
    sb, ssd = ctx.encode_summary()
    t = tick("encode_summary", t)
    rep = codec._report(img, cfg, pool, stream, sb, ssd, 0.0, 0.0, 0, 0.0, [], {})
    t = tick("_report", t)
for k, v in T.items():
    print(f"{k:24s} {1e3 * v / N:7.3f} ms")
t = time.perf_counter()
for _ in range(N):
    fc.encode(img, cfg, context=ctx, device_image=d)
print("fc.encode(device image) total", 1e3 * (time.perf_counter() - t) / N, "ms")
