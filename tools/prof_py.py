"""cProfile of the host side of fc.encode (+ serialize) on c2 (development tool)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

wl = W.WORKLOADS["c2"]
img = fc.GrayImage(wl.image(0))
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
for _ in range(5):
    fc.serialize(fc.encode(img, cfg, context=ctx)[0])
t0 = time.perf_counter()
for _ in range(50):
    fc.serialize(fc.encode(img, cfg, context=ctx)[0])
print("encode+serialize ms", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    fc.serialize(fc.encode(img, cfg, context=ctx)[0])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
