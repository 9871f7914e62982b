"""One c4 encode on the tensor path (the profiling target for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = W.WORKLOADS[name]
img = wl.image(0)
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds, path="tensor")
stream, rep = fc.encode(fc.GrayImage(img), cfg, context=_native.Context(0))
print(name, "records", rep.record_count, "scan ms", round(rep.scan_device_ms, 2))
