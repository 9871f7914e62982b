"""Three c2 encodes (first warms up); the launch-list profiling target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for _ in range(3):
    stream, rep = fc.encode(fc.GrayImage(img), cfg, context=ctx)
print(name, "records", rep.record_count, {k: round(v, 3) for k, v in rep.phase_ms.items()})
