"""One s-histogram analysis of a workload (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = W.WORKLOADS[name]
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
ctx = _native.Context(0)
if os.environ.get("FC_REAL_CUDA_CORES"):
    ctx.set_option("real_cuda_cores", 1)
h = fc.s_histogram(fc.GrayImage(wl.image(0)), fc.EncoderConfig(pool=params, thresholds=wl.thresholds), context=ctx)
print("coded", h.coded_blocks)
