import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import workloads as W, _native

ctx = _native.Context(0)
for name in sys.argv[1:] or ["c2"]:
    wl = W.WORKLOADS[name]
    img = wl.image(0)
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    caps = tuple(1 if one else 10**9 for one in wl.cap_one)
    params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
    cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds, path="exact")
    for it in range(3):
        t0 = time.perf_counter()
        stream, rep = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        t1 = time.perf_counter()
        print(f"{name} it{it}: wall {t1-t0:.4f}s pool {rep.pool_time_s:.4f}s scan_dev {rep.scan_device_ms:.2f}ms "
              f"comparisons {rep.comparisons:.4g} -> {rep.comparisons/(rep.scan_device_ms*1e-3):.4g} cmp/s (scan) "
              f"pools {rep.pool_sizes} steps {rep.step_blocks}", flush=True)
