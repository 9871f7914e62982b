"""Median device time of full c2 encodes (development A/B tool).

python tools/step_time.py [WORKLOAD] [STEPS]: CUDA events on the library stream
around fc.encode (image resident in HBM, L2 flushed before each step)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
wl = W.WORKLOADS[name]
img = wl.image(0)
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream_handle())
g = fc.GrayImage(img)
d = torch.from_numpy(img.copy()).cuda()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for _ in range(5):
    fc.encode(g, cfg, context=ctx, device_image=d)
ts = []
for _ in range(steps):
    flush.zero_()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fc.encode(g, cfg, context=ctx, device_image=d)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
print(f"{os.environ.get('TAG', '')} median {np.median(ts):.4f} ms  p10 {np.percentile(ts, 10):.4f}  "
      f"p90 {np.percentile(ts, 90):.4f}", flush=True)
