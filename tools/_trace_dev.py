"""c2 encodes with the image resident (bench value path) and FC_TRACE=2 marks."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native, workloads as W
wl = W.WORKLOADS["c2"]; img = wl.image(0)
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
d = torch.from_numpy(img.copy()).cuda()
for i in range(6):
    if i == 5: print("=== last", flush=True)
    fc.encode(fc.GrayImage(img), cfg, context=ctx, device_image=d)
