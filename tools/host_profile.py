"""Host-side cost of a c2 encode (development tool): Python / ctypes steps
timed in a loop, then a cProfile of whole encodes.  python tools/host_profile.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native, workloads as W
from paper_1502_00324_b200.pool import _adopt_device_image
wl = W.WORKLOADS["c2"]; cfg = W.encoder_config("c2")
img = wl.image(0); g = fc.GrayImage(img); ctx = _native.Context(0)
d = torch.from_numpy(img.copy()).cuda()
for _ in range(5): fc.encode(g, cfg, context=ctx, device_image=d)
torch.cuda.synchronize()
N = 200
def t(f, name):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(N): f()
    torch.cuda.synchronize(); print(f"{name:40s} {1e6*(time.perf_counter()-t0)/N:8.1f} us")
t(lambda: _adopt_device_image(ctx, d, g), "adopt_device_image")
t(lambda: cfg.pool.native_args(), "native_args")
t(lambda: ctx.set_image_device(int(d.data_ptr()), g.width, g.height), "set_image_device")
t(lambda: fc.build_pool(g, cfg.pool, context=ctx, device_image=d), "build_pool (incl sync)")
t(lambda: fc.encode(g, cfg, context=ctx, device_image=d), "encode total")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(50): fc.encode(g, cfg, context=ctx, device_image=d)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(18)
