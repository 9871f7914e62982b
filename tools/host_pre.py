"""Host-side cost of the Python calls in front of the first pool kernel (development tool)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native, workloads as W
wl = W.WORKLOADS["c2"]
img = fc.GrayImage(wl.image(0))
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds)
ctx = _native.Context(0)
d = torch.from_numpy(img.pixels.copy()).cuda()
for _ in range(10): fc.encode(img, cfg, context=ctx, device_image=d)
torch.cuda.synchronize()
def T(name, f, n=2000):
    f(); t = time.perf_counter()
    for _ in range(n): f()
    print(f"{name:28s} {1e6*(time.perf_counter()-t)/n:8.2f} us", flush=True)
T("set_image_device", lambda: ctx.set_image_device(int(d.data_ptr()), 512, 512))
T("native_args", lambda: params.native_args())
na = params.native_args()
def prep():
    s = np.ascontiguousarray(na[0], dtype=np.int32); c = np.ascontiguousarray(na[1], dtype=np.int64)
    t = np.ascontiguousarray(na[2], dtype=np.float64); u = np.ascontiguousarray(na[3], dtype=np.int32)
    out = np.zeros(4, dtype=np.int64); ctx._detach_views()
T("pool_build py prep", prep)
T("s_sets", lambda: tuple(cfg.policy.s_set(level) for level in (1, 2, 3, 4)))
T("int(d.data_ptr())", lambda: int(d.data_ptr()))
T("lib.fc_set_device_io", lambda: ctx.lib.fc_set_device_io(ctx.handle, 0))
# whole encode wall (host), steady state
t = time.perf_counter()
for _ in range(200): fc.encode(img, cfg, context=ctx, device_image=d)
print("encode wall us", 1e6*(time.perf_counter()-t)/200)
