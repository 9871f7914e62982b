"""Wall-clock split of the bench's e2e step (fc.encode from host pixels, then
fc.serialize) for a workload.  Usage: python tools/e2e_breakdown.py [c5]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
ctx = _native.Context(0)
cfg = W.encoder_config(name)
img = fc.GrayImage(W.make_image(name))
for it in range(4):
    t0 = time.perf_counter()
    stream, rep = fc.encode(img, cfg, context=ctx)
    t1 = time.perf_counter()
    data = fc.serialize(stream)
    t2 = time.perf_counter()
    print(f"encode {1e3 * (t1 - t0):8.2f} ms  serialize {1e3 * (t2 - t1):6.2f} ms  bytes {len(data)}  "
          f"phases {', '.join(f'{k} {v:.1f}' for k, v in rep.phase_ms.items())}", flush=True)
