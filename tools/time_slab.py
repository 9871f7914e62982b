"""Per-rank work of range sharding, measured on one GPU (development tool).

Runs ``encode_shard`` for every rank of world sizes 1/2/4/8 one after the
other on cuda:0 and prints each rank's device time (CUDA events on the
context's stream, image already in HBM) and the projected strong-scaling
efficiency t(1) / (N * max_rank t(N)).  This is the compute side of the
multi-GPU step only: the record all-gather (1 MB at c5) is not included.

    python tools/time_slab.py c5 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = W.WORKLOADS[name]
cfg = W.encoder_config(name, "auto")
img = wl.image(0)
gimg = fc.GrayImage(img)
ctx = _native.Context(0)
dimg = torch.from_numpy(img.copy()).cuda()
stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", 0))


def timed(rank, world):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rec, _, stats = fc.encode_shard(gimg, cfg, rank, world, context=ctx, device_image=dimg)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    comps = sum(s["comparisons"] for s in stats)
    return best, comps, len(rec)


timed(0, 1)  # warm-up
t1 = None
for world in (1, 2, 4, 8):
    rows = [timed(r, world) for r in range(world)]
    tmax = max(r[0] for r in rows)
    if world == 1:
        t1 = tmax
    eff = t1 / (world * tmax)
    per = " ".join(f"{ms:.2f}" for ms, _, _ in rows)
    print(f"{name} world {world}: per-rank ms [{per}] max {tmax:.2f} "
          f"comparisons {sum(r[1] for r in rows):.4g} records {sum(r[2] for r in rows)} "
          f"projected efficiency {eff:.3f}", flush=True)
