"""Per-rank work of range sharding, measured on one GPU (development tool).

Runs ``encode_shard`` for every rank of world sizes 1/2/4/8 one after the
other on cuda:0 and prints each rank's device time (CUDA events on the
context's stream, image already in HBM) and the projected strong-scaling
efficiency t(1) / (N * max_rank t(N)).  This is the compute side of the
multi-GPU step only: the record all-gather (1 MB at c5) is not included.

    python tools/time_slab.py c5 [reps] [--sharded-pool]

--sharded-pool: each rank's pool phase is its slice of the entropy pass
(fc_pool_entropy over its window rows) plus the replicated ranking
(fc_pool_rank), as in encode_distributed; the all-gather between them is not
included, and the buffers are completed once up front by a full pass (timing
only: with threshold pools the slice pass overwrites the survivor list, so the
records are not checked).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
sharded = "--sharded-pool" in sys.argv
name = args[0] if args else "c5"
reps = int(args[1]) if len(args) > 1 else 2
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
        if sharded:
            pool = pool_slice(rank, world)
            rec, _, stats = fc.encode_shard(gimg, cfg, rank, world, context=ctx, pool=pool)
        else:
            rec, _, stats = fc.encode_shard(gimg, cfg, rank, world, context=ctx, device_image=dimg)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    comps = sum(s["comparisons"] for s in stats)
    return best, comps, len(rec)


def pool_slice(rank, world):
    from paper_1502_00324_b200 import sharding
    from paper_1502_00324_b200.pool import LEVEL_RANGE_SIDES, DomainPool

    strides, caps, taus, use_tau = cfg.pool.native_args()
    lo, hi = [], []
    for level, st in zip((1, 2, 3, 4), strides):
        side = 2 * LEVEL_RANGE_SIDES[level - 1]
        a, b = sharding.slab_for_rank((img.shape[0] - side) // st + 1, rank, world)
        lo.append(a)
        hi.append(b)
    ctx.pool_entropy(strides, caps, taus, use_tau, lo, hi)
    sizes = ctx.pool_rank(full_sel)
    return DomainPool(cfg.pool, gimg.width, gimg.height, sizes, ctx)


full_sel = None
if sharded:
    fc.build_pool(gimg, cfg.pool, context=ctx, device_image=dimg)
    _, _, taus_, use_tau_ = cfg.pool.native_args()
    ctx.pool_entropy(*cfg.pool.native_args())
    full_sel = [ctx.pool_window_buffers(lv, local_sel=bool(use_tau_[lv - 1]))["sel"] or 0
                for lv in (1, 2, 3, 4)]
    ctx.pool_rank(full_sel)
timed(0, 1)  # warm-up
t1 = None
for world in (1, 2, 4, 8):
    rows = [timed(r, world) for r in range(world)]
    tmax = max(r[0] for r in rows)
    if world == 1:
        t1 = tmax
    eff = t1 / (world * tmax)
    per = " ".join(f"{ms:.2f}" for ms, _, _ in rows)
    print(f"{name}{' sharded-pool' if sharded else ''} world {world}: per-rank ms [{per}] max {tmax:.2f} "
          f"comparisons {sum(r[1] for r in rows):.4g} records {sum(r[2] for r in rows)} "
          f"projected efficiency {eff:.3f}", flush=True)
