"""Per-level scan timing on a workload's pools (development tool).

Usage: python tools/bench_level.py [WORKLOAD [LEVEL:M ...]] ; env FC_BENCH_REPS.
FC_MODE=baseline: baseline mode (10 s values); FC_PATH=exact: the CUDA-core scan.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

reps = int(os.environ.get("FC_BENCH_REPS", "10"))
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
specs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[2:]] or [(1, 1024), (2, 1884), (3, 2420)]
wl = W.WORKLOADS[name]
img = wl.image(0)
taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
caps = tuple(1 if one else 10**9 for one in wl.cap_one)
params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
ctx = _native.Context(0)
pool = fc.build_pool(fc.GrayImage(img), params, context=ctx)
base = os.environ.get("FC_MODE", "proposed") == "baseline"
policy = fc.SPolicy(mode="baseline" if base else "proposed")
path = {"exact": _native.PATH_EXACT, "tensor": _native.PATH_TENSOR}[os.environ.get("FC_PATH", "tensor")]
rng = np.random.default_rng(0)
for level, M in specs:
    side = (16, 8, 4, 2)[level - 1]
    ys, xs = np.mgrid[0:img.shape[0]:side, 0:img.shape[1]:side]
    allo = np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.int32)
    o = allo[np.sort(rng.choice(allo.shape[0], size=min(M, allo.shape[0]), replace=False))]
    ctx.level_prepare(level, base, policy.s_set(level), path)
    mains, fixes = [], []
    for _ in range(reps):
        ctx.match_level(level, o)
        st = ctx.stats()
        mains.append(st.main_ms)
        fixes.append(st.fix_ms)
    print(f"{name} L{level} M={o.shape[0]} cols={st.columns} main {np.median(mains):.3f} ms "
          f"fix {np.median(fixes):.3f} ms fix_pairs {st.fix_pairs} "
          f"cmp/s {st.comparisons / (np.median(mains) * 1e-3):.3g}", flush=True)
