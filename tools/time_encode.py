"""Quick device timing of whole encodes per workload (development tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_00324_b200 as fc  # noqa: E402
from paper_1502_00324_b200 import _native, workloads as W  # noqa: E402

path = os.environ.get("FC_PATH", "auto")
reps = int(os.environ.get("FC_REPS", "3"))
mode = os.environ.get("FC_MODE", "proposed")  # or "baseline"
ctx = _native.Context(0)
for name in sys.argv[1:] or ["c2"]:
    wl = W.WORKLOADS[name]
    img = wl.image(0)
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    caps = tuple(1 if one else 10**9 for one in wl.cap_one)
    params = fc.PoolParams(pool_cap=10**9, strides=wl.strides, level_caps=caps, entropy_thresholds=taus)
    cfg = fc.EncoderConfig(pool=params, thresholds=wl.thresholds, path=path,
                           policy=fc.SPolicy(mode=mode))
    for it in range(reps):
        t0 = time.perf_counter()
        stream, rep = fc.encode(fc.GrayImage(img), cfg, context=ctx)
        t1 = time.perf_counter()
        st = ctx.stats()
        print(f"{name} {mode} {path} it{it}: wall {t1-t0:.4f}s pool {rep.pool_time_s:.4f}s scan_dev {rep.scan_device_ms:.2f}ms "
              f"cmp {rep.comparisons:.4g} -> {rep.comparisons/(rep.scan_device_ms*1e-3):.4g} cmp/s | last level: "
              f"main {st.main_ms:.2f}ms fix {st.fix_ms:.2f}ms fix_pairs {st.fix_pairs} rescans {st.rescans} path {st.path} "
              f"pools {rep.pool_sizes} steps {rep.step_blocks}", flush=True)
        if it == reps - 1:
            for ls in rep.level_stats:
                print("   ", ls, flush=True)
            print("    phases(ms):", {k: round(v, 3) for k, v in rep.phase_ms.items()}, flush=True)
