#!/usr/bin/env python3
"""Benchmark: range-domain comparisons/sec of the B200 fractal encoder search.

Metric (BASELINE.json): range-domain comparisons/sec, with encode Mpixel/s
alongside.  A comparison is one (range, domain, isometry, s) candidate whose
exact SSD the reference evaluates (_scan.py:35-57); comparisons per level =
ranges * pool * 8 * |S|.

Default workload: c5 (BASELINE configs[4]: 2048^2 fBm, exhaustive B=8 level
over all 4,133,089 domains, 4.33e12 comparisons per encode), the largest
configuration that fits one GPU.  A "step" is one full encode: entropy pools
for all levels, every quadtree level's exhaustive search, split decisions and
records.  ``value`` is timed with CUDA events on the library's own stream with
the image already resident in HBM (L2 flushed between steps); ``e2e`` is the
same encode through the public API ``fc.encode`` from host pixels plus
``fc.serialize`` of the result (wall clock).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
        python bench.py --impl reference ...   (CPU arm: oracle port on all host cores)
--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (one process per GPU).  c2/c4/c5 shard the ranges of
one image (top-level slabs, replicated pool, records all-gathered over NCCL);
c3 shards its 64 images.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "c5"  # BASELINE.json configs[4]: the largest single-GPU config
SAMPLED = ("c4", "c5")   # CPU arm: sampled ranges / top blocks


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--path", default="auto", choices=["auto", "exact", "tensor"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="auto", choices=["auto", "images", "ranges", "balanced"],
                    help="auto: images for c3 (its 64-image batch), ranges otherwise; "
                         "images: one seeded image per rank (weak scaling); "
                         "ranges: one image split into top-level slabs (encode_distributed); "
                         "balanced: every level re-sliced evenly over the ranks (encode_balanced)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def relaunch_distributed(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def shard_mode(args) -> str:
    if args.shard != "auto":
        return args.shard
    return "images" if args.workload == "c3" else "ranges"


# ---------------------------------------------------------------------------
# CPU arm (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------

class CpuSample:
    """The reference's algorithm on the host, timed on a bounded sample.

    c1-c3: one full encode per step (oracle.encode: numpy pool, C/OpenMP
    scan restating _scan.py).  c4/c5 (BASELINE.md section 3 sampled mode):
    the pools and base operands are built once (untimed, reported), then
    every step matches `per_step` ranges (c5) or top-level blocks' quadtree
    subtrees (c4), drawn with default_rng(5), against the full pool; the rate
    is sampled comparisons / matching time (extrapolates linearly: the work
    is linear in the ranges)."""

    def __init__(self, name: str, threads: int):
        from oracle import fracodec_oracle as O
        from paper_1502_00324_b200 import workloads as W

        self.O, self.W = O, W
        self.name = name
        self.wl = W.WORKLOADS[name]
        self.threads = threads
        self.rng = np.random.default_rng(5)
        self.setup_s = 0.0
        self.img = self.wl.image(0)
        self.image_index = 0
        self.per_step = max(threads, 1)
        if name in SAMPLED:
            t0 = time.perf_counter()
            self.pools = {}
            levels = (2,) if name == "c5" else (1, 2, 3)
            caps = self.caps(self.img)
            for level in levels:
                cap = caps[level - 1]
                xs, ys, _ = O.pool_order(self.img, level, self.wl.strides[level - 1], cap, threads)
                tiles, means, _ = O.pool_tiles(self.img, level, xs, ys)
                sv = O.DEFAULT_PROPOSED_SETS[level - 1]
                self.pools[level] = (means, O.base_operands(tiles, means, sv, False), sv)
            self.setup_s = time.perf_counter() - t0

    def caps(self, img):
        O, wl = self.O, self.wl
        caps = []
        for li in range(4):
            if wl.cap_one[li]:
                caps.append(1)
                continue
            _, _, ent = O.grid_entropies_parallel(img, O.LEVEL_DOMAIN_SIDES[li], wl.strides[li],
                                                  self.threads)
            caps.append(len(ent) if wl.taus[li] is None else max(1, int((ent > wl.taus[li]).sum())))
        return tuple(caps)

    def _match(self, level, origins):
        O = self.O
        side = O.LEVEL_RANGE_SIDES[level - 1]
        means, qb, sv = self.pools[level]
        r = np.stack([self.img[y:y + side, x:x + side].reshape(-1) for x, y in origins]).astype(np.int16)
        rm = r.astype(np.int64).sum(axis=1) / (side * side)
        err, idx = O.scan_candidates_base(r, rm, qb, means, sv, False, self.threads)
        return err, idx, rm, len(origins) * qb.shape[0] * 8

    def step(self):
        """-> (comparisons, seconds, sample description, checks) for one step."""
        O = self.O
        if self.name not in SAMPLED:
            idx = self.image_index % self.wl.images
            self.image_index += 1
            img = self.wl.image(idx)
            caps = self.caps(img)
            t0 = time.perf_counter()
            enc = O.encode(img, caps, self.wl.strides, "proposed", self.wl.thresholds,
                           threads=self.threads)
            dt = time.perf_counter() - t0
            comps = sum(len(errs) * len(enc.pools[lv - 1]) * 8 * len(enc.s_sets[lv - 1])
                        for lv, (errs, _i, _r, _o) in enc.scans.items())
            return comps, dt, f"full encode of image {idx}", {"image": idx, "bytes": O.serialize(enc)}
        if self.name == "c5":
            pick = np.sort(self.rng.choice(65536, self.per_step, replace=False))
            origins = [(int(p % 256) * 8, int(p // 256) * 8) for p in pick]
            t0 = time.perf_counter()
            err, idx, rm, comps = self._match(2, origins)
            dt = time.perf_counter() - t0
            means, _, sv = self.pools[2]
            rows = []
            for (x, y), e_, i_, m_ in zip(origins, err, idx, rm):
                e, iso, si = O.decode_index(int(i_), len(sv))
                rows.append((x, y, int(e_), e, iso, si, O.stored_offset(m_, sv, means, e, si, False)))
            return comps, dt, f"{len(origins)} level-2 ranges x the full pool", {"ranges": rows}
        # c4: quadtree subtrees of sampled top blocks, level by level (codec.py:114-161)
        n_top = (self.img.shape[1] // 16) * (self.img.shape[0] // 16)
        tops = np.sort(self.rng.choice(n_top, self.per_step, replace=False))
        nx = self.img.shape[1] // 16
        frontier = [(int(t % nx) * 16, int(t // nx) * 16) for t in tops]
        comps, dt, leaves = 0, 0.0, {}
        for level in (1, 2, 3):
            if not frontier:
                break
            t0 = time.perf_counter()
            err, idx, rm, c = self._match(level, frontier)
            dt += time.perf_counter() - t0
            comps += c
            side = O.LEVEL_RANGE_SIDES[level - 1]
            nxt = []
            means, _, sv = self.pools[level]
            for (x, y), e_, i_, m_ in zip(frontier, err, idx, rm):
                if level < 3 and int(e_) > self.wl.thresholds[level - 1] ** 2 * side * side:
                    h = side // 2
                    nxt += [(x, y), (x + h, y), (x, y + h), (x + h, y + h)]
                else:
                    e, iso, si = O.decode_index(int(i_), len(sv))
                    leaves[(level, x, y)] = (int(e_), e, iso, si,
                                             O.stored_offset(m_, sv, means, e, si, False))
            frontier = nxt
        return comps, dt, f"quadtree subtrees of {len(tops)} top-level blocks", {
            "tops": [int(t) for t in tops], "leaves": leaves}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    cpu = CpuSample(args.workload, threads)
    for _ in range(args.warmup):
        cpu.step()
    total_t, total_c = 0.0, 0
    desc = ""
    for _ in range(args.steps):
        comps, dt, desc, _ = cpu.step()
        total_t += dt
        total_c += comps
    value = total_c / total_t
    from paper_1502_00324_b200 import workloads as W

    sample = (f"{args.workload}: {desc} per step, {args.steps} steps (oracle/: numpy pool + "
              f"C/OpenMP exhaustive scan restating _scan.py, {threads} threads)")
    if args.workload in SAMPLED:
        sample += f"; pool + operand setup {cpu.setup_s:.1f} s, untimed (matching-only rate)"
    line = {
        "impl": "reference", "metric": "range-domain comparisons/sec", "value": value,
        "unit": "comparisons/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "description": W.WORKLOADS[args.workload].description},
        "cpu_baseline": {"value": value, "unit": "comparisons/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "comparisons/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clock / throttle-reason samples during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "samples": len(rows), "reasons": sorted(reasons)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def cublas_int8_tops(torch):
    """cuBLASLt int8 8192^3 (torch._int_mm), best of 5: a cross-check of the peak."""
    try:
        n = 8192
        a = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
        for _ in range(2):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    except Exception:  # noqa: BLE001
        return None


def window_count(wl, width, height):
    from paper_1502_00324_b200.pool import LEVEL_DOMAIN_SIDES, candidate_count

    return sum(candidate_count((width, height), D, s) for D, s in zip(LEVEL_DOMAIN_SIDES, wl.strides))


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native, sharding, workloads as W

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"{world} ranks but only {torch.cuda.device_count()} visible GPUs")
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    ctx = _native.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", local))
    wl = W.WORKLOADS[args.workload]
    cfg = W.encoder_config(args.workload, args.path)
    mode = shard_mode(args)
    ranges = mode in ("ranges", "balanced")
    if ranges:  # every rank holds the same image and encodes its slab of top-level slots
        idx = [0]
    elif wl.images > 1:
        idx = sharding.images_for_rank(wl.images, rank, world)
    else:
        idx = [rank]
    imgs = [wl.image(i) for i in idx]
    gimgs = [fc.GrayImage(im) for im in imgs]
    dimgs = [torch.from_numpy(im.copy()).cuda() for im in imgs]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")  # 512 MB > L2
    # one process: the sharded drivers reduce to the plain public encode
    enc = ({"ranges": fc.encode_distributed, "balanced": fc.encode_balanced}.get(mode, fc.encode)
           if world > 1 else fc.encode)

    # a batch of independent images per rank (c3): encode_batch overlaps them
    # on several contexts / streams; every encode is synchronous at return,
    # so events on the first context's stream bracket the whole batch
    batch = len(gimgs) > 1 and not ranges
    n_ctx = int(os.environ.get("FC_BATCH_CONTEXTS", str(max(len(gimgs), 1))))
    bctxs = [ctx] + [_native.Context(local) for _ in range(n_ctx - 1)] if batch else [ctx]

    def step_device():
        if batch:
            return [r for _, r in fc.encode_batch(gimgs, cfg, contexts=bctxs, device_images=dimgs)]
        reps = []
        for g, d in zip(gimgs, dimgs):
            _, rep = enc(g, cfg, context=ctx, device_image=d)
            reps.append(rep)
        return reps

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    clocks = ClockSampler(local)
    launches0 = sum(bc.launch_count() for bc in bctxs)
    clocks.start()
    total_ms = main_ms = pool_ms = ent_ms = 0.0
    comps = alg_ops = 0
    level_rows = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = step_device()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
        for rep in reps:
            # this rank's own comparisons (its slab under range sharding), summed below
            for ls in rep.level_stats:
                comps += ls["comparisons"]
                if ls["path"] == _native.PATH_TENSOR:
                    n = fc.pool.LEVEL_RANGE_SIDES[ls["level"] - 1] ** 2
                    alg_ops += 2 * n * ls["comparisons"]
                    main_ms += ls["main_ms"]
        if not batch:
            pt = ctx.pool_times()
            ent_ms += pt[0]
            pool_ms += pt[2]
        level_rows = reps[0].level_stats
    torch.cuda.synchronize()
    barrier()
    launches = sum(bc.launch_count() for bc in bctxs) - launches0
    launches //= max(args.steps, 1)
    if batch:
        # overlapped builds share the device: the pool phase is measured on its
        # own, one image at a time on one context, outside the timed region
        for g, d in zip(gimgs, dimgs):
            fc.build_pool(g, cfg.pool, context=ctx, device_image=d)
            pt = ctx.pool_times()
            ent_ms += pt[0] * args.steps
            pool_ms += pt[2] * args.steps
    pixels_per_step = sum(im.size for im in imgs) if (rank == 0 or not ranges) else 0

    # e2e: public API from host pixels, result serialised to bytes; one
    # untimed call first (the host-image path's pinned upload buffers)
    def step_e2e():
        if batch:
            for stream_out, _ in fc.encode_batch(gimgs, cfg, contexts=bctxs):
                fc.serialize(stream_out)
        else:
            for g in gimgs:
                stream_out, _ = enc(g, cfg, context=ctx)
                fc.serialize(stream_out)

    step_e2e()
    e2e_t = 0.0
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        step_e2e()
        e2e_t += time.perf_counter() - t0
    clk = clocks.stop()  # sampled across both timed regions (device-timed and end-to-end)
    h2d = d2h = 0
    for g in gimgs:  # bytes that cross PCIe per step (counted from the buffers copied)
        _, rep = fc.encode(g, cfg, context=ctx)
        h2d += g.width * g.height                         # pixels
        d2h += 24 * rep.record_count                      # int32 [n, 6] leaf records
        d2h += sum(4 * s for s in rep.pool_sizes)         # pool coordinates (stream header)
        d2h += 4 * (16 + 8 + 2 * 4)                       # counts, fix pairs, survivor counts

    red = sharding.reduce_metrics(
        dict(step_ms_total=total_ms, e2e_s_total=e2e_t, kernel_ms_total=main_ms, comparisons=comps,
             pixels=pixels_per_step * args.steps, alg_ops=alg_ops), device=f"cuda:{local}")
    total_ms_all, e2e_all = red["step_ms_total"], red["e2e_s_total"]
    comps_all, pix_all = red["comparisons"], red["pixels"] / args.steps

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    value = comps_all / (total_ms_all * 1e-3)
    peaks = measured_peaks()
    peak = ctx.probe_int8_peak()
    peak_src = ("measured in-run on this B200: dense tcgen05.mma kind::i8 M=128 N=256 from smem, "
                "all SMs (fc_probe_int8_peak)")
    cub = cublas_int8_tops(torch)
    if cub:
        peak_src += f"; cuBLASLt int8 8192^3 in the same run: {cub:.0f} TOP/s"
    achieved = (alg_ops / (main_ms * 1e-3)) / 1e12 if main_ms > 0 else None
    # DRAM bytes per tc_scan_kernel launch from the committed ncu --set full
    # capture of this workload (dram__bytes_read.sum + dram__bytes_write.sum)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02", f"tc_scan_{args.workload}_traffic.json")
    if os.path.exists(tpath):
        prof = json.load(open(tpath))["launches"]
        if prof:
            traffic = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in prof) / len(prof)
    hbm = peaks.get("hbm_gbs", 6650.0)
    wins = window_count(wl, imgs[0].shape[1], imgs[0].shape[0]) * len(imgs) * args.steps
    ent_bytes = imgs[0].size * len(imgs) * args.steps + 8 * wins
    ent_gbs = ent_bytes / (ent_ms * 1e-3) / 1e9 if ent_ms > 0 else None
    line = {
        "metric": "range-domain comparisons/sec",
        "value": value,
        "unit": "comparisons/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms_all / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if ranges or wl.images > 1 else "weak",
        "vs_baseline": None,
        "dtype": "u8 x s8 -> s32 (int8 tensor cores), int64 keys",
        "data": "synthetic (seeded generators, workloads.py)",
        "config": {
            "workload": args.workload,
            "description": wl.description,
            "images_per_rank": len(imgs), "path": args.path,
            "sharding": {"ranges": "range slabs of one image, pool replicated, records all-gathered (NCCL)",
                         "balanced": "every level's ranges re-sliced evenly, results all-gathered per level (NCCL)",
                         }.get(mode, "independent images per rank, no data-path collective"),
            "l2": "flushed (512 MB write) before every timed step",
            "pool_sizes": list(reps[0].pool_sizes), "step_blocks": list(reps[0].step_blocks),
            "comparisons_per_step": comps_all / args.steps,
        },
        "encode_mpix_per_s": pix_all * args.steps / (total_ms_all * 1e-3) / 1e6,
        "e2e": {"value": comps_all / e2e_all, "unit": "comparisons/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "encode_mpix_per_s": pix_all * args.steps / e2e_all / 1e6,
                "timing": "wall clock around fc.encode(host image) + fc.serialize"},
        "gpu_launches": launches,
        "roofline": {
            "kernel": "tc_scan_kernel (tcgen05 kind::i8 contraction + fused argmin epilogue)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_ops": "2 * B^2 int8 MAC-ops per comparison (one MAC per pixel)",
            "kernel_ms_per_step": main_ms / args.steps,
        },
        "pool_roofline": {
            "kernel": "entropy_all_kernel (every lattice window of all 4 levels)",
            "bound": "hbm", "achieved": ent_gbs, "peak": hbm, "unit": "GB/s",
            "frac": (ent_gbs / hbm) if ent_gbs else None,
            "algorithmic_bytes": "image once + 8 B entropy key per window",
            "windows_per_s": wins / (ent_ms * 1e-3) if ent_ms > 0 else None,
            "entropy_ms_per_step": ent_ms / args.steps,
            "pool_ms_per_step": pool_ms / args.steps,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
            "binding_resource": ("not HBM: per window 2 * stride * D shared-memory histogram "
                                 "updates and up to 256 LUT loads + fp64 adds in numpy's pairwise "
                                 "order; latency / issue-bound (ncu at c5: 17% warps active, 46% "
                                 "issue; profiles/r02/SUMMARY.md)"),
        },
        "levels": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in ls.items()}
                   for ls in level_rows],
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"], line["parity"] = cpu_baseline_leg(args, fc, ctx, cfg, gimgs[0])
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def cpu_baseline_leg(args, fc, ctx, cfg, gimg):
    """One step of the CPU arm on this host plus parity of that sample."""
    threads = os.cpu_count() or 1
    cpu = CpuSample(args.workload, threads)
    comps, dt, desc, chk = cpu.step()
    base = {"value": comps / dt, "unit": "comparisons/s", "cores": threads, "kind": "port",
            "sample": f"{args.workload}: {desc} by oracle/ (C/OpenMP scan restating _scan.py), "
                      f"{dt:.2f} s"}
    if args.workload in SAMPLED:
        base["sample"] += f"; pool + operand setup {cpu.setup_s:.1f} s untimed"
    parity = {}
    if args.workload not in SAMPLED:
        img = fc.GrayImage(cpu.wl.image(chk["image"]))
        stream_out, _ = fc.encode(img, cfg, context=ctx)
        parity["stream_bytes_equal_to_oracle"] = fc.serialize(stream_out) == chk["bytes"]
        return base, parity
    rec, _, _ = fc.encode_shard(gimg, cfg, 0, 1, context=ctx)
    if args.workload == "c5":
        ok = 0
        for x, y, err, e, iso, si, off in chk["ranges"]:
            r = rec[((y // 16) * 128 + x // 16) * 4 + ((y % 16) // 8) * 2 + (x % 16) // 8]
            ok += (int(r[5]), int(r[3]), int(r[2]), int(r[4]), int(r[1])) == (err, e, iso, si, off)
        parity["sampled_ranges_equal_to_oracle"] = f"{ok}/{len(chk['ranges'])}"
    else:
        side = np.array([0, 16, 8, 4, 2])[rec[:, 0]]
        area = np.cumsum(side.astype(np.int64) ** 2)
        ends = np.searchsorted(area, np.arange(1, area[-1] // 256 + 1) * 256) + 1
        starts = np.concatenate([[0], ends])
        want = chk["leaves"]
        ok = total = 0
        for t in chk["tops"]:
            x0, y0 = (t % (gimg.width // 16)) * 16, (t // (gimg.width // 16)) * 16
            pos = [(x0, y0, 16)]
            got = rec[starts[t]:starts[t + 1]]
            # walk the block's depth-first leaves to their origins
            out = []
            for r in got:
                lvl = int(r[0])
                while True:
                    x, y, s = pos.pop()
                    if s == fc.pool.LEVEL_RANGE_SIDES[lvl - 1]:
                        out.append((lvl, x, y, r))
                        break
                    h = s // 2
                    pos += [(x + h, y + h, h), (x, y + h, h), (x + h, y, h), (x, y, h)]
            for lvl, x, y, r in out:
                total += 1
                exp = want.get((lvl, x, y))
                ok += exp is not None and exp == (int(r[5]), int(r[3]), int(r[2]), int(r[4]), int(r[1]))
        parity["sampled_subtree_leaves_equal_to_oracle"] = f"{ok}/{total} (of {len(want)} oracle leaves)"
    return base, parity


if __name__ == "__main__":
    sys.exit(main())
