#!/usr/bin/env python3
"""Benchmark: range-domain comparisons/sec of the B200 fractal encoder search.

Metric (BASELINE.json): range-domain comparisons/sec, with encode Mpixel/s
alongside.  A comparison is one (range, domain, isometry, s) candidate whose
exact SSD the reference evaluates (_scan.py:35-57); comparisons per level =
ranges * pool * 8 * |S|.

A "step" is one full encode of the workload image(s): entropy pools for all
levels, every quadtree level's exhaustive search, the split decisions and the
output records.  ``value`` is timed with CUDA events on the library's own
stream with the image already resident in HBM (L2 flushed between steps);
``e2e`` is the same encode through the public API ``fc.encode`` from host
pixels plus ``fc.serialize`` of the result, wall-clocked.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
        python bench.py --impl reference ...   (CPU oracle arm)
Multi-GPU: launched by torchrun; every rank encodes its own seeded image
(weak scaling, no collective on the data path); c3 splits its 64 images.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "c2"  # BASELINE.json configs[1]


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--path", default="auto", choices=["auto", "exact", "tensor"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="images", choices=["images", "ranges"],
                    help="images: weak scaling, one seeded image per rank (c3: its 64 images); "
                         "ranges: strong scaling, one image split into top-level slabs "
                         "(encode_distributed, records all-gathered over NCCL)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def images_for_rank(name: str, rank: int, world: int):
    """Weak scaling: one seeded image per rank; c3 shards its 64 images."""
    from paper_1502_00324_b200 import sharding, workloads as W

    wl = W.WORKLOADS[name]
    if wl.images > 1:
        return [wl.image(i) for i in sharding.images_for_rank(wl.images, rank, world)]
    return [wl.image(rank)]


def encoder_config(name: str, path: str):
    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import workloads as W

    wl = W.WORKLOADS[name]
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    caps = tuple(1 if one else 2**31 - 1 for one in wl.cap_one)
    params = fc.PoolParams(pool_cap=2**31 - 1, strides=wl.strides, level_caps=caps,
                           entropy_thresholds=taus)
    return fc.EncoderConfig(pool=params, thresholds=wl.thresholds, path=path)


def oracle_caps(name: str, img):
    """Reference-side pool caps for a workload image: #{entropy > tau}."""
    from oracle import fracodec_oracle as O
    from paper_1502_00324_b200 import workloads as W

    wl = W.WORKLOADS[name]
    caps = []
    for li in range(4):
        if wl.cap_one[li]:
            caps.append(1)
            continue
        _, _, ent = O.grid_entropies(img, O.LEVEL_DOMAIN_SIDES[li], wl.strides[li])
        caps.append(len(ent) if wl.taus[li] is None else max(1, int((ent > wl.taus[li]).sum())))
    return tuple(caps)


def oracle_encode(name: str, img, caps, threads: int):
    """One reference-algorithm encode on the host (oracle port; CPU arm)."""
    from oracle import fracodec_oracle as O
    from paper_1502_00324_b200 import workloads as W

    wl = W.WORKLOADS[name]
    t0 = time.perf_counter()
    enc = O.encode(img, caps, wl.strides, "proposed", wl.thresholds, threads=threads)
    dt = time.perf_counter() - t0
    comps = 0
    for level, (errs, _idx, _rm, _o) in enc.scans.items():
        comps += len(errs) * len(enc.pools[level - 1]) * 8 * len(enc.s_sets[level - 1])
    return enc, dt, comps


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


def measured_int8_peak(torch):
    """Dense int8 tensor-core peak measured in-run with cuBLASLt (torch._int_mm)."""
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
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12, "measured in-run: cuBLASLt int8 8192^3 (torch._int_mm), best of 5"
    except Exception as exc:  # noqa: BLE001
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        bf16 = peaks.get("bf16_tflops", 1590.0)
        return 2.0 * bf16, f"derived: 2 x measured bf16 dense ({bf16} TF/s); int8 probe failed: {exc}"


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)).get("hbm_gbs", 6650.0), "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback (B200_PROFILING.md)"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    img = images_for_rank(args.workload, 0, 1)[0]
    caps = oracle_caps(args.workload, img)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_encode(args.workload, img, caps, threads)
    total_t, total_c = 0.0, 0
    for _ in range(args.steps):
        _, dt, comps = oracle_encode(args.workload, img, caps, threads)
        total_t += dt
        total_c += comps
    value = total_c / total_t
    from paper_1502_00324_b200 import workloads as W

    line = {
        "impl": "reference", "metric": "range-domain comparisons/sec", "value": value,
        "unit": "comparisons/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "description": W.WORKLOADS[args.workload].description,
                   "caps": list(caps)},
        "cpu_baseline": {"value": value, "unit": "comparisons/s", "cores": threads, "kind": "port",
                         "sample": f"full {args.workload} encode (oracle/: numpy pool + C/OpenMP "
                                   f"exhaustive scan restating _scan.py), image seed 0"},
        "e2e": {"value": value, "unit": "comparisons/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native, workloads as W

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    ctx = _native.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", local))
    cfg = encoder_config(args.workload, args.path)
    ranges = args.shard == "ranges"
    # ranges: every rank holds the same image and encodes its slab of top-level
    # slots (encode_distributed all-gathers the records); images: weak scaling
    imgs = images_for_rank(args.workload, 0, 1)[:1] if ranges else images_for_rank(args.workload, rank, world)
    gimgs = [fc.GrayImage(im) for im in imgs]
    dimgs = [torch.from_numpy(im.copy()).cuda() for im in imgs]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")  # 512 MB > L2
    enc = fc.encode_distributed if ranges else fc.encode

    def step_device():
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
    launches0 = ctx.launch_count()
    clocks.start()
    total_ms = 0.0
    comps = 0
    main_ms = 0.0
    alg_ops = 0
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
            # this rank's own comparisons (its slab under --shard ranges), summed below
            comps += sum(ls["comparisons"] for ls in rep.level_stats)
            for ls in rep.level_stats:
                if ls["path"] == _native.PATH_TENSOR:
                    n = fc.pool.LEVEL_RANGE_SIDES[ls["level"] - 1] ** 2
                    alg_ops += 2 * n * ls["comparisons"]
                    main_ms += ls["main_ms"]
        level_rows = reps[0].level_stats
    torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count() - launches0
    pixels_per_step = sum(im.size for im in imgs) if (rank == 0 or not ranges) else 0

    # e2e: public API from host pixels, result serialised to bytes
    e2e_t = 0.0
    h2d = d2h = 0
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        for g in gimgs:
            stream_out, rep = enc(g, cfg, context=ctx)
            data = fc.serialize(stream_out)
        e2e_t += time.perf_counter() - t0
    clk = clocks.stop()  # sampled across both timed regions (device-timed and end-to-end)
    for g in gimgs:  # bytes that cross PCIe per step (counted from the buffers copied)
        _, rep = fc.encode(g, cfg, context=ctx)
        h2d += g.width * g.height                         # pixels
        d2h += 24 * rep.record_count                      # int32 [n, 6] leaf records
        d2h += sum(4 * s for s in rep.pool_sizes)         # pool coordinates (stream header)
        d2h += 4 * (16 + 8 + 2 * 4)                       # counts, fix pairs, survivor counts

    from paper_1502_00324_b200 import sharding

    red = sharding.reduce_metrics(
        dict(step_ms_total=total_ms, e2e_s_total=e2e_t, kernel_ms_total=main_ms, comparisons=comps,
             pixels=pixels_per_step * args.steps, alg_ops=alg_ops), device="cuda")
    total_ms_all, e2e_all = red["step_ms_total"], red["e2e_s_total"]
    comps_all, pix_all = red["comparisons"], red["pixels"] / args.steps

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    value = comps_all / (total_ms_all * 1e-3)
    peak = ctx.probe_int8_peak()
    peak_src = ("measured in-run on this B200: dense tcgen05.mma kind::i8 M=128 N=256 from smem, "
                "all SMs (fc_probe_int8_peak)")
    try:
        cublas, _ = measured_int8_peak(torch)
        peak_src += f"; cuBLASLt int8 8192^3 in the same run: {cublas:.0f} TOP/s"
    except Exception:  # noqa: BLE001
        pass
    achieved = (alg_ops / (main_ms * 1e-3)) / 1e12 if main_ms > 0 else None
    # DRAM bytes per tc_scan_kernel launch from the committed ncu --set full capture
    # (dram__bytes_read.sum + dram__bytes_write.sum, averaged over the c2 levels)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01", "tc_scan_c2_traffic.json")
    if args.workload == "c2" and os.path.exists(tpath):
        prof = json.load(open(tpath))["launches"]
        if prof:
            traffic = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in prof) / len(prof)
    line = {
        "metric": "range-domain comparisons/sec",
        "value": value,
        "unit": "comparisons/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms_all / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if ranges or W.WORKLOADS[args.workload].images > 1 else "weak",
        "vs_baseline": None,
        "dtype": "u8 x s8 -> s32 (int8 tensor cores), int64 keys",
        "data": "synthetic (seeded generators, workloads.py)",
        "config": {
            "workload": args.workload,
            "description": W.WORKLOADS[args.workload].description,
            "images_per_rank": len(imgs), "path": args.path,
            "sharding": ("range slabs of one image, pool replicated, records all-gathered (NCCL)"
                         if ranges else "independent images per rank, no data-path collective"),
            "l2": "flushed (512 MB write) before every timed step",
            "pool_sizes": list(reps[0].pool_sizes), "step_blocks": list(reps[0].step_blocks),
            "comparisons_per_step": comps_all / args.steps,
        },
        "encode_mpix_per_s": pix_all * args.steps / (total_ms_all * 1e-3) / 1e6,
        "e2e": {"value": comps_all / e2e_all, "unit": "comparisons/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "encode_mpix_per_s": pix_all * args.steps / e2e_all / 1e6,
                "timing": "wall clock around fc.encode(host image) + fc.serialize (pageable host buffers)"},
        "gpu_launches": launches,
        "roofline": {
            "kernel": "tc_scan_kernel (tcgen05 kind::i8 contraction + fused argmin epilogue)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_ops": "2 * B^2 int8 MAC-ops per comparison (one MAC per pixel)",
            "kernel_ms_per_step": main_ms / args.steps,
        },
        "levels": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in ls.items()}
                   for ls in level_rows],
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        img = imgs[0]
        caps = oracle_caps(args.workload, img)
        threads = os.cpu_count() or 1
        enc, dt, cc = oracle_encode(args.workload, img, caps, threads)
        from oracle import fracodec_oracle as O

        stream_out, _ = fc.encode(gimgs[0], cfg, context=ctx)
        line["cpu_baseline"] = {
            "value": cc / dt, "unit": "comparisons/s", "cores": threads, "kind": "port",
            "sample": f"one full {args.workload} encode of the rank-0 image by oracle/ "
                      f"(numpy pool + C/OpenMP scan restating _scan.py), {dt:.2f} s",
        }
        line["parity"] = {"stream_bytes_equal_to_oracle": fc.serialize(stream_out) == O.serialize(enc)}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
