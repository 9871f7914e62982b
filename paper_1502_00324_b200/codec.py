"""Four-step quadtree encoder (device search) and the iterative decoder.

``encode(image, config)`` keeps the reference's entry point and output
(codec.py:171-254 there): pool construction and every level's exhaustive
range-domain search run on the B200 through the C ABI; the host keeps the
quadtree bookkeeping (split rule codec.py:132-141, depth-first leaf order
codec.py:145-161) and assembles the records and the FRAK stream.

``decode`` / ``decode_trace`` are the reference's attractor iteration
(codec.py:269-363), run on the device (fc_decode); the host only lays out
the leaf table.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .image import GrayImage
from .matcher import BASELINE, PATHS, PROPOSED, SPolicy, split_index, stored_offsets
from .pool import LEVEL_RANGE_SIDES, CoordTable, PoolParams, build_pool, build_pool_sharded
from .stream import CompressedStream, RecordTable, header_bytes, leaf_origins

TOP_SIDE = 16


@dataclass(frozen=True)
class EncoderConfig:
    pool: PoolParams
    policy: SPolicy = field(default_factory=SPolicy)
    thresholds: tuple = (8.0, 8.0, 8.0)
    threads: int | None = None  # accepted for interface parity; the search runs on the GPU
    path: str = "auto"  # "auto" | "exact" | "tensor" (device kernel choice)

    def __post_init__(self):
        if len(self.thresholds) != 3 or any(t <= 0 for t in self.thresholds):
            raise ValueError("thresholds must be 3 positive RMS values")
        object.__setattr__(self, "thresholds", tuple(float(t) for t in self.thresholds))
        if self.path not in PATHS:
            raise ValueError(f"path must be one of {sorted(PATHS)}")


@dataclass
class EncodeReport:
    width: int
    height: int
    mode: str
    pool_cap: int
    pool_sizes: tuple
    strides: tuple
    thresholds: tuple
    step_blocks: tuple
    record_count: int
    collage_ssd: int
    payload_bits: int
    header_bytes: int
    file_bytes: int
    bpp_payload: float
    bpp_total: float
    comp_ratio_payload: float
    comp_ratio_total: float
    pool_time_s: float
    encode_time_s: float
    comparisons: int = 0
    scan_device_ms: float = 0.0
    level_stats: list = field(default_factory=list)  # per matched level: device counters
    phase_ms: dict = field(default_factory=dict)       # host wall time per encode phase

    def to_lines(self) -> list:
        rows = [
            ("width", self.width), ("height", self.height), ("mode", self.mode),
            ("pool_cap", self.pool_cap),
            ("pool_sizes", ",".join(str(v) for v in self.pool_sizes)),
            ("strides", ",".join(str(v) for v in self.strides)),
            ("thresholds", ",".join(f"{t:g}" for t in self.thresholds)),
            ("step1_blocks", self.step_blocks[0]), ("step2_blocks", self.step_blocks[1]),
            ("step3_blocks", self.step_blocks[2]), ("step4_blocks", self.step_blocks[3]),
            ("records", self.record_count), ("collage_ssd", self.collage_ssd),
            ("payload_bits", self.payload_bits), ("header_bytes", self.header_bytes),
            ("file_bytes", self.file_bytes), ("bpp_payload", f"{self.bpp_payload:.6f}"),
            ("bpp_total", f"{self.bpp_total:.6f}"),
            ("comp_ratio_payload", f"{self.comp_ratio_payload:.4f}"),
            ("comp_ratio_total", f"{self.comp_ratio_total:.4f}"),
            ("pool_time_s", f"{self.pool_time_s:.3f}"),
            ("encode_time_s", f"{self.encode_time_s:.3f}"),
        ]
        return [f"{k}={v}" for k, v in rows]


def _quadtree(width: int, height: int, thresholds, match_fn):
    """Vectorised level loop with the reference's split rule and DFS order.

    match_fn(level, origins[int32 M,2]) -> errs.  Returns (per-level origin
    arrays, leaves as (level, j) arrays in depth-first order).
    """
    ys, xs = np.mgrid[0:height:TOP_SIDE, 0:width:TOP_SIDE]
    origins = {1: np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.int32)}
    # DFS sort code: top index * 64 + d1 * 16 + d2 * 4 + d3 (children TL, TR, BL, BR = 0..3)
    codes = {1: np.arange(origins[1].shape[0], dtype=np.int64) * 64}
    leaf_level, leaf_j, leaf_code = [], [], []
    for level in (1, 2, 3, 4):
        o = origins.get(level)
        if o is None or o.shape[0] == 0:
            break
        errs = np.asarray(match_fn(level, o))
        side = LEVEL_RANGE_SIDES[level - 1]
        if level == 4:
            split = np.zeros(o.shape[0], dtype=bool)
        else:
            split = errs > thresholds[level - 1] ** 2 * side * side
        keep = np.nonzero(~split)[0]
        leaf_level.append(np.full(keep.shape[0], level, dtype=np.int64))
        leaf_j.append(keep)
        leaf_code.append(codes[level][keep])
        par = np.nonzero(split)[0]
        if par.shape[0]:
            h = side // 2
            offs = np.array([[0, 0], [h, 0], [0, h], [h, h]], dtype=np.int32)
            origins[level + 1] = (o[par][:, None, :] + offs[None]).reshape(-1, 2)
            weight = 4 ** (3 - level)
            codes[level + 1] = (codes[level][par][:, None]
                                + np.arange(4, dtype=np.int64)[None] * weight).reshape(-1)
    lv = np.concatenate(leaf_level)
    jj = np.concatenate(leaf_j)
    cc = np.concatenate(leaf_code)
    order = np.argsort(cc, kind="stable")
    return origins, lv[order], jj[order]


def run_quadtree(width: int, height: int, thresholds, match_level):
    """Reference-compatible driver (codec.py:114-161): match_level(level,
    origins as a list of (x, y)) -> errs; returns leaves (level, x, y, j)."""
    origins, lv, jj = _quadtree(
        width, height, thresholds,
        lambda level, o: match_level(level, [(int(x), int(y)) for x, y in o]))
    leaves = [(int(level), int(origins[level][j, 0]), int(origins[level][j, 1]), int(j))
              for level, j in zip(lv, jj)]
    covered = sum(LEVEL_RANGE_SIDES[level - 1] ** 2 for level, _, _, _ in leaves)
    assert covered == width * height, "leaf footprints must tile the image"
    return leaves


def encode(image: GrayImage, config: EncoderConfig, context=None, device_image=None, pool=None):
    """Compress an image whose sides are multiples of 16 -> (CompressedStream, EncodeReport).

    codec.py:114-224 semantics.  The whole quadtree runs on the device
    (fc_encode: split tests, child ranges and depth-first records never leave
    HBM; one host synchronisation per level).  ``device_image``: optional
    HBM-resident copy of the pixels (see build_pool).
    """
    if image.width % 16 or image.height % 16:
        raise ValueError(f"dimensions not multiple of 16: {image.width}x{image.height}")
    t_start = time.perf_counter()
    ctx = context if context is not None else _native.default_context()
    if pool is None:  # else: built on this context already (encode_batch)
        pool = build_pool(image, config.pool, context=ctx, device_image=device_image)
    pool_time = time.perf_counter() - t_start
    policy = config.policy
    baseline = policy.mode == BASELINE
    s_sets = tuple(policy.s_set(level) for level in (1, 2, 3, 4))
    t_q = time.perf_counter()
    rec = ctx.encode(config.thresholds, baseline, s_sets, PATHS[config.path],
                     capacity=image.width * image.height // 4)
    t_r = time.perf_counter()
    phase = {"pool": 1e3 * pool_time, "quadtree": 1e3 * (t_r - t_q)}
    level_stats = _level_stats(ctx)
    comparisons = sum(ls["comparisons"] for ls in level_stats)
    scan_ms = sum(ls["scan_ms"] for ls in level_stats)
    records = RecordTable._trusted(rec[:, :5])  # int32 view of the device records
    stream = CompressedStream(
        width=image.width, height=image.height, mode=policy.mode, strides=pool.params.strides,
        s_sets=s_sets, pools=pool.all_coords(), records=records)
    encode_time = time.perf_counter() - t_start
    phase["records_stream"] = 1e3 * (time.perf_counter() - t_r)
    step_blocks, collage_ssd = ctx.encode_summary()
    return stream, _report(image, config, pool, stream, step_blocks, collage_ssd,
                           pool_time, encode_time, comparisons, scan_ms, level_stats, phase)


def encode_shard(image: GrayImage, config: EncoderConfig, rank: int, world: int, context=None,
                 device_image=None, pool=None):
    """Range sharding: this rank's contiguous raster slab of
    16x16 top-level slots (sharding.slab_for_rank), encoded against the full,
    replicated pool -> (int32 records [n, 6] of the slab in depth-first
    order, DomainPool, per-level statistics of the slab as in EncodeReport).  Slabs of ranks 0..world-1
    concatenate into exactly encode()'s record list: a top-level block's
    subtree depends only on its own errors (codec.py:134-142)."""
    from . import sharding

    if image.width % 16 or image.height % 16:
        raise ValueError(f"dimensions not multiple of 16: {image.width}x{image.height}")
    ctx = context if context is not None else _native.default_context()
    if pool is None:  # else: built on this context already (e.g. build_pool_sharded)
        pool = build_pool(image, config.pool, context=ctx, device_image=device_image)
    policy = config.policy
    s_sets = tuple(policy.s_set(level) for level in (1, 2, 3, 4))
    n_top = (image.width // 16) * (image.height // 16)
    begin, end = sharding.slab_for_rank(n_top, rank, world)
    if begin == end:
        return np.zeros((0, 6), dtype=np.int32), pool, []
    ctx.set_top_slab(begin, end)
    try:
        rec = ctx.encode(config.thresholds, policy.mode == BASELINE, s_sets, PATHS[config.path],
                         capacity=(end - begin) * 256)
    finally:
        ctx.set_top_slab(0, -1)
    return np.array(rec, dtype=np.int32), pool, _level_stats(ctx)


def _level_stats(ctx) -> list:
    out = []
    for level in (1, 2, 3, 4):
        st = ctx.encode_level_stats(level)
        if st.ranges == 0:
            continue
        out.append(dict(level=level, ranges=int(st.ranges), columns=int(st.columns),
                        comparisons=int(st.comparisons), path=int(st.path),
                        launches=int(st.kernel_launches), scan_ms=float(st.scan_ms),
                        main_ms=float(st.main_ms), fix_ms=float(st.fix_ms),
                        fix_pairs=int(st.fix_pairs), rescans=int(st.rescans)))
    return out


def encode_distributed(image: GrayImage, config: EncoderConfig, context=None, device_image=None):
    """Range-sharded encode over the initialised torch.distributed group (one
    process per GPU): the pool's entropy pass is sharded by window rows and
    all-gathered, every rank ranks the same windows into the replicated pool
    (build_pool_sharded) and encodes its slab (encode_shard), the records are
    all-gathered (NCCL over NVLink for a CUDA context; the collectives run on
    the context's device) and every rank returns the full (CompressedStream,
    EncodeReport) -- byte-identical to encode()."""
    import torch.distributed as dist

    from . import sharding

    t_start = time.perf_counter()
    ctx = context if context is not None else _native.default_context()
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank() if dist_on else 0
    world = dist.get_world_size() if dist_on else 1
    coll = _collective_device(ctx)
    # the entropy pass sharded by window rows, then every rank ranks the
    # all-gathered windows (the same pool everywhere)
    pool = build_pool_sharded(image, config.pool, context=ctx, device_image=device_image,
                              collective_device=coll)
    rec, pool, level_stats = encode_shard(image, config, rank, world, ctx, device_image, pool=pool)
    allrec = sharding.gather_rows(rec, device=coll)
    policy = config.policy
    s_sets = tuple(policy.s_set(level) for level in (1, 2, 3, 4))
    stream = CompressedStream(
        width=image.width, height=image.height, mode=policy.mode, strides=pool.params.strides,
        s_sets=s_sets, pools=pool.all_coords(), records=RecordTable._trusted(allrec[:, :5]))
    step_blocks = tuple(int(v) for v in np.bincount(allrec[:, 0], minlength=5)[1:5])
    collage_ssd = int(allrec[:, 5].sum(dtype=np.int64))
    encode_time = time.perf_counter() - t_start
    comparisons = image_comparisons(step_blocks, pool.sizes, s_sets)
    # comparisons: the whole image (all ranks, from the gathered leaves);
    # level_stats: this rank's slab
    return stream, _report(image, config, pool, stream, step_blocks, collage_ssd, 0.0, encode_time,
                           comparisons, sum(ls["scan_ms"] for ls in level_stats), level_stats,
                           {"sharded_ranks": world})


_BATCH_CONTEXTS = {}


def encode_batch(images, config: EncoderConfig, contexts=None, device_images=None,
                 workers: int = 8):
    """Encode a batch of independent images (the c3 workload) -> list of
    (CompressedStream, EncodeReport) in input order, each identical to
    encode(image, config).

    Small images leave most of the GPU idle inside one encode, so the batch
    is spread over ``workers`` contexts -- each its own CUDA stream, device
    buffers and graph -- driven from host threads (the C calls release the
    GIL), and the encodes overlap on the device."""
    from concurrent.futures import ThreadPoolExecutor

    images = list(images)
    if contexts is None:
        dev = _native.default_context().device
        ctxs = _BATCH_CONTEXTS.setdefault(dev, [])
        while len(ctxs) < workers:
            ctxs.append(_native.Context(dev))
        contexts = ctxs[:workers]
    contexts = list(contexts)
    n = len(contexts)
    out = [None] * len(images)
    same_size = len({(im.width, im.height) for im in images}) == 1
    if n >= len(images) > 1 and same_size:
        # a context per image: every image's entropy pass in one pair of
        # launches (small images leave the GPU idle one at a time), then
        # per-context ranking and encode from the worker threads
        from .pool import DomainPool, _adopt_device_image

        ctxs = contexts[:len(images)]

        def set_one(i):
            if device_images is not None:
                _adopt_device_image(ctxs[i], device_images[i], images[i])
            else:
                ctxs[i].set_image(images[i].pixels)

        def run_one(i):
            c = ctxs[i]
            pool = DomainPool(config.pool, images[i].width, images[i].height, c.pool_rank(), c)
            out[i] = encode(images[i], config, context=c, pool=pool)

        # host pixels: the uploads (staging copies) in parallel; device
        # images: adopted from this thread (measured: adopting them from the
        # worker threads delayed the shared launch, c3 14.9 -> 18.7 ms)
        par = device_images is None
        with ThreadPoolExecutor(max_workers=min(workers, len(images))) as ex:
            if par:
                for f in [ex.submit(set_one, i) for i in range(len(images))]:
                    f.result()
            else:
                for i in range(len(images)):
                    set_one(i)
            _native.Context.pool_entropy_batch(ctxs, *config.pool.native_args())
            for f in [ex.submit(run_one, i) for i in range(len(images))]:
                f.result()
        return out

    def run(w):
        for i in range(w, len(images), n):
            dimg = device_images[i] if device_images is not None else None
            out[i] = encode(images[i], config, context=contexts[w], device_image=dimg)

    if n == 1 or len(images) <= 1:
        run(0) if n == 1 else [run(w) for w in range(n)]
        return out
    with ThreadPoolExecutor(max_workers=n) as ex:
        for f in [ex.submit(run, w) for w in range(n)]:
            f.result()
    return out


def _collective_device(ctx) -> str:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return f"cuda:{ctx.device}"


def encode_balanced(image: GrayImage, config: EncoderConfig, context=None, device_image=None):
    """Range-sharded encode with per-level re-balancing: the
    level-wise driver with every level's ranges split evenly over the ranks
    (encode_levelwise(balanced=True)); the collective per level is one
    all-gather of the level's (err, index, mean) rows."""
    return encode_levelwise(image, config, context, device_image, balanced=True)


def image_comparisons(step_blocks, pool_sizes, s_sets) -> int:
    """Comparisons of a whole encode from its leaf counts: the level-l ranges
    are the quadtree nodes at depth l, and the leaves at levels >= l cover
    exactly their area (every split has four children, codec.py:141), so
    ranges_l = sum_{k >= l} leaves_k / 4^(k - l)."""
    total = 0
    for level in (1, 2, 3, 4):
        area = sum(step_blocks[k - 1] * 4 ** (4 - k) for k in range(level, 5))  # in 2x2 units
        ranges = area // 4 ** (4 - level)
        total += ranges * int(pool_sizes[level - 1]) * 8 * len(s_sets[level - 1])
    return total


def _report(image, config, pool, stream, step_blocks, collage_ssd, pool_time, encode_time,
            comparisons, scan_ms, level_stats, phase) -> "EncodeReport":
    pixels = image.width * image.height
    payload = sum(c * stream.record_bits(lv) for lv, c in zip((1, 2, 3, 4), step_blocks))
    head = header_bytes(stream)
    file_bytes = head + (payload + 7) // 8
    return EncodeReport(
        width=image.width, height=image.height, mode=config.policy.mode,
        pool_cap=config.pool.pool_cap, pool_sizes=pool.sizes, strides=pool.params.strides,
        thresholds=config.thresholds, step_blocks=step_blocks, record_count=len(stream.records),
        collage_ssd=collage_ssd, payload_bits=payload, header_bytes=head, file_bytes=file_bytes,
        bpp_payload=payload / pixels, bpp_total=file_bytes * 8 / pixels,
        comp_ratio_payload=pixels * 8 / payload if payload else float("inf"),
        comp_ratio_total=pixels / file_bytes, pool_time_s=pool_time, encode_time_s=encode_time,
        comparisons=comparisons, scan_device_ms=scan_ms, level_stats=level_stats, phase_ms=phase)


def encode_levelwise(image: GrayImage, config: EncoderConfig, context=None, device_image=None,
                     balanced: bool = False):
    """Same result as encode(), driven level by level from the host through the
    match_level seam (fc_level_prepare + fc_match_level):
    the host runs the split test and builds the child origins.

    balanced=True (one process per GPU, torch.distributed initialised): every
    level's range list is re-sliced evenly over the ranks and the shares'
    results all-gathered (sharding.balanced_match), so data-dependent splits
    never leave a rank with more than its share of a level; every rank
    returns the full, byte-identical stream."""
    if image.width % 16 or image.height % 16:
        raise ValueError(f"dimensions not multiple of 16: {image.width}x{image.height}")
    t_start = time.perf_counter()
    ctx = context if context is not None else _native.default_context()
    if balanced:  # the entropy pass sharded over the ranks too (build_pool_sharded)
        pool = build_pool_sharded(image, config.pool, context=ctx, device_image=device_image,
                                  collective_device=_collective_device(ctx))
    else:
        pool = build_pool(image, config.pool, context=ctx, device_image=device_image)
    pool_time = time.perf_counter() - t_start
    policy = config.policy
    baseline = policy.mode == BASELINE
    path = PATHS[config.path]
    scans = {}
    comparisons = 0
    scan_ms = 0.0
    level_stats = []
    phase = {"pool": 1e3 * pool_time}

    def match_fn(level, o):
        nonlocal comparisons, scan_ms
        if pool.size(level) == 0:
            from .errors import EmptyPoolError

            raise EmptyPoolError(f"no domain entries at level {level}")
        lvl_path = path
        if path == _native.PATH_TENSOR and level == 4:
            lvl_path = _native.PATH_EXACT  # the contraction covers B >= 4 (both modes)
        t0 = time.perf_counter()
        ctx.level_prepare(level, baseline, policy.s_set(level), lvl_path)
        t1 = time.perf_counter()
        if balanced:
            from . import sharding

            err, idx, rmean = sharding.balanced_match(
                lambda share: ctx.match_level(level, share), np.asarray(o, dtype=np.int32),
                device=_collective_device(ctx))
        else:
            err, idx, rmean = ctx.match_level(level, o)
        t2 = time.perf_counter()
        phase[f"prepare_l{level}"] = 1e3 * (t1 - t0)
        phase[f"match_l{level}"] = 1e3 * (t2 - t1)
        st = ctx.stats()
        comparisons += int(st.comparisons)
        scan_ms += float(st.scan_ms)
        level_stats.append(dict(level=level, ranges=int(st.ranges), columns=int(st.columns),
                                comparisons=int(st.comparisons), path=int(st.path),
                                launches=int(st.kernel_launches), scan_ms=float(st.scan_ms),
                                main_ms=float(st.main_ms), fix_ms=float(st.fix_ms),
                                fix_pairs=int(st.fix_pairs), rescans=int(st.rescans)))
        scans[level] = (err, idx, rmean)
        return err

    t_q = time.perf_counter()
    origins, leaf_lv, leaf_j = _quadtree(image.width, image.height, config.thresholds, match_fn)
    t_r = time.perf_counter()
    phase["quadtree"] = 1e3 * (t_r - t_q)

    n = leaf_lv.shape[0]
    steps = leaf_lv
    offs = np.empty(n, dtype=np.int64)
    isos = np.empty(n, dtype=np.int64)
    addrs = np.empty(n, dtype=np.int64)
    sidx = np.empty(n, dtype=np.int64)
    errs = np.empty(n, dtype=np.int64)
    for level in (1, 2, 3, 4):
        sel = np.nonzero(leaf_lv == level)[0]
        if sel.shape[0] == 0:
            continue
        err, idx, rmean = scans[level]
        j = leaf_j[sel]
        S = len(policy.s_set(level))
        e, iso, si = split_index(idx[j], S)
        o = stored_offsets(rmean[j], e, si, policy.s_set(level),
                           pool.means(level) if baseline else None, baseline)
        offs[sel], isos[sel], addrs[sel], sidx[sel], errs[sel] = o, iso, e, si, err[j]
    records = RecordTable(np.stack([steps, offs, isos, addrs, sidx], axis=1))
    stream = CompressedStream(
        width=image.width, height=image.height, mode=policy.mode, strides=pool.params.strides,
        s_sets=tuple(policy.s_set(level) for level in (1, 2, 3, 4)),
        pools=tuple(pool.coords(level) for level in (1, 2, 3, 4)), records=records)
    encode_time = time.perf_counter() - t_start
    phase["records_stream"] = 1e3 * (time.perf_counter() - t_r)
    step_blocks = tuple(int((leaf_lv == lv).sum()) for lv in (1, 2, 3, 4))
    return stream, _report(image, config, pool, stream, step_blocks, int(errs.sum()), pool_time,
                           encode_time, comparisons, scan_ms, level_stats, phase)


# ---------------------------------------------------------------------------
# decoder (codec.py:257-363 semantics, on the device: fc_decode)
# ---------------------------------------------------------------------------

def decode_trace(stream: CompressedStream, iterations: int = 15, tolerance: int = 0,
                 context=None):
    """Iterate the collage map from a constant-128 image (codec.py:339-363):
    -> (GrayImage, per-pass max |delta|), stopping once a pass changes no
    pixel by more than ``tolerance``.  Runs on the device (fc_decode: one
    launch per pass, one host synchronisation per decode); bit-identical to
    the reference's host decoder (tests/test_gpu_parity.py against oracle/)."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if tolerance < 0:
        raise ValueError("tolerance must be >= 0")
    ctx = context if context is not None else _native.default_context()
    leaves = decoder_leaves(stream)
    img, deltas = ctx.decode(leaves, stream.width, stream.height, stream.s_sets,
                             stream.mode == PROPOSED, iterations, tolerance)
    return GrayImage(img), deltas


def decode(stream: CompressedStream, iterations: int = 15, tolerance: int = 0,
           context=None) -> GrayImage:
    return decode_trace(stream, iterations, tolerance, context)[0]


def decoder_leaves(stream: CompressedStream) -> np.ndarray:
    """int32 [leaves, 8] rows (x, y, step, domain x, domain y, isometry, s
    index, offset) in record order: the decoder kernel's input."""
    rec = stream.records.array if isinstance(stream.records, RecordTable) else \
        RecordTable(stream.records).array
    x, y, _side = leaf_origins(stream)
    out = np.empty((rec.shape[0], 8), dtype=np.int32)
    out[:, 0], out[:, 1], out[:, 2] = x, y, rec[:, 0]
    for level in (1, 2, 3, 4):
        sel = rec[:, 0] == level
        if sel.any():
            p = stream.pools[level - 1]
            # (a CoordTable passed to np.asarray would be walked as a Python sequence)
            coords = np.asarray(p.array if isinstance(p, CoordTable) else CoordTable(p).array,
                                dtype=np.int32)
            out[sel, 3:5] = coords[rec[sel, 3]]
    out[:, 5], out[:, 6], out[:, 7] = rec[:, 2], rec[:, 4], rec[:, 1]
    return out


# device names kept for callers of the earlier API
decode_trace_device = decode_trace
decode_device = decode
