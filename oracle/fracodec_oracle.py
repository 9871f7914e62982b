"""CPU restatement of the fracodec encoder (test infrastructure only).

Every function cites the reference line(s) it restates (paths relative to
``/root/reference/pkg/src/fracodec``).  Arithmetic follows the reference
exactly: numpy float64 with IEEE round-half-to-even (``np.rint``), floor 2x2
decimation, exact int64 SSDs, first strict minimum over the candidate order
(domain, isometry, s index).  The exhaustive scan itself runs in C
(``oracle/scan_oracle.c``, OpenMP over ranges like the reference's numba
``prange``); a pure numpy scan is kept for tiny cases and as a cross-check.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
from dataclasses import dataclass

import numpy as np

LEVEL_RANGE_SIDES = (16, 8, 4, 2)  # pool.py:20
LEVEL_DOMAIN_SIDES = (32, 16, 8, 4)  # pool.py:21
DEFAULT_STRIDES = (8, 4, 2, 2)  # pool.py:23
ENTROPY_CHUNK = 4096  # pool.py:25
DEFAULT_BASELINE_SET = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0)  # matcher.py:30
DEFAULT_PROPOSED_SETS = ((0.1,), (0.2, 0.4), (0.3, 0.8), (0.5, 0.9))  # matcher.py:31
TOP_SIDE = 16  # codec.py:30


# ---------------------------------------------------------------------------
# raster primitives
# ---------------------------------------------------------------------------

def decimate(tile: np.ndarray) -> np.ndarray:
    """2x2 mean with floor rounding on the last two axes (image.py:116-130)."""
    t = np.asarray(tile).astype(np.int32)
    s = t[..., 0::2, 0::2] + t[..., 0::2, 1::2] + t[..., 1::2, 0::2] + t[..., 1::2, 1::2]
    return (s // 4).astype(np.uint8)


def isometry_index_map(side: int, iso: int) -> np.ndarray:
    """Flat source index per output pixel for isometry ``iso``.

    Restates image.py:140-155 (0-3 clockwise rotations, 4-7 the same rotation
    followed by a left-right mirror) as explicit maps: out[i][j] = t[src].
    """
    b = side - 1
    i, j = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    rows, cols = {
        0: (i, j),
        1: (b - j, i),
        2: (b - i, b - j),
        3: (j, b - i),
        4: (i, b - j),
        5: (j, i),
        6: (b - i, j),
        7: (b - j, b - i),
    }[iso]
    return (rows * side + cols).ravel()


def apply_isometry(tile: np.ndarray, iso: int) -> np.ndarray:
    """Isometry on the last two (square) axes (image.py:140-155)."""
    t = np.asarray(tile)
    side = t.shape[-1]
    flat = t.reshape(t.shape[:-2] + (side * side,))
    return flat[..., isometry_index_map(side, iso)].reshape(t.shape)


# ---------------------------------------------------------------------------
# domain pool (pool.py)
# ---------------------------------------------------------------------------

def entropy_from_counts(counts: np.ndarray, n: int) -> np.ndarray:
    """Rows of 256-bin counts -> entropy in nats (pool.py:88-92).

    Uses numpy's own division, log and pairwise row sum so the float bits are
    the reference's on the same host.
    """
    p = counts / n
    terms = p * np.log(np.where(counts > 0, p, 1.0))
    return -terms.sum(axis=1)


def grid_entropies(pixels: np.ndarray, side: int, stride: int):
    """Raster-order lattice windows and their entropies (pool.py:120-135)."""
    h, w = pixels.shape
    ny = (h - side) // stride + 1
    nx = (w - side) // stride + 1
    ys = np.repeat(np.arange(ny) * stride, nx)
    xs = np.tile(np.arange(nx) * stride, ny)
    n = side * side
    ent = np.empty(ny * nx)
    view = np.lib.stride_tricks.sliding_window_view(pixels, (side, side))[::stride, ::stride]
    flat = view.reshape(ny * nx, n)
    for lo in range(0, flat.shape[0], ENTROPY_CHUNK):
        part = flat[lo : lo + ENTROPY_CHUNK].astype(np.int64)
        rows = part.shape[0]
        key = (np.arange(rows, dtype=np.int64)[:, None] << 8) | part
        counts = np.bincount(key.ravel(), minlength=rows * 256).reshape(rows, 256)
        ent[lo : lo + rows] = entropy_from_counts(counts, n)
    return xs, ys, ent


def candidate_count(width: int, height: int, side: int, stride: int) -> int:
    """Lattice placements of a side x side square (pool.py:106-117)."""
    if side > width or side > height:
        return 0
    return ((width - side) // stride + 1) * ((height - side) // stride + 1)


@dataclass
class OraclePoolLevel:
    xs: np.ndarray  # int64 [E] rank order
    ys: np.ndarray
    entropy: np.ndarray  # float64 [E]
    tiles: np.ndarray  # uint8 [E, B, B] decimated
    means: np.ndarray  # float64 [E]
    cnorm: np.ndarray  # float64 [E]


def build_pool_level(pixels: np.ndarray, level: int, stride: int, cap: int) -> OraclePoolLevel:
    """Rank, truncate and describe one level's pool (pool.py:138-178)."""
    side = LEVEL_DOMAIN_SIDES[level - 1]
    h, w = pixels.shape
    if side > w or side > h:
        raise ValueError(f"level {level} domain side {side} exceeds image {w}x{h}")
    xs, ys, ent = grid_entropies(pixels, side, stride)
    order = np.argsort(-ent, kind="stable")[:cap]
    xs, ys, ent = xs[order], ys[order], ent[order]
    view = np.lib.stride_tricks.sliding_window_view(pixels, (side, side))
    tiles = decimate(view[ys, xs])
    flat = tiles.reshape(len(order), -1).astype(np.int64)
    n = flat.shape[1]
    s1 = flat.sum(axis=1)
    s2 = (flat * flat).sum(axis=1)
    means = s1 / n
    cnorm = s2 - s1 * s1 / n
    return OraclePoolLevel(xs, ys, ent, tiles, means, cnorm)


def level_caps_for_threshold(pixels: np.ndarray, strides, taus) -> tuple:
    """Map entropy thresholds tau_l onto reference caps: #{ent > tau}.

    ``None`` keeps the whole level.  Caps are floored at 1 (PoolParams
    requires positive caps, pool.py:47-48).
    """
    caps = []
    for li in range(4):
        side = LEVEL_DOMAIN_SIDES[li]
        tau = taus[li]
        if tau is None:
            caps.append(max(1, candidate_count(pixels.shape[1], pixels.shape[0], side, strides[li])))
            continue
        _, _, ent = grid_entropies(pixels, side, strides[li])
        caps.append(max(1, int((ent > tau).sum())))
    return tuple(caps)


# ---------------------------------------------------------------------------
# candidate operands and the scan (matcher.py, _scan.py)
# ---------------------------------------------------------------------------

def candidate_operands(tiles: np.ndarray, means: np.ndarray, svals, baseline: bool):
    """q[(e*8+iso)*S+si, :] as int16 (matcher.py:143-159)."""
    E, B, _ = tiles.shape
    t = tiles.astype(np.float64)
    if not baseline:
        t = t - means[:, None, None]
    sv = np.asarray(svals, dtype=np.float64)
    bases = np.rint(sv[None, :, None, None] * t[:, None, :, :]).astype(np.int16)  # [E,S,B,B]
    S = sv.shape[0]
    q = np.empty((E, 8, S, B * B), dtype=np.int16)
    flat = bases.reshape(E, S, B * B)
    for iso in range(8):
        q[:, iso] = flat[:, :, isometry_index_map(B, iso)]
    return np.ascontiguousarray(q.reshape(E * 8 * S, B * B))


# ---------------------------------------------------------------------------
# full-size helpers (BASELINE c4/c5: millions of windows) -- same arithmetic,
# bounded memory, bands of window rows on several host processes
# ---------------------------------------------------------------------------

def _entropy_band(args):
    pixels, side, stride, y0, ny = args
    sub = pixels[y0 * stride : (y0 + ny - 1) * stride + side]
    return grid_entropies(sub, side, stride)[2]


def grid_entropies_parallel(pixels: np.ndarray, side: int, stride: int, workers: int = 0):
    """grid_entropies (pool.py:120-135) over bands of window rows on several
    processes.  Every window's entropy is a function of its own 256 counts
    only (pool.py:88-92 reduces each row separately), so the bands
    concatenate into exactly the single-process result."""
    h, w = pixels.shape
    ny = (h - side) // stride + 1
    nx = (w - side) // stride + 1
    ys = np.repeat(np.arange(ny) * stride, nx)
    xs = np.tile(np.arange(nx) * stride, ny)
    workers = workers or os.cpu_count() or 1
    if workers <= 1 or ny * nx < 200_000:
        return grid_entropies(pixels, side, stride)
    import concurrent.futures as cf
    import multiprocessing as mp

    per = max(1, -(-ny // (4 * workers)))
    jobs = [(pixels, side, stride, y0, min(per, ny - y0)) for y0 in range(0, ny, per)]
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("forkserver")) as ex:
        parts = list(ex.map(_entropy_band, jobs))
    return xs, ys, np.concatenate(parts)


def pool_order(pixels: np.ndarray, level: int, stride: int, cap: int, workers: int = 0):
    """Rank order of one level's pool (pool.py:171: argsort(-ent, stable)[:cap])
    -> (xs, ys, ent) in rank order, without tiles."""
    side = LEVEL_DOMAIN_SIDES[level - 1]
    xs, ys, ent = grid_entropies_parallel(pixels, side, stride, workers)
    order = np.argsort(-ent, kind="stable")[:cap]
    return xs[order], ys[order], ent[order]


def pool_tiles(pixels: np.ndarray, level: int, xs, ys, chunk: int = 1 << 18):
    """Decimated tiles, means and centered norms of the domains at (xs, ys)
    (image.py:116-130, pool.py:138-152), in chunks."""
    side = LEVEL_DOMAIN_SIDES[level - 1]
    b = side // 2
    view = np.lib.stride_tricks.sliding_window_view(pixels, (side, side))
    E = len(xs)
    tiles = np.empty((E, b, b), dtype=np.uint8)
    means = np.empty(E)
    cnorm = np.empty(E)
    for lo in range(0, E, chunk):
        hi = min(E, lo + chunk)
        t = decimate(view[ys[lo:hi], xs[lo:hi]])
        tiles[lo:hi] = t
        flat = t.reshape(hi - lo, -1).astype(np.int64)
        s1 = flat.sum(axis=1)
        s2 = (flat * flat).sum(axis=1)
        means[lo:hi] = s1 / (b * b)
        cnorm[lo:hi] = s2 - s1 * s1 / (b * b)
    return tiles, means, cnorm


def base_operands(tiles: np.ndarray, means: np.ndarray, svals, baseline: bool, chunk: int = 1 << 17):
    """qbase[e*S + si, :] = rint(s*(tile - mean)) (proposed) or rint(s*tile)
    (baseline) as int16, before any isometry (matcher.py:143-154)."""
    E, B, _ = tiles.shape
    sv = np.asarray(svals, dtype=np.float64)
    S = sv.shape[0]
    out = np.empty((E, S, B * B), dtype=np.int16)
    for lo in range(0, E, chunk):
        hi = min(E, lo + chunk)
        t = tiles[lo:hi].reshape(hi - lo, B * B).astype(np.float64)
        if not baseline:
            t = t - means[lo:hi, None]
        out[lo:hi] = np.rint(sv[None, :, None] * t[:, None, :]).astype(np.int16)
    return out.reshape(E * S, B * B)


def scan_candidates_base(ranges, rmeans, qbase, dmeans, svals, baseline, threads: int = 0):
    """scan_candidates (_scan.py:14-63) over the base operand with the
    isometries applied on the fly (scan_oracle.c) -> (err int64[M], idx int64[M])."""
    ranges = np.ascontiguousarray(ranges, dtype=np.int16)
    rmeans = np.ascontiguousarray(rmeans, dtype=np.float64)
    qbase = np.ascontiguousarray(qbase, dtype=np.int16)
    dmeans = np.ascontiguousarray(dmeans, dtype=np.float64)
    svals = np.ascontiguousarray(svals, dtype=np.float64)
    M, n = ranges.shape
    side = int(round(n ** 0.5))
    isomap = np.ascontiguousarray(
        np.stack([isometry_index_map(side, k) for k in range(8)]).astype(np.int32))
    out_err = np.empty(M, dtype=np.int64)
    out_idx = np.empty(M, dtype=np.int64)
    if M == 0:
        return out_err, out_idx
    _scan_lib().oracle_scan_candidates_base(
        M, n, ranges.ctypes.data, rmeans.ctypes.data, qbase.ctypes.data, dmeans.shape[0],
        dmeans.ctypes.data, svals.shape[0], svals.ctypes.data, int(bool(baseline)),
        isomap.ctypes.data, out_err.ctypes.data, out_idx.ctypes.data, int(threads),
    )
    return out_err, out_idx


_LIB = None


def _scan_lib():
    global _LIB
    if _LIB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "_build", "liboracle_scan.so")
        if not os.path.exists(path):
            from . import build as _b

            _b.build()
        lib = ctypes.CDLL(path)
        lib.oracle_scan_candidates_base.restype = None
        lib.oracle_scan_candidates_base.argtypes = [
            ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int32,
        ]
        lib.oracle_scan_candidates.restype = None
        lib.oracle_scan_candidates.argtypes = [
            ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int32,
        ]
        _LIB = lib
    return _LIB


def scan_candidates(ranges, rmeans, q, dmeans, svals, baseline, threads: int = 0):
    """Exhaustive first-strict-minimum scan (_scan.py:14-63), run in C.

    Returns (err int64[M], idx int64[M]).
    """
    ranges = np.ascontiguousarray(ranges, dtype=np.int16)
    rmeans = np.ascontiguousarray(rmeans, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.int16)
    dmeans = np.ascontiguousarray(dmeans, dtype=np.float64)
    svals = np.ascontiguousarray(svals, dtype=np.float64)
    M, n = ranges.shape
    out_err = np.empty(M, dtype=np.int64)
    out_idx = np.empty(M, dtype=np.int64)
    if M == 0:
        return out_err, out_idx
    _scan_lib().oracle_scan_candidates(
        M, n, ranges.ctypes.data, rmeans.ctypes.data, q.ctypes.data, dmeans.shape[0],
        dmeans.ctypes.data, svals.shape[0], svals.ctypes.data, int(bool(baseline)),
        out_err.ctypes.data, out_idx.ctypes.data, int(threads),
    )
    return out_err, out_idx


def scan_candidates_numpy(ranges, rmeans, q, dmeans, svals, baseline):
    """Vectorised numpy twin of the scan for small cases (_scan.py:29-63)."""
    ranges = np.asarray(ranges, dtype=np.int64)
    q = np.asarray(q, dtype=np.int64)
    svals = np.asarray(svals, dtype=np.float64)
    E, S = len(dmeans), len(svals)
    errs, idxs = [], []
    for m in range(ranges.shape[0]):
        if baseline:
            o = np.rint(rmeans[m] - svals[None, :] * np.asarray(dmeans)[:, None])  # [E,S]
            o = np.clip(o, 0, 255).astype(np.int64)
            o = np.broadcast_to(o[:, None, :], (E, 8, S)).reshape(-1)
        else:
            o = np.full(E * 8 * S, int(np.rint(rmeans[m])), dtype=np.int64)
        rec = np.clip(q + o[:, None], 0, 255)
        err = ((rec - ranges[m][None, :]) ** 2).sum(axis=1)
        c = int(np.argmin(err))  # first minimum == first strict minimum in order
        errs.append(int(err[c]))
        idxs.append(c)
    return np.array(errs, dtype=np.int64), np.array(idxs, dtype=np.int64)


def decode_index(idx: int, S: int):
    """flat index -> (domain, isometry, s index) (matcher.py:178-188)."""
    e, rem = divmod(int(idx), 8 * S)
    iso, si = divmod(rem, S)
    return e, iso, si


def stored_offset(rmean: float, svals, dmeans, e: int, si: int, baseline: bool) -> int:
    """The 8-bit O field (matcher.py:183-187)."""
    if baseline:
        return min(255, max(0, int(np.rint(rmean - svals[si] * dmeans[e]))))
    return int(np.rint(rmean))


def naive_best_match(range_tile, tiles, means, s_set, mode):
    """Plain-loop single-range match (the reference test oracle's semantics,
    tests/oracles.py:43-69).  Returns (error, domain, isometry, s_index, offset)."""
    r = np.asarray(range_tile, dtype=np.int64)
    n = r.size
    rmean = int(r.sum()) / n
    best = None
    for e in range(len(tiles)):
        for iso in range(8):
            d = apply_isometry(tiles[e], iso).astype(np.float64)
            for si, s in enumerate(s_set):
                if mode == "baseline":
                    o = min(255, max(0, int(np.rint(rmean - s * means[e]))))
                    rec = np.rint(s * d) + o
                else:
                    o = int(np.rint(rmean))
                    rec = np.rint(s * (d - means[e])) + o
                rec = np.clip(rec, 0, 255).astype(np.int64)
                err = int(((rec - r.reshape(d.shape)) ** 2).sum())
                if best is None or err < best[0]:
                    best = (err, e, iso, si, o)
    return best


# ---------------------------------------------------------------------------
# quadtree driver and encoder (codec.py)
# ---------------------------------------------------------------------------

def run_quadtree(width: int, height: int, thresholds, match_level):
    """Level loop, split rule and depth-first leaves (codec.py:114-161)."""
    tops = [(x, y) for y in range(0, height, TOP_SIDE) for x in range(0, width, TOP_SIDE)]
    by_level = {1: tops}
    split = {}
    index = {}
    for level in (1, 2, 3, 4):
        origins = by_level.get(level)
        if not origins:
            continue
        errs = match_level(level, origins)
        side = LEVEL_RANGE_SIDES[level - 1]
        limit = thresholds[level - 1] ** 2 * side * side if level < 4 else None
        kids = []
        for j, (x, y) in enumerate(origins):
            index[(level, x, y)] = j
            if level == 4 or errs[j] <= limit:
                split[(level, x, y)] = False
            else:
                split[(level, x, y)] = True
                h = side // 2
                kids += [(x, y), (x + h, y), (x, y + h), (x + h, y + h)]
        if kids:
            by_level[level + 1] = kids
    leaves = []

    def walk(level, x, y):
        if split[(level, x, y)]:
            h = LEVEL_RANGE_SIDES[level - 1] // 2
            for dx, dy in ((0, 0), (h, 0), (0, h), (h, h)):
                walk(level + 1, x + dx, y + dy)
        else:
            leaves.append((level, x, y, index[(level, x, y)]))

    for x, y in tops:
        walk(1, x, y)
    return leaves


def gather_tiles(pixels: np.ndarray, origins, side: int) -> np.ndarray:
    """Range tiles at origins, row-major within the tile (codec.py:164-168)."""
    win = np.lib.stride_tricks.sliding_window_view(pixels, (side, side))
    xs = np.array([o[0] for o in origins], dtype=np.int64)
    ys = np.array([o[1] for o in origins], dtype=np.int64)
    return win[ys, xs].reshape(len(origins), side * side)


@dataclass
class OracleEncoding:
    width: int
    height: int
    mode: str
    strides: tuple
    s_sets: tuple
    pools: tuple  # per level tuple of (x, y)
    records: list  # (step, offset, iso, addr, s_index)
    errors: list  # per record SSD
    scans: dict  # level -> (errs, idxs, rmeans, origins)

    @property
    def collage_ssd(self) -> int:
        return int(sum(self.errors))


def encode(pixels: np.ndarray, caps, strides=DEFAULT_STRIDES, mode="proposed",
           thresholds=(8.0, 8.0, 8.0), s_sets=None, threads: int = 0) -> OracleEncoding:
    """Whole encoder: pool, quadtree, records (codec.py:171-254)."""
    pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
    h, w = pixels.shape
    if w % 16 or h % 16:
        raise ValueError(f"dimensions not multiple of 16: {w}x{h}")
    baseline = mode == "baseline"
    if s_sets is None:
        s_sets = (DEFAULT_BASELINE_SET,) * 4 if baseline else DEFAULT_PROPOSED_SETS
    pools = [build_pool_level(pixels, lv, strides[lv - 1], caps[lv - 1]) for lv in (1, 2, 3, 4)]
    operands = {}
    scans = {}

    def match_level(level, origins):
        pl = pools[level - 1]
        if len(pl.xs) == 0:
            raise ValueError(f"no domain entries at level {level}")
        if level not in operands:
            operands[level] = candidate_operands(pl.tiles, pl.means, s_sets[level - 1], baseline)
        side = LEVEL_RANGE_SIDES[level - 1]
        tiles = gather_tiles(pixels, origins, side).astype(np.int16)
        rmeans = tiles.astype(np.int64).sum(axis=1) / (side * side)
        errs, idxs = scan_candidates(tiles, rmeans, operands[level], pl.means,
                                     s_sets[level - 1], baseline, threads)
        scans[level] = (errs, idxs, rmeans, list(origins))
        return errs

    leaves = run_quadtree(w, h, thresholds, match_level)
    records, errors = [], []
    for level, _x, _y, j in leaves:
        errs, idxs, rmeans, _ = scans[level]
        S = len(s_sets[level - 1])
        e, iso, si = decode_index(idxs[j], S)
        o = stored_offset(rmeans[j], s_sets[level - 1], pools[level - 1].means, e, si, baseline)
        records.append((level, o, iso, e, si))
        errors.append(int(errs[j]))
    return OracleEncoding(
        width=w, height=h, mode=mode, strides=tuple(strides),
        s_sets=tuple(tuple(float(v) for v in s) for s in s_sets),
        pools=tuple(tuple(zip(pl.xs.tolist(), pl.ys.tolist())) for pl in pools),
        records=records, errors=errors, scans=scans,
    )


# ---------------------------------------------------------------------------
# wire format (stream.py:175-207) and decoder (codec.py:269-358)
# ---------------------------------------------------------------------------

def _bits(count: int) -> int:
    return (count - 1).bit_length()  # stream.py:82-86


def serialize(enc: OracleEncoding) -> bytes:
    """FRAK v1 bytes (stream.py:3-22, 175-207)."""
    head = bytearray(b"FRAK")
    head += struct.pack("<BB", 1, 0 if enc.mode == "baseline" else 1)
    head += struct.pack("<II", enc.width, enc.height)
    head += struct.pack("<4H", *enc.strides)
    for s in enc.s_sets:
        head += struct.pack("<B", len(s)) + struct.pack(f"<{len(s)}d", *s)
    for coords in enc.pools:
        head += struct.pack("<I", len(coords))
        head += np.asarray(coords, dtype="<u2").reshape(-1).tobytes()
    head += struct.pack("<I", len(enc.records))
    acc, nbits = 0, 0
    for step, off, iso, addr, si in enc.records:
        for val, width in ((step - 1, 2), (off, 8), (iso, 3),
                           (addr, _bits(len(enc.pools[step - 1]))),
                           (si, _bits(len(enc.s_sets[step - 1])))):
            acc = (acc << width) | val
            nbits += width
    pad = (-nbits) % 8
    payload = (acc << pad).to_bytes((nbits + pad) // 8, "big") if nbits else b""
    head += struct.pack("<Q", nbits)
    return bytes(head) + payload


def iter_leaves(width, height, records):
    """(record, x, y, side) in depth-first order (stream.py:322-356)."""
    out = []
    pos = 0

    def walk(level, x, y, side):
        nonlocal pos
        step = records[pos][0]
        if step == level:
            out.append((records[pos], x, y, side))
            pos += 1
            return
        h = side // 2
        for dx, dy in ((0, 0), (h, 0), (0, h), (h, h)):
            walk(level + 1, x + dx, y + dy, h)

    for ty in range(0, height, 16):
        for tx in range(0, width, 16):
            walk(1, tx, ty, 16)
    return out


def collage_pass(cur: np.ndarray, enc: OracleEncoding, leaves) -> np.ndarray:
    """One application of the collage map (codec.py:319-336), loop form."""
    out = np.empty_like(cur)
    proposed = enc.mode != "baseline"
    for (step, off, iso, addr, si), x, y, side in leaves:
        dx, dy = enc.pools[step - 1][addr]
        dom = cur[dy : dy + 2 * side, dx : dx + 2 * side]
        d = apply_isometry(decimate(dom), iso).astype(np.float64)
        s = enc.s_sets[step - 1][si]
        if proposed:
            mean = int(d.astype(np.int64).sum()) / d.size
            q = np.rint(s * (d - mean))
        else:
            q = np.rint(s * d)
        out[y : y + side, x : x + side] = np.clip(q.astype(np.int32) + off, 0, 255)
    return out


def decode(enc: OracleEncoding, iterations: int = 15, tolerance: int = 0):
    """Iterate from a constant-128 image (codec.py:339-363)."""
    leaves = iter_leaves(enc.width, enc.height, enc.records)
    cur = np.full((enc.height, enc.width), 128, dtype=np.uint8)
    deltas = []
    for _ in range(iterations):
        new = collage_pass(cur, enc, leaves)
        delta = int(np.abs(new.astype(np.int16) - cur.astype(np.int16)).max())
        cur = new
        deltas.append(delta)
        if delta <= tolerance:
            break
    return cur, deltas


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """PSNR against an 8-bit peak (metrics.py:24-40)."""
    diff = a.astype(np.int64) - b.astype(np.int64)
    err = float((diff * diff).sum()) / diff.size
    return math.inf if err == 0.0 else 10.0 * math.log10(255.0 * 255.0 / err)


# ---------------------------------------------------------------------------
# real-valued slope analysis (bench.py:104-193)
# ---------------------------------------------------------------------------

S_BIN_EDGES = np.round(np.arange(-0.5, 1.5 + 0.05 / 2, 0.05), 10)  # bench.py:31-32


def level_basis(pool: OraclePoolLevel):
    """Centered isometry variants [E*8, n] (row e*8 + iso) and their norms
    (bench.py:104-114)."""
    centered = pool.tiles.astype(np.float64) - pool.means[:, None, None]
    side = centered.shape[-1]
    rows = np.stack([apply_isometry(centered, iso) for iso in range(8)], axis=1)
    return rows.reshape(-1, side * side), np.repeat(pool.cnorm.astype(np.float64), 8)


def real_s_matches(tiles: np.ndarray, basis: np.ndarray, norms: np.ndarray, chunk: int = 4096):
    """Per range tile: minimal projection error, slope and flat index of the
    first minimum (bench.py:117-139; the reference returns the first two)."""
    m, n = tiles.shape
    t = tiles.astype(np.float64)
    rc = t - (tiles.astype(np.int64).sum(axis=1) / n)[:, None]
    rnorm = (rc * rc).sum(axis=1)
    flat = norms == 0.0
    safe = np.where(flat, 1.0, norms)
    err = np.empty(m)
    slope = np.empty(m)
    pick_all = np.empty(m, dtype=np.int64)
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        cross = basis @ rc[lo:hi].T
        gain = np.where(flat[:, None], 0.0, cross * cross / safe[:, None])
        errs = np.maximum(rnorm[lo:hi][None, :] - gain, 0.0)
        pick = errs.argmin(axis=0)
        cols = np.arange(hi - lo)
        err[lo:hi] = errs[pick, cols]
        slope[lo:hi] = np.where(flat[pick], 0.0, cross[pick, cols] / safe[pick])
        pick_all[lo:hi] = pick
    return err, slope, pick_all


def s_histogram(pixels: np.ndarray, caps, strides=DEFAULT_STRIDES, thresholds=(8.0, 8.0, 8.0)):
    """bench.py:142-193 -> (raw_counts, clamped_counts, coded_blocks, raw_means, clamped_means)."""
    pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
    h, w = pixels.shape
    pools = [build_pool_level(pixels, lv, strides[lv - 1], caps[lv - 1]) for lv in (1, 2, 3, 4)]
    bases = {}
    s_by_level = {}

    def match_level(level, origins):
        if level not in bases:
            bases[level] = level_basis(pools[level - 1])
        tiles = gather_tiles(pixels, origins, LEVEL_RANGE_SIDES[level - 1])
        errs, slopes, _ = real_s_matches(tiles, *bases[level])
        s_by_level[level] = slopes
        return errs

    leaves = run_quadtree(w, h, thresholds, match_level)
    coded = {1: [], 2: [], 3: [], 4: []}
    for level, _x, _y, j in leaves:
        coded[level].append(float(s_by_level[level][j]))
    raw = np.zeros((4, len(S_BIN_EDGES) - 1), dtype=np.int64)
    clamped = np.zeros_like(raw)
    raw_means, clamped_means = [], []
    for level in (1, 2, 3, 4):
        v = np.array(coded[level])
        if v.size:
            raw[level - 1] = np.histogram(np.clip(v, S_BIN_EDGES[0], S_BIN_EDGES[-1]), bins=S_BIN_EDGES)[0]
            clamped[level - 1] = np.histogram(np.clip(v, 0.0, 1.0), bins=S_BIN_EDGES)[0]
            raw_means.append(float(v.mean()))
            clamped_means.append(float(np.clip(v, 0.0, 1.0).mean()))
        else:
            raw_means.append(None)
            clamped_means.append(None)
    return raw, clamped, tuple(len(coded[lv]) for lv in (1, 2, 3, 4)), raw_means, clamped_means
