"""Entropy-ranked, truncated domain pools built on the device.

Same interface and results as the reference's pool.py (PoolParams,
DomainEntry, DomainPool, build_pool, block_entropy, candidate_count).  The
ranking, decimation and moments run in CUDA (csrc/fc_pool.cu) and stay
resident on the device for the matcher; entries are copied back only when a
caller inspects them.  Extension: ``PoolParams.entropy_thresholds`` keeps
every window whose entropy exceeds tau_l (threshold compaction); it equals the
reference with ``level_caps[l] = #{entropy > tau_l}``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import PoolConfigError  # noqa: F401  (re-export)
from .image import GrayImage

LEVEL_RANGE_SIDES = (16, 8, 4, 2)
LEVEL_DOMAIN_SIDES = (32, 16, 8, 4)
LEVEL_COUNT = 4
DEFAULT_STRIDES = (8, 4, 2, 2)


@dataclass(frozen=True)
class PoolParams:
    pool_cap: int
    strides: tuple = DEFAULT_STRIDES
    level_caps: tuple | None = None
    entropy_thresholds: tuple | None = None  # per level float or None

    def __post_init__(self):
        if self.pool_cap < 1:
            raise ValueError("pool_cap must be >= 1")
        if len(self.strides) != LEVEL_COUNT or any(s < 1 for s in self.strides):
            raise ValueError("strides must be 4 positive integers")
        if self.level_caps is not None:
            if len(self.level_caps) != LEVEL_COUNT or any(c < 1 for c in self.level_caps):
                raise ValueError("level_caps must be 4 positive integers")
            object.__setattr__(self, "level_caps", tuple(int(c) for c in self.level_caps))
        if self.entropy_thresholds is not None:
            if len(self.entropy_thresholds) != LEVEL_COUNT:
                raise ValueError("entropy_thresholds needs one entry (or None) per level")
            object.__setattr__(self, "entropy_thresholds", tuple(
                None if t is None else float(t) for t in self.entropy_thresholds))
        object.__setattr__(self, "strides", tuple(int(s) for s in self.strides))

    def cap(self, level: int) -> int:
        if self.level_caps is not None:
            return self.level_caps[level - 1]
        return self.pool_cap

    def tau(self, level: int):
        if self.entropy_thresholds is None:
            return None
        return self.entropy_thresholds[level - 1]

    def native_args(self) -> tuple:
        """(strides, caps, taus, use_tau) as the C ABI's arrays, built once."""
        args = self.__dict__.get("_native")
        if args is None:
            taus = [self.tau(level) for level in (1, 2, 3, 4)]
            args = (np.asarray(self.strides, dtype=np.int32),
                    np.asarray([self.cap(level) for level in (1, 2, 3, 4)], dtype=np.int64),
                    np.asarray([0.0 if t is None else t for t in taus], dtype=np.float64),
                    np.asarray([0 if t is None else 1 for t in taus], dtype=np.int32))
            for a in args:
                a.flags.writeable = False
            object.__setattr__(self, "_native", args)
        return args


@dataclass(frozen=True, eq=False)
class DomainEntry:
    x: int
    y: int
    entropy: float
    tile: np.ndarray
    mean: float
    centered_norm_sq: float


class CoordTable:
    """Read-only sequence of (x, y) pool origins backed by an [E, 2] array.

    Compares equal to another table or to a tuple of (x, y) tuples, so stream
    objects compare like the reference's tuple-of-tuples headers without
    materialising millions of Python tuples.
    """

    __slots__ = ("array", "__weakref__")

    def __init__(self, array):
        a = np.asarray(array.array if isinstance(array, CoordTable) else array)
        if a.dtype != np.uint16:  # device tables arrive as u16 pairs (the stream format)
            a = a.astype(np.int64)
        a = a.reshape(-1, 2)
        a.flags.writeable = False
        self.array = a

    def _detach(self):
        """Own a private copy (the table was a view of context memory)."""
        a = self.array.copy()
        a.flags.writeable = False
        self.array = a

    def __len__(self):
        return self.array.shape[0]

    def __array__(self, dtype=None, copy=None):
        # np.asarray(table) takes the backing array (a Python walk of the
        # sequence protocol would build millions of tuples)
        a = self.array if dtype is None else self.array.astype(dtype)
        return a.copy() if copy else a

    def __getitem__(self, i):
        if isinstance(i, slice):
            return tuple((int(x), int(y)) for x, y in self.array[i])
        x, y = self.array[i]
        return (int(x), int(y))

    def __iter__(self):
        return ((int(x), int(y)) for x, y in self.array)

    def __eq__(self, other):
        if isinstance(other, CoordTable):
            return np.array_equal(self.array, other.array)
        try:
            o = np.asarray(other, dtype=np.int64).reshape(-1, 2)
        except (TypeError, ValueError):
            return NotImplemented
        return np.array_equal(self.array, o)

    def __hash__(self):
        return hash(self.array.astype(np.int64).tobytes())

    def __repr__(self):
        return f"CoordTable({len(self)} origins)"


class DomainPool:
    """Device-resident per-level pools (entropy-descending, raster tie order)."""

    def __init__(self, params: PoolParams, width: int, height: int, sizes, context):
        self.params = params
        self.width = width
        self.height = height
        self.sizes = tuple(int(s) for s in sizes)
        self.context = context
        # device data is fetched lazily: it must still be this pool's
        self._generation = context.pool_generation
        self._coords = {}
        self._entries = {}
        self._means = {}
        self._tables = None

    def _check_current(self):
        if self.context.pool_generation != self._generation:
            raise RuntimeError("this pool was superseded by a later pool build on its context")

    def size(self, level: int) -> int:
        return self.sizes[level - 1]

    def coords_array(self, level: int) -> np.ndarray:
        if level not in self._coords:
            self._check_current()
            self._coords[level] = self.context.pool_coords(level, self.size(level))
        return self._coords[level]

    def coords(self, level: int) -> CoordTable:
        return CoordTable(self.coords_array(level))

    def all_coords(self) -> tuple:
        """CoordTable of every level without a host copy when the context can
        lend its pinned buffer (copied on the next pool build), else one call."""
        if self._tables is None and len(self._coords) < 4:
            self._check_current()
            self._tables = self.context.pool_coord_tables(self.sizes, CoordTable)
        if self._tables is not None:
            return self._tables
        if len(self._coords) < 4:
            for level, arr in zip((1, 2, 3, 4), self.context.pool_coords_all(self.sizes)):
                self._coords.setdefault(level, arr)
        return tuple(CoordTable(self._coords[level]) for level in (1, 2, 3, 4))

    def means(self, level: int) -> np.ndarray:
        if level not in self._means:
            self._check_current()
            _, _, m, _ = self.context.pool_entries(level, self.size(level),
                                                   LEVEL_RANGE_SIDES[level - 1], want=("means",))
            self._means[level] = m
        return self._means[level]

    def entries(self, level: int) -> tuple:
        if level not in self._entries:
            self._check_current()
            side = LEVEL_RANGE_SIDES[level - 1]
            ent, tiles, means, cnorm = self.context.pool_entries(level, self.size(level), side)
            xy = self.coords_array(level)
            self._entries[level] = tuple(
                DomainEntry(int(xy[i, 0]), int(xy[i, 1]), float(ent[i]), tiles[i], float(means[i]),
                            float(cnorm[i])) for i in range(self.size(level)))
        return self._entries[level]

    @property
    def levels(self):
        return tuple(self.entries(lv) for lv in (1, 2, 3, 4))

    @classmethod
    def from_tiles(cls, tiles_by_level: dict, device: int = 0, width: int = 512, height: int = 512):
        """Synthetic pool from decimated tiles per level (the reference tests'
        make_test_pool, tests/oracles.py:29-40)."""
        ctx = _native.Context(device)
        sizes = []
        for level in (1, 2, 3, 4):
            side = LEVEL_RANGE_SIDES[level - 1]
            tiles = np.asarray(tiles_by_level.get(level, []), dtype=np.uint8).reshape(-1, side, side)
            ctx.pool_set_level(level, tiles)
            sizes.append(tiles.shape[0])
        cap = max(1, max(sizes))
        return cls(PoolParams(pool_cap=cap), width, height, sizes, ctx)


def build_pool(image: GrayImage, params: PoolParams, context=None, device_image=None) -> DomainPool:
    """Rank every lattice domain by entropy and keep the top cap per level (device).

    ``device_image`` (optional): an object exposing ``data_ptr()`` (e.g. a CUDA
    uint8 tensor) holding the same pixels already resident in HBM; the
    context then adopts it instead of copying ``image`` from the host.
    """
    ctx = context if context is not None else _native.Context()
    if device_image is not None:
        _adopt_device_image(ctx, device_image, image)
    else:
        ctx.set_image(image.pixels)
    sizes = ctx.pool_build(*params.native_args())
    return DomainPool(params, image.width, image.height, sizes, ctx)


class _DeviceArray:
    """A raw device buffer of the context seen by torch (CUDA array interface)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def build_pool_sharded(image: GrayImage, params: PoolParams, context=None, device_image=None,
                       collective_device=None, force: bool = False) -> DomainPool:
    """build_pool with the entropy pass sharded over the torch.distributed
    ranks ("all-gather the entropy keys, then a replicated
    sort").  Each rank computes the windows of its slice of window rows per
    level (fc_pool_entropy), the slices are all-gathered into every rank's
    window buffers -- entropies and, without a threshold, the keys; with one,
    the survivors' (key, index) pairs, whose order the ranking restores -- and
    every rank then ranks the same complete set (fc_pool_rank): the pool is
    identical to build_pool's on every rank.  Falls back to build_pool when
    not distributed, or on a single rank unless ``force`` (tests: the
    exchange path over a one-rank NCCL group)."""
    import torch
    import torch.distributed as dist

    from . import sharding

    if not (dist.is_available() and dist.is_initialized()) or (dist.get_world_size() == 1 and not force):
        return build_pool(image, params, context, device_image)
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = context if context is not None else _native.Context()
    if device_image is not None:
        _adopt_device_image(ctx, device_image, image)
    else:
        ctx.set_image(image.pixels)
    coll = collective_device or f"cuda:{ctx.device}"
    strides, caps, taus, use_tau = params.native_args()
    # equal blocks of window rows per rank (the last ones may be short), so
    # every rank knows every slice and the exchange needs no size round
    rpr, lo, hi = [], [], []
    for level, stride in zip((1, 2, 3, 4), strides):
        side = 2 * LEVEL_RANGE_SIDES[level - 1]
        ny = max((image.height - side) // stride + 1 if image.height >= side else 0, 0)
        r = -(-ny // world)
        rpr.append(r)
        lo.append(min(rank * r, ny))
        hi.append(min(rank * r + r, ny))
    ctx.pool_entropy(strides, caps, taus, use_tau, lo, hi)
    dev = torch.device("cuda", ctx.device)
    ext = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    sel = [0, 0, 0, 0]
    with torch.cuda.device(dev):
        cur = torch.cuda.current_stream(dev)
        cur.wait_stream(ext)  # the entropy pass before the collectives read its buffers
        bufs = []
        for li in range(4):
            b = ctx.pool_window_buffers(li + 1, local_sel=bool(use_tau[li]))
            nwin = b["nx"] * b["ny"]
            bufs.append(None if nwin == 0 else dict(
                nx=b["nx"], nwin=nwin, sel=b["sel"],
                ent=torch.as_tensor(_DeviceArray(b["ent"], nwin, "<i8"), device=dev),  # f64 bits
                key=torch.as_tensor(_DeviceArray(b["key"], nwin, "<i8"), device=dev),
                val=torch.as_tensor(_DeviceArray(b["val"], nwin, "<i4"), device=dev)))
        # 1. one all-gather of every level's row slice of entropies (and keys
        #    without a threshold), each padded to the block size: rank r's
        #    block of a level lands at r * block, i.e. the full raster array
        parts, off = [], 0
        for li, b in enumerate(bufs):
            if b is None:
                continue
            blk = rpr[li] * b["nx"]
            w0, w1 = lo[li] * b["nx"], hi[li] * b["nx"]
            for name in ("ent",) if use_tau[li] else ("ent", "key"):
                parts.append((li, name, off, blk, b[name][w0:w1]))
                off += blk
        mine = torch.zeros(off, dtype=torch.int64, device=coll)
        for _, _, o, _, src in parts:
            mine[o:o + src.numel()].copy_(src)
        out = torch.empty(world * off, dtype=torch.int64, device=coll)
        dist.all_gather(list(out.chunk(world)), mine)
        out = out.view(world, off)
        for li, name, o, blk, _ in parts:
            b = bufs[li]
            b[name].copy_(out[:, o:o + blk].reshape(-1)[:b["nwin"]].to(dev))
            if name == "key":
                b["val"].copy_(torch.arange(b["nwin"], dtype=torch.int32, device=dev))
        # 2. threshold levels: the survivors' (key, window) lists, variable
        #    length: one count exchange, one padded all-gather
        tau_lv = [li for li, b in enumerate(bufs) if b is not None and use_tau[li]]
        if tau_lv:
            cnt = torch.tensor([bufs[li]["sel"] for li in tau_lv], dtype=torch.int64, device=coll)
            cnts = torch.empty(world * len(tau_lv), dtype=torch.int64, device=coll)
            dist.all_gather(list(cnts.chunk(world)), cnt)
            cnts = cnts.view(world, len(tau_lv)).tolist()
            cap = [max(max(row[k] for row in cnts), 1) for k in range(len(tau_lv))]
            width = 2 * sum(cap)
            mine = torch.zeros(width, dtype=torch.int64, device=coll)
            o = 0
            for k, li in enumerate(tau_lv):
                n = bufs[li]["sel"]
                mine[o:o + n].copy_(bufs[li]["key"][:n])
                mine[o + cap[k]:o + cap[k] + n].copy_(bufs[li]["val"][:n])
                o += 2 * cap[k]
            out = torch.empty(world * width, dtype=torch.int64, device=coll)
            dist.all_gather(list(out.chunk(world)), mine)
            out = out.view(world, width)
            o = 0
            for k, li in enumerate(tau_lv):
                keys = torch.cat([out[r, o:o + cnts[r][k]] for r in range(world)])
                vals = torch.cat([out[r, o + cap[k]:o + cap[k] + cnts[r][k]] for r in range(world)])
                sel[li] = int(keys.numel())
                bufs[li]["key"][:sel[li]].copy_(keys.to(dev))
                bufs[li]["val"][:sel[li]].copy_(vals.to(dev, torch.int32))
                o += 2 * cap[k]
        ext.wait_stream(cur)  # the completed buffers before the ranking
    sizes = ctx.pool_rank(sel)
    return DomainPool(params, image.width, image.height, sizes, ctx)


def _adopt_device_image(ctx, dev, image: GrayImage):
    """Let the context read an HBM-resident copy of ``image`` in place.

    The tensor must be a contiguous uint8 (height, width) CUDA tensor on the
    context's device; the context stream waits for the producer's current
    stream, so a copy still in flight is never read early.  No record_stream:
    every encode is synchronous at return, and an allocator event recorded on
    the context's stream would outlive that stream (fc_ctx_destroy)."""
    import torch

    if not isinstance(dev, torch.Tensor):
        raise TypeError("device_image must be a torch CUDA tensor")
    if dev.dtype != torch.uint8 or not dev.is_cuda or dev.device.index != ctx.device:
        raise ValueError(f"device_image must be a uint8 tensor on cuda:{ctx.device}")
    if tuple(dev.shape) != (image.height, image.width) or not dev.is_contiguous():
        raise ValueError(f"device_image must be contiguous with shape {(image.height, image.width)}")
    ext = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev.device)
    ext.wait_stream(torch.cuda.current_stream(dev.device))
    ctx.set_image_device(int(dev.data_ptr()), image.width, image.height)


def block_entropy(tile) -> float:
    """Entropy in nats of a tile's 256-bin histogram (pool.py:95-103), host
    helper: the same float64 terms as the device kernel (the run-time numpy
    LUT of p*log(p) for the tile size) summed in bin order by numpy."""
    a = np.asarray(tile)
    n = a.size
    if n == 0:
        raise ValueError("tile must be non-empty")
    flat = a.astype(np.int64).ravel()
    if flat.min() < 0 or flat.max() > 255:
        raise ValueError("pixel values must lie in [0, 255]")
    counts = np.bincount(flat, minlength=256)
    p = counts / n
    logs = np.log(np.where(counts > 0, p, 1.0))
    return float(-(p * logs).reshape(1, 256).sum(axis=1)[0])


def candidate_count(image_size, domain_side: int, stride: int) -> int:
    """Lattice windows of side ``domain_side`` at ``stride`` (pool.py:106-117):
    the level's candidate count before any truncation."""
    w, h = image_size if isinstance(image_size, (tuple, list)) else (image_size, image_size)
    per_axis = [(dim - domain_side) // stride + 1 if dim >= domain_side else 0 for dim in (w, h)]
    return per_axis[0] * per_axis[1]
