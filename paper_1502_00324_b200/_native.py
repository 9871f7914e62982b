"""ctypes binding of libfracodec_b200.so (include/fracodec_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is visible, every device entry point raises DeviceUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libfracodec_b200.so")

FC_OK = 0
FC_ERR_CUDA = 1
FC_ERR_ARG = 2
FC_ERR_POOL_CONFIG = 3
FC_ERR_EMPTY_POOL = 4
FC_ERR_TILE_SIZE = 5
FC_ERR_DIMS = 6
FC_ERR_NO_DEVICE = 7
FC_ERR_STATE = 8

PATH_AUTO, PATH_EXACT, PATH_TENSOR = 0, 1, 2


class DeviceUnavailableError(RuntimeError):
    """The CUDA library or an sm_100 device is not available (no CPU fallback)."""


class DeviceError(RuntimeError):
    """A CUDA runtime failure inside the native library."""


class FcStats(ctypes.Structure):
    _fields_ = [
        ("comparisons", ctypes.c_int64),
        ("ranges", ctypes.c_int64),
        ("columns", ctypes.c_int64),
        ("path", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("scan_ms", ctypes.c_float),
        ("main_ms", ctypes.c_float),
        ("fix_ms", ctypes.c_float),
        ("fix_pairs", ctypes.c_int64),
        ("rescans", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_SIGNATURES = {
    "fc_version": ([], ctypes.c_int),
    "fc_ctx_create": ([ctypes.c_int, ctypes.POINTER(_P)], ctypes.c_int),
    "fc_ctx_destroy": ([_P], None),
    "fc_last_error": ([_P], ctypes.c_char_p),
    "fc_synchronize": ([_P], ctypes.c_int),
    "fc_set_device_io": ([_P, ctypes.c_int], ctypes.c_int),
    "fc_set_option": ([_P, ctypes.c_char_p, _I64], ctypes.c_int),
    "fc_set_entropy_lut": ([_P, ctypes.c_int, _P], ctypes.c_int),
    "fc_set_image": ([_P, _P, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "fc_pool_build": ([_P, _P, _P, _P, _P, _P], ctypes.c_int),
    "fc_pool_entropy": ([_P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "fc_pool_window_buffers": ([_P, ctypes.c_int, ctypes.POINTER(_P), ctypes.POINTER(_P),
                                ctypes.POINTER(_P), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                ctypes.POINTER(_I64)], ctypes.c_int),
    "fc_pool_rank": ([_P, _P, _P], ctypes.c_int),
    "fc_pool_entropy_batch": ([_P, ctypes.c_int, _P, _P, _P, _P], ctypes.c_int),
    "fc_pool_set_level": ([_P, ctypes.c_int, _I64, _P], ctypes.c_int),
    "fc_pool_size": ([_P, ctypes.c_int, _P], ctypes.c_int),
    "fc_pool_coords": ([_P, ctypes.c_int, _P], ctypes.c_int),
    "fc_pool_coords_all": ([_P, _P], ctypes.c_int),
    "fc_pack_records": ([_P, ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P, _P, ctypes.c_int64,
                         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
                        ctypes.c_int),
    "fc_pool_coords_view": ([_P, ctypes.POINTER(_P)], ctypes.c_int),
    "fc_pool_entries": ([_P, ctypes.c_int, _P, _P, _P, _P], ctypes.c_int),
    "fc_level_prepare": ([_P, ctypes.c_int, ctypes.c_int, _P, _I32, _I32], ctypes.c_int),
    "fc_match_level": ([_P, ctypes.c_int, _P, _I64, _P, _P, _P], ctypes.c_int),
    "fc_match_tiles": ([_P, ctypes.c_int, _P, _I64, _P, _P, _P], ctypes.c_int),
    "fc_real_match_level": ([_P, ctypes.c_int, _P, _I64, _P, _P, _P], ctypes.c_int),
    "fc_scan_candidates": ([_P, _P, _P, _I64, _I32, _P, _P, _I64, _P, _I32, _I32, _P, _P],
                           ctypes.c_int),
    "fc_encode": ([_P, _P, _I32, _P, _P, _I32, _P, _I64, ctypes.POINTER(_I64)], ctypes.c_int),
    "fc_encode_records": ([_P, _P, _I64], ctypes.c_int),
    "fc_encode_level_stats": ([_P, ctypes.c_int, ctypes.POINTER(FcStats)], ctypes.c_int),
    "fc_encode_summary": ([_P, _P], ctypes.c_int),
    "fc_decode": ([_P, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _P, _P, ctypes.c_int32,
                   ctypes.c_int32, ctypes.c_int32, _P, _P, ctypes.POINTER(ctypes.c_int32)],
                  ctypes.c_int),
    "fc_last_stats": ([_P, ctypes.POINTER(FcStats)], ctypes.c_int),
    "fc_get_stream": ([_P, ctypes.POINTER(_P)], ctypes.c_int),
    "fc_launch_count": ([_P, ctypes.POINTER(_I64)], ctypes.c_int),
    "fc_probe_int8_peak": ([_P, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "fc_pool_times": ([_P, _P], ctypes.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load the shared library; raise loudly if it is absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailableError(
                f"{LIB_PATH} is missing: run `python -m paper_1502_00324_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def exported_symbols():
    return list(_SIGNATURES)


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def entropy_lut(n: int) -> np.ndarray:
    """terms[k-1] = (k/n) * log(k/n) evaluated by this host's numpy with the
    same array operations pool.py:90-91 applies, so the device reproduces the
    reference's float64 entropy bits exactly."""
    p = np.arange(1, n + 1, dtype=np.int64) / n
    return np.ascontiguousarray(p * np.log(p), dtype=np.float64)


class Context:
    """One fc_ctx: a CUDA stream plus device-resident image, pools and operands."""

    def __init__(self, device: int = 0):
        from .errors import raise_for_status  # local import (cycle-free)

        self._raise = raise_for_status
        self.lib = load_library()
        h = ctypes.c_void_p()
        rc = self.lib.fc_ctx_create(int(device), ctypes.byref(h))
        if rc == FC_ERR_NO_DEVICE:
            raise DeviceUnavailableError("no sm_100 CUDA device visible (no CPU fallback)")
        if rc != FC_OK:
            raise DeviceError(f"fc_ctx_create failed with status {rc}")
        self.handle = h
        self.device = device
        # CoordTables viewing the context's pinned coordinate buffer; they get
        # their own copy before anything can overwrite or free that buffer
        self._views = []  # weakref.ref (identity, not the tables' content hash)
        self.pool_generation = 0  # bumped whenever the device pool is replaced
        for n in (16, 64, 256, 1024):
            lut = entropy_lut(n)
            self.check(self.lib.fc_set_entropy_lut(self.handle, n, _ptr(lut)))

    def check(self, rc: int):
        if rc != FC_OK:
            msg = self.lib.fc_last_error(self.handle)
            self._raise(rc, msg.decode() if msg else "")

    def _detach_views(self):
        views = getattr(self, "_views", None)
        if not views:
            return
        for ref in views:
            t = ref()
            if t is not None:
                t._detach()
        views.clear()

    def close(self):
        self._detach_views()
        if getattr(self, "handle", None):
            self.lib.fc_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- thin wrappers -----------------------------------------------------
    def set_option(self, name: str, value: int):
        self.check(self.lib.fc_set_option(self.handle, name.encode(), int(value)))

    def set_image(self, pixels: np.ndarray):
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        self.check(self.lib.fc_set_image(self.handle, _ptr(a), a.shape[1], a.shape[0]))

    def set_image_device(self, dev_ptr: int, width: int, height: int):
        self.check(self.lib.fc_set_device_io(self.handle, 1))
        try:
            self.check(self.lib.fc_set_image(self.handle, dev_ptr, width, height))
        finally:
            self.check(self.lib.fc_set_device_io(self.handle, 0))

    def pool_build(self, strides, caps, taus, use_tau):
        s = np.ascontiguousarray(strides, dtype=np.int32)
        c = np.ascontiguousarray(caps, dtype=np.int64)
        t = np.ascontiguousarray(taus, dtype=np.float64)
        u = np.ascontiguousarray(use_tau, dtype=np.int32)
        out = np.zeros(4, dtype=np.int64)
        self._detach_views()  # the build rewrites (and may reallocate) the pinned coordinates
        self.pool_generation += 1
        self.check(self.lib.fc_pool_build(self.handle, _ptr(s), _ptr(c), _ptr(t), _ptr(u), _ptr(out)))
        return tuple(int(v) for v in out)

    def pool_entropy(self, strides, caps, taus, use_tau, row_lo=None, row_hi=None):
        """Phase 1 of pool_build over window rows [row_lo[l], row_hi[l]) per level."""
        s = np.ascontiguousarray(strides, dtype=np.int32)
        c = np.ascontiguousarray(caps, dtype=np.int64)
        t = np.ascontiguousarray(taus, dtype=np.float64)
        u = np.ascontiguousarray(use_tau, dtype=np.int32)
        lo = None if row_lo is None else np.ascontiguousarray(row_lo, dtype=np.int32)
        hi = None if row_hi is None else np.ascontiguousarray(row_hi, dtype=np.int32)
        self._detach_views()
        self.pool_generation += 1
        self.check(self.lib.fc_pool_entropy(self.handle, _ptr(s), _ptr(c), _ptr(t), _ptr(u),
                                            None if lo is None else _ptr(lo),
                                            None if hi is None else _ptr(hi)))

    def pool_window_buffers(self, level: int, local_sel: bool = False) -> dict:
        """Device pointers and grid of a level's window buffers after pool_entropy."""
        key, val, ent = _P(), _P(), _P()
        nx, ny, sel = _I64(), _I64(), _I64()
        self.check(self.lib.fc_pool_window_buffers(
            self.handle, level, ctypes.byref(key), ctypes.byref(val), ctypes.byref(ent),
            ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(sel) if local_sel else None))
        return {"key": key.value, "val": val.value, "ent": ent.value, "nx": nx.value, "ny": ny.value,
                "sel": sel.value if local_sel else None}

    @staticmethod
    def pool_entropy_batch(contexts, strides, caps, taus, use_tau):
        """Phase 1 of pool_build for several contexts (images of one size) in one
        pair of launches; each context then calls pool_rank()."""
        contexts = list(contexts)
        c0 = contexts[0]
        handles = (_P * len(contexts))(*[c.handle for c in contexts])
        s = np.ascontiguousarray(strides, dtype=np.int32)
        cp = np.ascontiguousarray(caps, dtype=np.int64)
        t = np.ascontiguousarray(taus, dtype=np.float64)
        u = np.ascontiguousarray(use_tau, dtype=np.int32)
        for c in contexts:
            c._detach_views()
            c.pool_generation += 1
        c0.check(c0.lib.fc_pool_entropy_batch(ctypes.cast(handles, _P), len(contexts), _ptr(s), _ptr(cp),
                                              _ptr(t), _ptr(u)))

    def pool_rank(self, sel_counts=None):
        """Phase 2 of pool_build -> per-level pool sizes."""
        out = np.zeros(4, dtype=np.int64)
        sc = None if sel_counts is None else np.ascontiguousarray(sel_counts, dtype=np.int64)
        self.check(self.lib.fc_pool_rank(self.handle, None if sc is None else _ptr(sc), _ptr(out)))
        return tuple(int(v) for v in out)

    def pool_set_level(self, level: int, tiles: np.ndarray):
        t = np.ascontiguousarray(tiles, dtype=np.uint8)
        self.pool_generation += 1
        self.check(self.lib.fc_pool_set_level(self.handle, level, t.shape[0] if t.size else 0,
                                              _ptr(t) if t.size else None))

    def pool_coords(self, level: int, count: int) -> np.ndarray:
        out = np.empty((count, 2), dtype=np.uint16)
        if count:
            self.check(self.lib.fc_pool_coords(self.handle, level, _ptr(out)))
        return out

    def pool_coords_all(self, sizes) -> tuple:
        """(x, y) uint16 origins of all four levels in one call -> per-level views."""
        total = int(sum(sizes))
        out = np.empty((total, 2), dtype=np.uint16)
        if total:
            self.check(self.lib.fc_pool_coords_all(self.handle, _ptr(out)))
        bounds = np.cumsum((0,) + tuple(int(s) for s in sizes))
        return tuple(out[bounds[k]:bounds[k + 1]] for k in range(len(sizes)))

    def pool_coord_tables(self, sizes, table_cls) -> tuple | None:
        """Per-level ``table_cls`` objects viewing the pinned coordinates of the
        last fc_pool_build without a copy (None when there is no such view);
        each is detached (copied) before the next pool build or close()."""
        p = _P()
        self.check(self.lib.fc_pool_coords_view(self.handle, ctypes.byref(p)))
        if not p.value:
            return None
        total = int(sum(sizes))
        if total == 0:
            return tuple(table_cls(np.zeros((0, 2), dtype=np.uint16)) for _ in sizes)
        buf = (ctypes.c_uint16 * (2 * total)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=np.uint16).reshape(total, 2)
        bounds = np.cumsum((0,) + tuple(int(s) for s in sizes))
        tables = tuple(table_cls(arr[bounds[k]:bounds[k + 1]]) for k in range(len(sizes)))
        self._views.extend(weakref.ref(t) for t in tables)
        return tables

    def pool_entries(self, level: int, count: int, side: int, want=("entropy", "tiles", "means", "cnorm")):
        ent = np.empty(count) if "entropy" in want else None
        tiles = np.empty((count, side, side), dtype=np.uint8) if "tiles" in want else None
        means = np.empty(count) if "means" in want else None
        cnorm = np.empty(count) if "cnorm" in want else None
        if count:
            self.check(self.lib.fc_pool_entries(self.handle, level, _ptr(ent), _ptr(tiles),
                                                _ptr(means), _ptr(cnorm)))
        return ent, tiles, means, cnorm

    def level_prepare(self, level: int, baseline: bool, svals, path: int = PATH_AUTO):
        s = np.ascontiguousarray(svals, dtype=np.float64)
        self.check(self.lib.fc_level_prepare(self.handle, level, int(bool(baseline)), _ptr(s),
                                             len(s), int(path)))

    def match_level(self, level: int, origins):
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.int32).reshape(-1, 2))
        M = o.shape[0]
        err = np.empty(M, dtype=np.int64)
        idx = np.empty(M, dtype=np.int64)
        rmean = np.empty(M, dtype=np.float64)
        self.check(self.lib.fc_match_level(self.handle, level, _ptr(o), M, _ptr(err), _ptr(idx),
                                           _ptr(rmean)))
        return err, idx, rmean

    def match_tiles(self, level: int, tiles: np.ndarray):
        t = np.ascontiguousarray(tiles, dtype=np.uint8)
        M = t.shape[0]
        err = np.empty(M, dtype=np.int64)
        idx = np.empty(M, dtype=np.int64)
        rmean = np.empty(M, dtype=np.float64)
        self.check(self.lib.fc_match_tiles(self.handle, level, _ptr(t), M, _ptr(err), _ptr(idx),
                                           _ptr(rmean)))
        return err, idx, rmean

    def real_match_level(self, level: int, origins):
        """fc_real_match_level: (errs f64, slopes f64, flat index e*8 + iso int64)."""
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.int32).reshape(-1, 2))
        M = o.shape[0]
        err = np.empty(M, dtype=np.float64)
        slope = np.empty(M, dtype=np.float64)
        idx = np.empty(M, dtype=np.int64)
        self.check(self.lib.fc_real_match_level(self.handle, level, _ptr(o), M, _ptr(err),
                                                _ptr(slope), _ptr(idx)))
        return err, slope, idx

    def match_level_device(self, level: int, origins_ptr: int, count: int, err_ptr: int,
                           idx_ptr: int, rmean_ptr: int):
        self.check(self.lib.fc_set_device_io(self.handle, 1))
        try:
            self.check(self.lib.fc_match_level(self.handle, level, ctypes.c_void_p(origins_ptr), count,
                                               ctypes.c_void_p(err_ptr), ctypes.c_void_p(idx_ptr),
                                               ctypes.c_void_p(rmean_ptr)))
        finally:
            self.check(self.lib.fc_set_device_io(self.handle, 0))

    def scan_candidates(self, ranges, rmeans, q, dmeans, svals, baseline):
        r = np.ascontiguousarray(ranges, dtype=np.int16)
        rm = np.ascontiguousarray(rmeans, dtype=np.float64)
        qq = np.ascontiguousarray(q, dtype=np.int16)
        dm = np.ascontiguousarray(dmeans, dtype=np.float64)
        sv = np.ascontiguousarray(svals, dtype=np.float64)
        M, n = r.shape
        err = np.empty(M, dtype=np.int64)
        idx = np.empty(M, dtype=np.int64)
        self.check(self.lib.fc_scan_candidates(self.handle, _ptr(r), _ptr(rm), M, n, _ptr(qq),
                                               _ptr(dm), len(dm), _ptr(sv), len(sv),
                                               int(bool(baseline)), _ptr(err), _ptr(idx)))
        return err, idx

    def encode(self, thresholds, baseline: bool, s_sets, path: int = PATH_AUTO,
               capacity: int | None = None) -> np.ndarray:
        """Device quadtree encode (fc_encode): int32 records [n, 6] =
        (step, offset, iso, addr, sidx, err) in depth-first order."""
        th = np.zeros(3, dtype=np.float64)
        th[:len(thresholds[:3])] = np.asarray(thresholds[:3], dtype=np.float64)
        counts = np.array([len(s) for s in s_sets], dtype=np.int32)
        sv = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.float64) for s in s_sets]))
        if capacity is None:
            capacity = 1 << 16
        out = np.empty((capacity, 6), dtype=np.int32)
        n = ctypes.c_int64()
        rc = self.lib.fc_encode(self.handle, _ptr(th), int(bool(baseline)), _ptr(sv), _ptr(counts),
                                int(path), _ptr(out), capacity, ctypes.byref(n))
        count = int(n.value)
        if rc == FC_ERR_ARG and count > capacity:  # undersized buffer: fetch again
            out = np.empty((count, 6), dtype=np.int32)
            self.check(self.lib.fc_encode_records(self.handle, _ptr(out), count))
            return out
        self.check(rc)
        return out[:count]

    def encode_level_stats(self, level: int) -> FcStats:
        st = FcStats()
        self.check(self.lib.fc_encode_level_stats(self.handle, level, ctypes.byref(st)))
        return st

    def decode(self, leaves: np.ndarray, width: int, height: int, s_sets, proposed: bool,
               iterations: int, tolerance: int):
        """Device collage iterations (fc_decode) -> (uint8 [height, width], deltas)."""
        lv = np.ascontiguousarray(leaves, dtype=np.int32).reshape(-1, 8)
        counts = np.array([len(s) for s in s_sets], dtype=np.int32)
        sv = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.float64) for s in s_sets]))
        out = np.empty((height, width), dtype=np.uint8)
        deltas = np.zeros(max(int(iterations), 1), dtype=np.int32)
        passes = ctypes.c_int32()
        self.check(self.lib.fc_decode(self.handle, _ptr(lv), lv.shape[0], int(width), int(height),
                                      _ptr(sv), _ptr(counts), int(bool(proposed)), int(iterations),
                                      int(tolerance), _ptr(out), _ptr(deltas), ctypes.byref(passes)))
        return out, [int(v) for v in deltas[:passes.value]]

    def set_top_slab(self, begin: int = 0, end: int = -1):
        """Restrict fc_encode to the raster slab [begin, end) of top-level slots."""
        self.set_option("top_begin", int(begin))
        self.set_option("top_end", int(end))

    def encode_summary(self) -> tuple:
        """(leaf counts per step 1..4, collage SSD) of the last encode."""
        out = np.zeros(5, dtype=np.int64)
        self.check(self.lib.fc_encode_summary(self.handle, _ptr(out)))
        return tuple(int(v) for v in out[:4]), int(out[4])

    def stats(self) -> FcStats:
        st = FcStats()
        self.check(self.lib.fc_last_stats(self.handle, ctypes.byref(st)))
        return st

    def synchronize(self):
        self.check(self.lib.fc_synchronize(self.handle))

    def stream_handle(self) -> int:
        """cudaStream_t of this context (for timing with events on its stream)."""
        h = ctypes.c_void_p()
        self.check(self.lib.fc_get_stream(self.handle, ctypes.byref(h)))
        return int(h.value or 0)

    def probe_int8_peak(self) -> float:
        """Dense tcgen05 kind::i8 rate (TOP/s) measured on this GPU by the library."""
        v = ctypes.c_double()
        self.check(self.lib.fc_probe_int8_peak(self.handle, ctypes.byref(v)))
        return float(v.value)

    def pool_times(self) -> tuple:
        """(entropy kernels, ranking + survivors, total) device ms of the last pool build."""
        out = np.zeros(3, dtype=np.float32)
        self.check(self.lib.fc_pool_times(self.handle, _ptr(out)))
        return tuple(float(v) for v in out)

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        self.check(self.lib.fc_launch_count(self.handle, ctypes.byref(n)))
        return int(n.value)


_default = {}
_default_lock = threading.Lock()


def pack_records(r: np.ndarray, abits, sbits, plen, slen):
    """FRAK payload of int32 records (host C, stream.py serialisation) ->
    (bytes, nbits); raises IndexError(row) for an out-of-range record."""
    lib = load_library()
    n = r.shape[0]
    stride = r.strides[0] // 4
    ab = np.ascontiguousarray(abits, dtype=np.int32)
    sb = np.ascontiguousarray(sbits, dtype=np.int32)
    pl = np.ascontiguousarray(plen, dtype=np.int64)
    sl = np.ascontiguousarray(slen, dtype=np.int64)
    cap = (n * (13 + int(ab.max()) + int(sb.max())) + 7) // 8 + 16
    out = np.empty(cap, dtype=np.uint8)
    nbits, bad = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.fc_pack_records(ctypes.c_void_p(r.ctypes.data), stride, n, _ptr(ab), _ptr(sb), _ptr(pl),
                             _ptr(sl), _ptr(out), cap, ctypes.byref(nbits), ctypes.byref(bad))
    if rc != FC_OK:
        raise IndexError(int(bad.value))
    return out[:(nbits.value + 7) // 8].tobytes(), int(nbits.value)


def default_context(device: int = 0) -> Context:
    with _default_lock:
        ctx = _default.get(device)
        if ctx is None:
            ctx = Context(device)
            _default[device] = ctx
        return ctx
