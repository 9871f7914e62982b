"""Real-valued slope analysis (reference bench.py:31-34, 86-215: S_BIN_EDGES,
SHistogram, s_histogram, shist_rows, SHIST_COLUMNS).

The quadtree runs with an exhaustive real-valued slope search: per (domain,
isometry) the unconstrained least-squares slope, per range the candidate with
the minimal projection error.  That search is ``fc_real_match_level``
(csrc/fc_real.cu): u8 x u8 dot products on the device and the reference's
three rounded fp64 steps, bit-identical to numpy's exact fp64 GEMM (see the
kernel header).  Only the histogram of the coded slopes is host work.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .codec import EncoderConfig, _quadtree
from .image import GrayImage
from .pool import build_pool

S_BIN_WIDTH = 0.05  # bench.py:31
S_BIN_EDGES = np.round(np.arange(-0.5, 1.5 + S_BIN_WIDTH / 2, S_BIN_WIDTH), 10)  # bench.py:32
SHIST_COLUMNS = ("pool_size", "level", "bin_low", "bin_high", "raw_count", "clamped_count")


@dataclass(frozen=True, eq=False)
class SHistogram:
    """Per-level histograms of the winning least-squares slope (bench.py:86-100).

    ``raw_counts`` bins the unconstrained slope clipped into [-0.5, 1.5];
    ``clamped_counts`` bins it clamped to [0, 1].  Rows are levels 1..4 and
    sum to the number of blocks coded at that level.
    """

    pool_size: int
    bin_edges: np.ndarray
    raw_counts: np.ndarray  # int64 [4, bins]
    clamped_counts: np.ndarray
    coded_blocks: tuple
    raw_means: tuple
    clamped_means: tuple


def real_s_matches(context, level: int, origins):
    """Per origin (errs f64, slopes f64, flat index e*8 + iso): bench.py:117-139
    ``_real_s_matches`` over codec.py:164 ``_gather_tiles``, on the device."""
    return context.real_match_level(level, origins)


def s_histogram(image: GrayImage, config: EncoderConfig, context=None) -> SHistogram:
    """bench.py:142-193: quadtree with the real-valued slope search, then the
    histogram of the winning slope of every coded block, per level."""
    ctx = context if context is not None else _native.default_context()
    build_pool(image, config.pool, context=ctx)
    s_by_level = {}

    def match_fn(level, origins):
        errs, slopes, _ = ctx.real_match_level(level, origins)
        s_by_level[level] = slopes
        return errs

    _, lv, jj = _quadtree(image.width, image.height, config.thresholds, match_fn)
    coded_by_level = [s_by_level[level][jj[lv == level]] if level in s_by_level else np.zeros(0)
                      for level in (1, 2, 3, 4)]
    raw, clamped = _slope_histograms(coded_by_level)
    stats = [(int(v.size), float(v.mean()) if v.size else None,
              float(np.clip(v, 0.0, 1.0).mean()) if v.size else None) for v in coded_by_level]
    coded, raw_means, clamped_means = (tuple(c) for c in zip(*stats))
    return SHistogram(pool_size=config.pool.pool_cap, bin_edges=S_BIN_EDGES.copy(),
                      raw_counts=raw, clamped_counts=clamped, coded_blocks=coded,
                      raw_means=raw_means, clamped_means=clamped_means)


def _slope_histograms(values_by_level):
    """[4, bins] counts of the coded slopes per level: the raw slope saturated
    to the edge range, and the slope clamped to [0, 1] (the coder's range)."""
    lo, hi = float(S_BIN_EDGES[0]), float(S_BIN_EDGES[-1])
    out = np.zeros((2, 4, len(S_BIN_EDGES) - 1), dtype=np.int64)
    for li, v in enumerate(values_by_level):
        if v.size == 0:
            continue
        for k, (a, b) in enumerate(((lo, hi), (0.0, 1.0))):
            out[k, li] = np.histogram(np.minimum(np.maximum(v, a), b), bins=S_BIN_EDGES)[0]
    return out[0], out[1]


def shist_rows(hist: SHistogram) -> list:
    """One dict per (level, bin) with the SHIST_COLUMNS keys (bench.py:196-212)."""
    nb = hist.raw_counts.shape[1]
    lows = [round(float(x), 4) for x in hist.bin_edges[:nb]]
    highs = [round(float(x), 4) for x in hist.bin_edges[1:nb + 1]]
    return [dict(zip(SHIST_COLUMNS, (hist.pool_size, li + 1, lows[b], highs[b],
                                     int(hist.raw_counts[li, b]), int(hist.clamped_counts[li, b]))))
            for li in range(4) for b in range(nb)]
