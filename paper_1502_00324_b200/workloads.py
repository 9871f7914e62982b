"""Seeded synthetic inputs for the BASELINE.json configs (c1..c5).

No public dataset is involved: the reference's own test images are synthetic
stand-ins too (pkg/tools/make_fixtures.py).  These generators follow
SURVEY.md section 8(d); both the oracle and the device path consume the same
generated uint8 arrays, so generator details affect throughput, not parity.

fBm convention (frozen): spectral power proportional to |f|^-(2H+1) on a
Gaussian spectrum drawn from numpy.random.default_rng(seed), zero DC, real
part of the inverse FFT, min-max rescaled to [0, 255], np.rint, uint8.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _to_u8(a: np.ndarray) -> np.ndarray:
    lo, hi = float(a.min()), float(a.max())
    if hi == lo:
        return np.zeros(a.shape, dtype=np.uint8)
    return np.rint((a - lo) * (255.0 / (hi - lo))).astype(np.uint8)


def fbm(size: int, hurst: float, seed: int) -> np.ndarray:
    """Square fBm-like field with power spectrum ~ |f|^-(2H+1) (float64)."""
    rng = np.random.default_rng(seed)
    fy = np.fft.fftfreq(size)[:, None]
    fx = np.fft.fftfreq(size)[None, :]
    f = np.sqrt(fx * fx + fy * fy)
    f[0, 0] = 1.0
    amp = f ** (-(2.0 * hurst + 1.0) / 2.0)
    amp[0, 0] = 0.0
    spec = amp * (rng.standard_normal((size, size)) + 1j * rng.standard_normal((size, size)))
    return np.real(np.fft.ifft2(spec))


def fbm_image(size: int, hurst: float, seed: int, noise_sigma: float = 0.0) -> np.ndarray:
    img = _to_u8(fbm(size, hurst, seed)).astype(np.float64)
    if noise_sigma > 0:
        rng = np.random.default_rng(seed + 1_000_003)
        img = img + rng.normal(0.0, noise_sigma, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def mix_image(size: int, seed: int) -> np.ndarray:
    """Gradients + 12 constant rectangles + N(0, 8) noise (config 2/3)."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:size, 0:size].astype(np.float64) / size
    a, b = rng.uniform(-120, 120, 2)
    img = 128.0 + a * (x - 0.5) + b * (y - 0.5)
    cx, cy = rng.uniform(0.2, 0.8, 2)
    img += rng.uniform(-60, 60) * np.sqrt((x - cx) ** 2 + (y - cy) ** 2)
    for _ in range(12):
        w, h = rng.integers(size // 16, size // 3, 2)
        x0 = rng.integers(0, size - w)
        y0 = rng.integers(0, size - h)
        img[y0 : y0 + h, x0 : x0 + w] = rng.uniform(0, 255)
    img += rng.normal(0.0, 8.0, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config expressed in reference parameters."""

    name: str
    description: str
    size: int
    images: int
    strides: tuple
    thresholds: tuple
    # entropy threshold per level (device keeps ent > tau), None = keep all;
    # levels a config never codes use cap 1 on both sides (cap_one)
    taus: tuple
    cap_one: tuple

    def image(self, index: int = 0) -> np.ndarray:
        return make_image(self.name, index)


def make_image(name: str, index: int = 0) -> np.ndarray:
    if name == "c1":
        return fbm_image(128, 0.5, index)
    if name in ("c2", "c3"):
        return mix_image(512, index)
    if name == "c4":
        return fbm_image(2048, 0.7, index, noise_sigma=4.0)
    if name == "c5":
        return fbm_image(2048, 0.5, index)
    raise KeyError(name)


# Frozen entropy thresholds tau_l: np.quantile of each level's window
# entropies on the seed-0 image -- p50 for c1, p90 for c2-c4.
# None = keep every window of that level (c5: no pruning).
WORKLOADS = {
    "c1": Workload("c1", "128x128 fBm H=0.5; ranges 8->4, domains L=4, p50 entropy pools",
                   128, 1, (8, 4, 2, 2), (1e-9, 8.0, 1e9),
                   (None, 4.397750417928178, 3.7146239359169204, None),
                   (True, False, False, True)),
    "c2": Workload("c2", "512x512 gradients+rectangles+N(0,8); ranges 16->8->4, L=1, p90 entropy pools",
                   512, 1, (1, 1, 1, 1), (8.0, 8.0, 1e9),
                   (4.098931051341678, 3.8470957291411865, 3.3126049018053845, None),
                   (False, False, False, True)),
    "c3": Workload("c3", "64 x 512x512 (seeds 0..63); ranges 8->4, L=2, p90 entropy pools",
                   512, 64, (8, 2, 2, 2), (1e-9, 8.0, 1e9),
                   (None, 3.8470683733814868, 3.3126049018053845, None),
                   (True, False, False, True)),
    "c4": Workload("c4", "2048x2048 fBm H=0.7 + N(0,4); ranges 16->8->4, L=2, p90 entropy pools",
                   2048, 1, (2, 2, 2, 2), (8.0, 8.0, 1e9),
                   (4.17553672583301, 3.91019391709399, 3.4412086460607636, None),
                   (False, False, False, True)),
    "c5": Workload("c5", "2048x2048 fBm H=0.5; exhaustive B=8 level, L=1, no pruning",
                   2048, 1, (8, 1, 2, 2), (1e-9, 1e9, 1e9),
                   (None, None, None, None),
                   (True, False, True, True)),
}


def encoder_config(name: str, path: str = "auto"):
    """The EncoderConfig of a workload: frozen entropy thresholds as device
    threshold compaction (ent > tau), cap 1 on the levels it never codes."""
    from .codec import EncoderConfig
    from .pool import PoolParams

    wl = WORKLOADS[name]
    taus = tuple(None if one else t for one, t in zip(wl.cap_one, wl.taus))
    caps = tuple(1 if one else 2**31 - 1 for one in wl.cap_one)
    params = PoolParams(pool_cap=2**31 - 1, strides=wl.strides, level_caps=caps,
                        entropy_thresholds=taus)
    return EncoderConfig(pool=params, thresholds=wl.thresholds, path=path)
