"""Thresholds of the drop-in API (reference threshold.py), all on the device:
``apply_threshold`` and ``local_threshold`` are map operators through the
chunk executor; global Otsu is the two-pass operator of SURVEY.md §8(f) row 3."""

from __future__ import annotations

import numpy as np

from . import filters

LABEL_DTYPE = np.dtype("uint32")  # volume.py:23


def apply_threshold(data, t: float):
    """Binary labels: foreground (1) where v > t, as uint32 (threshold.py:110-112).

    Same comparison as NumPy 2: float32 data against float32(t), integer data
    in float64."""
    return filters.apply_program(data, filters.threshold_program(t))


# ---------------------------------------------------------------------------
# Global Otsu (threshold.py:25-131) as a two-pass operator on the device:
# pass 1 = device range + histogram (hb_minmax / hb_histogram, np.histogram
# bit for bit), host finalize = the Otsu split, pass 2 = the apply_threshold
# map program through the chunk executor.
# ---------------------------------------------------------------------------
from dataclasses import dataclass  # noqa: E402

from . import _native  # noqa: E402
from .errors import HarpiaError, ParameterError  # noqa: E402

DEFAULT_BINS = 256


@dataclass(frozen=True)
class Histogram:
    """Fixed-range counts, mergeable by addition (threshold.py:25-43) — the
    unit a multi-GPU job all-reduces (sharding.otsu_sharded)."""

    lo: float
    hi: float
    counts: np.ndarray  # int64

    @property
    def bin_count(self) -> int:
        return self.counts.size

    @property
    def bin_width(self) -> float:
        return (self.hi - self.lo) / self.bin_count

    def merge(self, other: "Histogram") -> "Histogram":
        if (self.lo, self.hi, self.bin_count) != (other.lo, other.hi, other.bin_count):
            raise ParameterError("histograms with different binning cannot merge")
        return Histogram(self.lo, self.hi, self.counts + other.counts)


def _device_array(data):
    a = data if hasattr(data, "data_ptr") else np.ascontiguousarray(data)
    dt = np.dtype(str(a.dtype).replace("torch.", "")) if hasattr(a, "data_ptr") else a.dtype
    if dt not in _native.DTYPE_CODE:
        a = np.ascontiguousarray(np.asarray(a), dtype=np.float32)
    return a


def data_minmax(data) -> tuple:
    """(min, max) of a float volume, reduced on the device (hb_minmax)."""
    return _native.minmax(_device_array(data))


def histogram_range(data) -> tuple:
    """Bin range (threshold.py:46-55): the full dtype range for integers,
    (min, max) for floats — min/max reduced on the device."""
    a = _device_array(data)
    dt = np.dtype(str(a.dtype).replace("torch.", "")) if hasattr(a, "data_ptr") else a.dtype
    if np.issubdtype(dt, np.integer):
        lim = np.iinfo(dt)
        return float(lim.min), float(lim.max) + 1.0
    lo, hi = data_minmax(a)
    return (lo, lo + 1.0) if lo == hi else (lo, hi)


def compute_histogram(data, bins: int = DEFAULT_BINS, rng=None) -> Histogram:
    """np.histogram(data, bins, range=rng) counts on the device (threshold.py:58-62)."""
    if bins < 1:
        raise ParameterError(f"bins must be >= 1, got {bins}")
    a = _device_array(data)
    if rng is None:
        rng = histogram_range(a)
    lo, hi = float(rng[0]), float(rng[1])
    dt = np.dtype(str(a.dtype).replace("torch.", "")) if hasattr(a, "data_ptr") else a.dtype
    # numpy's bin dtype: float32 for float32 data (python-float range is weak), else float64
    bin_type = np.float32 if dt == np.float32 else np.float64
    edges = np.linspace(lo, hi, int(bins) + 1, dtype=bin_type)
    counts = _native.histogram(a, int(bins), lo, hi, edges, bin_type == np.float32)
    return Histogram(lo, hi, counts)


def otsu_from_histogram(hist: Histogram) -> float:
    """The split maximising the between-class variance w0*w1*(mu0 - mu1)^2,
    first on ties; the left edge of the highest background bin
    (threshold.py:65-87, same float64 arithmetic)."""
    c = hist.counts.astype(np.float64)
    n = c.sum()
    if n <= 0:
        raise HarpiaError("empty histogram")
    k = np.arange(hist.bin_count, dtype=np.float64)
    cw = np.cumsum(c)
    cm = np.cumsum(c * k)
    rest_w = n - cw
    rest_m = cm[-1] - cm
    ok = (cw > 0) & (rest_w > 0)
    if not ok.any():
        raise HarpiaError("degenerate histogram: all voxels share one bin")
    with np.errstate(divide="ignore", invalid="ignore"):
        score = np.where(ok, cw * rest_w * (cm / cw - rest_m / rest_w) ** 2, -np.inf)
    return hist.lo + int(np.argmax(score)) * hist.bin_width


def otsu(data, bins: int = DEFAULT_BINS, budget=None) -> float:
    """Global Otsu threshold (threshold.py:90-107).  The device streams the
    volume in bounded slabs, so ``budget`` only matters for pass 2."""
    return otsu_from_histogram(compute_histogram(data, bins))


def otsu_binarize(data, bins: int = DEFAULT_BINS, budget=None, cancel=None):
    """Threshold with Otsu and binarize (threshold.py:115-131): (labels, t)."""
    from .chunking import OpProfile, execute_chunked

    t = otsu(data, bins, budget)
    prog = filters.threshold_program(t)
    if budget is None:
        return filters.apply_program(data, prog, cancel=cancel), t
    arr, _ = filters.coerce_input(data, prog)
    out, _ = execute_chunked(arr, prog, OpProfile(halo_z=0, scratch_factor=6, out_dtype=LABEL_DTYPE),
                             budget, cancel=cancel, fresh_job=False)
    return out, t


# ---------------------------------------------------------------------------
# Local adaptive thresholds (threshold.py:166-217) — one device map stage
# (local.cu); chunked like any map operator (halo = window).
# ---------------------------------------------------------------------------
LOCAL_KINDS = _native.LOCAL_KINDS


def default_sauvola_r(dtype) -> float:
    """Half the dtype range (127.5 for uint8); 0.5 for float data (threshold.py:166-171)."""
    if np.issubdtype(np.dtype(dtype), np.integer):
        info = np.iinfo(dtype)
        return (info.max - info.min) / 2.0
    return 0.5


def local_threshold(data, kind: str, window: int, k: float = 0.2, r=None, c: float = 0.0):
    """Adaptive binarization (threshold.py:174-217): labels = data > T with
    T from the clamped (2w+1)^3 window — mean: m - c; median: med - c;
    gaussian: gaussian-weighted mean (sigma = w/2) - c; niblack: m + k*s;
    sauvola: m*(1 + k*(s/R - 1)); s the population std-dev."""
    dt = data.dtype if hasattr(data, "dtype") else np.asarray(data).dtype
    dt = np.dtype(str(dt).replace("torch.", ""))
    return filters.apply_program(data, filters.local_threshold_program(kind, window, k, r, c, dtype=dt))
