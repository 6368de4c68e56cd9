"""Benchmark harness of the drop-in API (reference: harpia/bench.py:1-118):
repeated timed ``run_operator`` calls over a ladder of volume sizes, reporting
mean/std time plus peak and residual tracked memory, as the reference does —
with the device columns of the B200 path next to them.

Same scenario fields, seeded synthetic volumes (``synthesize`` draws exactly
the reference's arrays: ``np.random.default_rng(seed)``, U[0,1) for float32,
the full integer range otherwise, bench.py:63-68), same CSV header
(bench.py:25).  Per-row time is the sum of the chunk times (device events)
unless ``include_io`` asks for the host wall time of the whole call
(bench.py:96-98).
"""

from __future__ import annotations

import csv
import statistics
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .chunking import MemoryBudget
from .errors import ParameterError
from .registry import run_operator
from .volume import load_volume

CSV_HEADER = ("size_bytes", "mean_s", "std_s", "peak_bytes", "residual_bytes")
# extension: device-side columns of the B200 executor
CSV_HEADER_DEVICE = CSV_HEADER + ("gvox_s", "device_peak_bytes", "device_residual_bytes",
                                  "h2d_bytes", "d2h_bytes")

DEFAULT_REPEATS = 30


@dataclass
class BenchScenario:
    """bench.py:30-51: operator, parameters, Z ladder over a base_yx^2 plane."""

    op: str
    params: dict = field(default_factory=dict)
    ladder: tuple = (64, 128, 192, 256)  # Z-slice counts
    base_yx: int = 64
    repeats: int = DEFAULT_REPEATS
    budget_bytes: int = 256 * 1024 * 1024
    fraction: float = 1.0
    seed: int = 0
    dtype: str = "uint8"
    warm: bool = False
    include_io: bool = False
    input_path: Optional[str] = None

    def __post_init__(self):
        if self.repeats < 1:
            raise ParameterError("repeats must be >= 1")
        lad = list(self.ladder)
        if len(lad) < 1 or lad != sorted(set(lad)):
            raise ParameterError("size ladder must be strictly increasing")


@dataclass(frozen=True)
class BenchRow:
    size_bytes: int
    mean_s: float
    std_s: float
    peak_bytes: int
    residual_bytes: int
    # device extension (not part of the reference's CSV)
    gvox_s: float = 0.0
    device_peak_bytes: int = 0
    device_residual_bytes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def as_tuple(self):
        return (self.size_bytes, self.mean_s, self.std_s, self.peak_bytes, self.residual_bytes)

    def as_device_tuple(self):
        return self.as_tuple() + (self.gvox_s, self.device_peak_bytes, self.device_residual_bytes,
                                  self.h2d_bytes, self.d2h_bytes)


def synthesize(z: int, yx: int, dtype: str, seed: int) -> np.ndarray:
    """The reference's seeded synthetic volume (bench.py:63-68), bit for bit."""
    gen = np.random.default_rng(seed)
    if np.dtype(dtype) == np.float32:
        return gen.random((z, yx, yx), dtype=np.float32)
    lim = np.iinfo(dtype)
    return gen.integers(lim.min, lim.max + 1, size=(z, yx, yx), dtype=dtype)


def run_bench(scenario: BenchScenario) -> list:
    """bench.py:71-110 on the device executor: one row per ladder entry."""
    budget = MemoryBudget(scenario.budget_bytes, scenario.fraction)
    source = load_volume(scenario.input_path) if scenario.input_path is not None else None
    out = []
    for z in scenario.ladder:
        if source is not None:
            if z > source.shape[0]:
                raise ParameterError(f"ladder entry {z} exceeds input Z={source.shape[0]}")
            base = source.data[:z]
        else:
            base = synthesize(z, scenario.base_yx, scenario.dtype, scenario.seed)
        warm_input = np.ascontiguousarray(base)
        samples, peak, residual, rep = [], 0, 0, None
        for _ in range(scenario.repeats):
            # cold repeats hand the operator a fresh buffer, like the reference
            data = warm_input if scenario.warm else np.array(base, copy=True)
            t0 = time.perf_counter()
            _, rep = run_operator(data, scenario.op, scenario.params, budget)
            wall = time.perf_counter() - t0
            samples.append(wall if scenario.include_io else (rep.wall_seconds or wall))
            peak = max(peak, rep.peak_bytes)
            residual = rep.residual_bytes
        mean = statistics.fmean(samples)
        voxels = int(np.prod(base.shape))
        out.append(BenchRow(
            size_bytes=int(base.nbytes), mean_s=mean,
            std_s=statistics.stdev(samples) if len(samples) > 1 else 0.0,
            peak_bytes=peak, residual_bytes=residual,
            gvox_s=voxels / mean / 1e9 if mean > 0 else 0.0,
            device_peak_bytes=int(getattr(rep, "device_peak_bytes", 0)),
            device_residual_bytes=int(getattr(rep, "device_residual_bytes", 0)),
            h2d_bytes=int(getattr(rep, "h2d_bytes", 0)), d2h_bytes=int(getattr(rep, "d2h_bytes", 0))))
    return out


def write_csv(rows, path, device_columns: bool = False) -> None:
    """The reference's CSV (bench.py:113-118); ``device_columns`` appends the
    B200 executor's columns."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_HEADER_DEVICE if device_columns else CSV_HEADER)
        for r in rows:
            w.writerow(r.as_device_tuple() if device_columns else r.as_tuple())
