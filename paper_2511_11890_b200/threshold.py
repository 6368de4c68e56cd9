"""Thresholding map operator of the drop-in API (reference threshold.py).

Only the local map operator ``apply_threshold`` (threshold.py:110-112) is on
the device path; Otsu / local thresholds are two-pass global operators,
SURVEY.md §8(f) row 3 (not built here)."""

from __future__ import annotations

import numpy as np

from . import filters

LABEL_DTYPE = np.dtype("uint32")  # volume.py:23


def apply_threshold(data, t: float):
    """Binary labels: foreground (1) where v > t, as uint32 (threshold.py:110-112).

    Same comparison as NumPy 2: float32 data against float32(t), integer data
    in float64."""
    return filters.apply_program(data, filters.threshold_program(t))
