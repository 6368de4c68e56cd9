"""Connected-components labelling of the drop-in API (reference quantify.py).

``connected_components`` (quantify.py:60-111) runs on the device
(hb_connected_components, cc.cu): a lock-free union-find whose links point to
the smaller index, so each component's root is its first voxel in scan order,
then an exclusive scan numbers the roots — exactly the reference's canonical
labels (1..count in first-occurrence order, quantify.py:48-57), whatever the
chunk plan.  The per-label metrics, EDT and CSV export are out of scope
(SURVEY.md §8(f))."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ParameterError

LABEL_DTYPE = np.dtype("uint32")  # volume.py:23


def connected_components(mask, connectivity: int = 6, budget=None):
    """Label a binary mask (nonzero = foreground); returns (labels, count).

    ``budget`` is accepted for API compatibility: the device labels the whole
    volume in HBM (the reference's chunked path merges per-chunk labels with a
    host union-find and yields the same canonical labels)."""
    if connectivity not in (6, 26):
        raise ParameterError(f"connectivity must be 6 or 26, got {connectivity}")
    L = _native.load()
    if hasattr(mask, "data_ptr"):
        import torch

        x = mask.contiguous()
        if x.dtype == torch.bool:
            x = x.to(torch.uint8)
        out = torch.empty(tuple(x.shape), dtype=torch.uint32, device=x.device)
        vin, _ = _native._volume_of(x)
        vout, _ = _native._volume_of(out)
    else:
        x = np.asarray(mask)
        if x.ndim != 3:
            raise ParameterError(f"expected a 3D (Z, Y, X) volume, got shape {x.shape}")
        if x.dtype not in _native.DTYPE_CODE:
            x = (x != 0).astype(np.uint8)
        x = np.ascontiguousarray(x)
        out = np.empty(x.shape, LABEL_DTYPE)
        vin, _ = _native._volume_of(x)
        vout, _ = _native._volume_of(out)
    n = ctypes.c_int64()
    rc = L.hb_connected_components(ctypes.byref(vin), ctypes.byref(vout), int(connectivity),
                                   _native.current_device(), ctypes.byref(n))
    _native.raise_for_status(rc, _native.last_error())
    return out, int(n.value)


def edt(mask, spacing=(1.0, 1.0, 1.0), squared: bool = False):
    """Exact Euclidean distance of every nonzero voxel to the nearest zero
    voxel, with per-axis (z, y, x) spacing (quantify.py:161-175): float32, or
    the float64 squared distances when ``squared``; +inf without background.
    Device: one Felzenszwalb-Huttenlocher scan per line and axis (edt.cu)."""
    x = np.asarray(mask)
    if x.ndim != 3:
        raise ParameterError(f"expected a 3D (Z, Y, X) volume, got shape {x.shape}")
    if x.dtype not in _native.DTYPE_CODE:
        x = (x != 0).astype(np.uint8)
    x = np.ascontiguousarray(x)
    sp = np.ascontiguousarray([float(s) for s in spacing], dtype=np.float64)
    if sp.size != 3:
        raise ParameterError("spacing must have three entries (z, y, x)")
    out = np.empty(x.shape, np.float64 if squared else np.float32)
    vin, _ = _native._volume_of(x)
    vout = _native.HbVolume(out.ctypes.data, 4 if squared else _native.DTYPE_CODE[np.dtype(np.float32)],
                            _native.HB_HOST, *out.shape)  # 4 = HB_F64 (squared output only)
    rc = _native.load().hb_edt(ctypes.byref(vin), ctypes.byref(vout), sp.ctypes.data,
                               _native.current_device())
    _native.raise_for_status(rc, _native.last_error())
    return out
