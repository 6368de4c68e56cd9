"""Flat grey/binary morphology on the device (reference morphology.py:23-140).

``StructuringElement`` keeps the reference's value semantics (offset tuples,
``box``/``ball``/``cross``/``parse``/``reflect``/``extent``/``z_extent``) so
registry params, CLI strings ("ball:3") and plans are interchangeable.  The
window reduction itself (``_window_reduce``, morphology.py:103-111: edge pad
then a min/max fold over every offset) runs in ``morph.cu``: the SE is
decomposed into (dz, dy) rows of contiguous x-runs and each run's sliding
min/max is computed once per slice.

Binary morphology is the same code on {0, 1} uint8 volumes, exactly as in the
reference (clamp-to-edge, not scipy's border_value=0).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ParameterError

MORPH_OPS = ("erode", "dilate", "open", "close")


def _check_radius(r):
    if r < 1:
        raise ParameterError(f"structuring element radius must be >= 1, got {r}")


@dataclass(frozen=True)
class StructuringElement:
    """A set of integer (dz, dy, dx) displacements that contains the origin."""

    offsets: tuple
    name: str = "custom"

    def __post_init__(self):
        if not self.offsets:
            raise ParameterError("structuring element must not be empty")
        if (0, 0, 0) not in self.offsets:
            raise ParameterError("structuring element must contain the origin")

    @property
    def extent(self) -> tuple:
        arr = np.abs(np.asarray(self.offsets, dtype=np.int64))
        return tuple(int(v) for v in arr.max(axis=0))

    @property
    def z_extent(self) -> int:
        return self.extent[0]

    def reflect(self) -> "StructuringElement":
        return StructuringElement(tuple(sorted((-a, -b, -c) for a, b, c in self.offsets)),
                                  name=self.name)

    def as_array(self) -> np.ndarray:
        return np.asarray(self.offsets, dtype=np.int32).reshape(-1, 3)

    @staticmethod
    def _cube(r):
        rng = range(-r, r + 1)
        return [(a, b, c) for a in rng for b in rng for c in rng]

    @classmethod
    def box(cls, r: int) -> "StructuringElement":
        _check_radius(r)
        return cls(tuple(cls._cube(r)), name=f"box:{r}")

    @classmethod
    def ball(cls, r: int) -> "StructuringElement":
        # Euclidean norm in voxel units (morphology.py:60-71)
        _check_radius(r)
        return cls(tuple(o for o in cls._cube(r) if o[0] ** 2 + o[1] ** 2 + o[2] ** 2 <= r * r),
                   name=f"ball:{r}")

    @classmethod
    def cross(cls, r: int) -> "StructuringElement":
        _check_radius(r)
        pts = {(0, 0, 0)}
        for d in range(-r, r + 1):
            pts.update({(d, 0, 0), (0, d, 0), (0, 0, d)})
        return cls(tuple(sorted(pts)), name=f"cross:{r}")

    @classmethod
    def parse(cls, spec: str) -> "StructuringElement":
        """'ball:2' / 'box:1' / 'cross:1' (morphology.py:84-95)."""
        kind, _, r = str(spec).partition(":")
        makers = {"box": cls.box, "ball": cls.ball, "cross": cls.cross}
        if kind not in makers:
            raise ParameterError(f"unknown structuring element {spec!r}")
        try:
            radius = int(r)
        except ValueError:
            raise ParameterError(f"bad structuring element radius in {spec!r}") from None
        return makers[kind](radius)


def morph_program(op: str, se: StructuringElement, iterations: int = 1) -> _native.DeviceProgram:
    """Stage chain for morph(op, se, iterations) (morphology.py:124-140)."""
    if op not in MORPH_OPS:
        raise ParameterError(f"op must be one of {MORPH_OPS}, got {op!r}")
    if iterations < 1:
        raise ParameterError(f"iterations must be >= 1, got {iterations}")
    off = se.as_array()
    E = lambda: _native.Stage(_native.OP_ERODE, offsets=off)  # noqa: E731
    D = lambda: _native.Stage(_native.OP_DILATE, offsets=off)  # noqa: E731 (library reflects)
    one = {"erode": [E], "dilate": [D], "open": [E, D], "close": [D, E]}[op]
    return _native.DeviceProgram([mk() for _ in range(iterations) for mk in one])


def erode(data, se: StructuringElement):
    """(I erode B)(p) = min_b I(p + b)."""
    from .filters import apply_program

    return apply_program(data, morph_program("erode", se))


def dilate(data, se: StructuringElement):
    """(I dilate B)(p) = max_b I(p - b)."""
    from .filters import apply_program

    return apply_program(data, morph_program("dilate", se))


def morph(data, op: str, se: StructuringElement, iterations: int = 1):
    """erode/dilate/open/close; open = dilate(erode(I)), close = erode(dilate(I))."""
    from .filters import apply_program

    return apply_program(data, morph_program(op, se, iterations))


# ---------------------------------------------------------------------------
# Label-volume filters (global operators) on the device labelling (cc.cu)
# ---------------------------------------------------------------------------
def _label_filter(data, op: int, connectivity: int, min_size: int = 0):
    import ctypes

    from . import _native

    if connectivity not in (6, 26):
        raise ParameterError(f"connectivity must be 6 or 26, got {connectivity}")
    L = _native.load()
    if hasattr(data, "data_ptr"):
        import torch

        x = data.contiguous()
        out = torch.empty_like(x)
    else:
        x = np.asarray(data)
        if x.ndim != 3:
            raise ParameterError(f"expected a 3D (Z, Y, X) volume, got shape {x.shape}")
        if x.dtype not in _native.DTYPE_CODE:
            raise ParameterError(f"label filters need uint8/16/32 or float32 data, got {x.dtype}")
        x = np.ascontiguousarray(x)
        out = np.empty_like(x)
    vin, _ = _native._volume_of(x)
    vout, _ = _native._volume_of(out)
    rc = L.hb_label_filter(ctypes.byref(vin), ctypes.byref(vout), op, int(connectivity),
                           int(min_size), _native.current_device())
    _native.raise_for_status(rc, _native.last_error())
    return out


def fill_holes(mask, connectivity: int = 6):
    """Fill the zero components that do not touch a volume face with 1
    (morphology.py:176-194); dtype preserved."""
    return _label_filter(mask, 0, connectivity)


def remove_islands(data, min_size: int, connectivity: int = 6):
    """Zero the components smaller than ``min_size`` voxels; voxels connect
    only to equal nonzero values, so touching labels stay separate
    (morphology.py:209-229)."""
    if min_size < 1:
        raise ParameterError(f"min_size must be >= 1, got {min_size}")
    return _label_filter(data, 1, connectivity, min_size)


def geodesic_reconstruct(marker, mask, kind: str = "dilation"):
    """Reconstruction by iterated geodesic steps until the fixed point
    (morphology.py:143-165): dilation: marker <= mask, step =
    min(dilate(m, cross(1)), mask); erosion: marker >= mask, step =
    max(erode(m, cross(1)), mask).  On the device with in-place sweeps (same
    unique fixed point)."""
    import ctypes

    from . import _native

    if kind not in ("dilation", "erosion"):
        raise ParameterError(f"kind must be dilation or erosion, got {kind!r}")
    mk, ms = np.asarray(marker), np.asarray(mask)
    if mk.shape != ms.shape or ms.ndim != 3:
        raise ParameterError("marker and mask must be 3D volumes of the same shape")
    dt = np.result_type(mk, ms)  # np.minimum/np.maximum promote
    if dt not in _native.DTYPE_CODE:
        raise ParameterError(f"geodesic reconstruction needs uint8/16/32 or float32 data, got {dt}")
    mk = np.ascontiguousarray(mk, dtype=dt)
    ms = np.ascontiguousarray(ms, dtype=dt)
    out = np.empty_like(ms)
    vm, _ = _native._volume_of(mk)
    vk, _ = _native._volume_of(ms)
    vo, _ = _native._volume_of(out)
    sweeps = ctypes.c_int64()
    rc = _native.load().hb_geodesic(ctypes.byref(vm), ctypes.byref(vk), ctypes.byref(vo),
                                    1 if kind == "dilation" else 0, _native.current_device(),
                                    ctypes.byref(sweeps))
    _native.raise_for_status(rc, _native.last_error())
    return out
