"""Raw ``.vol`` volumes streamed straight into the device executor.

SURVEY.md §8(f) row 1: the reference reads a whole ``.vol`` into RAM before
processing (``load_volume``, volume.py:159-185), so its out-of-core story ends
at host memory.  Here the same on-disk format — raw little-endian C-order
(Z, Y, X) samples plus a ``.vol.meta`` text sidecar (volume.py:28-75,
README.md:34-48) — is memory-mapped, and ``filter_file`` runs a registry
operator from one file to another through the chunked streaming executor:
disk pages -> pinned staging -> sm_100a kernels -> pinned staging -> disk, with
host RAM bounded by the pipeline's staging buffers instead of the volume size.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import CorruptInputError, ParameterError, UnsupportedFormatError
from .ledger import LEDGER

SUPPORTED_DTYPES = {"uint8": np.dtype("uint8"), "uint16": np.dtype("uint16"),
                    "float32": np.dtype("float32")}
LABEL_DTYPE = np.dtype("uint32")


@dataclass
class VolumeMeta:
    """Sidecar fields (the reference's text format, volume.py:28-75)."""

    dtype: str
    shape: tuple
    spacing: tuple
    byte_order: str = "little"
    offset_bytes: int = 0
    description: str = ""

    def to_text(self) -> str:
        z, y, x = self.shape
        sz, sy, sx = self.spacing
        return (f"dtype: {self.dtype}\nshape: {z} {y} {x}\n"
                f"spacing: {sz!r} {sy!r} {sx!r}\nbyte_order: {self.byte_order}\n"
                f"offset_bytes: {self.offset_bytes}\ndescription: {self.description}\n")

    @classmethod
    def from_text(cls, text: str) -> "VolumeMeta":
        kv = {}
        for line in text.splitlines():
            if line.strip():
                k, _, v = line.partition(":")
                kv[k.strip()] = v.strip()
        try:
            dtype = kv["dtype"]
            shape = tuple(int(v) for v in kv["shape"].split())
            spacing = tuple(float(v) for v in kv["spacing"].split())
        except (KeyError, ValueError) as exc:
            raise UnsupportedFormatError(f"malformed sidecar: {exc}") from exc
        if dtype not in SUPPORTED_DTYPES:
            raise UnsupportedFormatError(f"unsupported dtype {dtype!r}")
        if len(shape) != 3 or len(spacing) != 3:
            raise UnsupportedFormatError("shape and spacing must have 3 components")
        return cls(dtype=dtype, shape=shape, spacing=spacing,
                   byte_order=kv.get("byte_order", "little"),
                   offset_bytes=int(kv.get("offset_bytes", "0")),
                   description=kv.get("description", ""))


@dataclass
class Volume:
    """Dense (Z, Y, X) scalar grid; ``data`` may be an in-RAM array or a memmap."""

    data: np.ndarray
    spacing: tuple = (1.0, 1.0, 1.0)
    description: str = ""

    def __post_init__(self):
        if self.data.ndim != 3:
            raise ParameterError(f"volume data must be 3D, got ndim={self.data.ndim}")
        if str(self.data.dtype) not in SUPPORTED_DTYPES:
            raise UnsupportedFormatError(f"unsupported dtype {self.data.dtype}")
        if len(self.spacing) != 3 or any(s <= 0 for s in self.spacing):
            raise ParameterError(f"spacing components must be strictly positive, got {self.spacing}")
        self.spacing = tuple(float(s) for s in self.spacing)

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    @property
    def nbytes(self) -> int:
        return self.data.nbytes

    def meta(self) -> VolumeMeta:
        return VolumeMeta(dtype=str(self.dtype), shape=tuple(self.shape), spacing=self.spacing,
                          description=self.description)


def default_meta_path(data_path) -> str:
    return str(data_path) + ".meta"


def _read_meta(data_path, meta_path):
    with open(meta_path or default_meta_path(data_path), "r", encoding="utf-8") as fh:
        meta = VolumeMeta.from_text(fh.read())
    if meta.byte_order != "little":
        raise UnsupportedFormatError("only little-endian volumes are supported")
    dt = SUPPORTED_DTYPES[meta.dtype]
    z, y, x = meta.shape
    expected = meta.offset_bytes + z * y * x * dt.itemsize
    actual = os.path.getsize(data_path)
    if actual != expected:
        raise CorruptInputError(
            f"{data_path}: file is {actual} bytes, sidecar implies {expected} "
            f"(offset {meta.offset_bytes} + {z * y * x} x {dt.itemsize})")
    return meta, dt


def load_volume(data_path, meta_path=None, mmap: bool = True) -> Volume:
    """Open a ``.vol`` (volume.py:159-185).  ``mmap=True`` (default) maps the
    file instead of reading it, so volumes larger than host RAM can be streamed
    through ``run_operator``; ``mmap=False`` reads it like the reference and
    charges the ledger."""
    meta, dt = _read_meta(data_path, meta_path)
    if mmap:
        data = np.memmap(data_path, dtype=dt, mode="r", offset=meta.offset_bytes, shape=meta.shape)
    else:
        with open(data_path, "rb") as fh:
            fh.seek(meta.offset_bytes)
            data = np.frombuffer(fh.read(), dtype=dt).reshape(meta.shape)
        LEDGER.charge(data.nbytes)
    return Volume(data=data, spacing=meta.spacing, description=meta.description)


def create_volume(data_path, shape, dtype, spacing=(1.0, 1.0, 1.0), description="",
                  meta_path=None) -> Volume:
    """Create a writable memory-mapped ``.vol`` (+ sidecar) of the given geometry."""
    dt = np.dtype(dtype)
    if str(dt) not in SUPPORTED_DTYPES:
        raise UnsupportedFormatError(f"unsupported dtype {dt}")
    vol = Volume(data=np.memmap(data_path, dtype=dt, mode="w+", shape=tuple(shape)),
                 spacing=spacing, description=description)
    with open(meta_path or default_meta_path(data_path), "w", encoding="utf-8") as fh:
        fh.write(vol.meta().to_text())
    return vol


def save_volume(volume: Volume, data_path, meta_path=None) -> None:
    """Write raw little-endian samples plus the sidecar (volume.py:188-198)."""
    out = create_volume(data_path, volume.shape, volume.dtype, volume.spacing,
                        volume.description, meta_path)
    step = max(1, (256 << 20) // max(1, volume.data[0].nbytes))
    for z0 in range(0, volume.shape[0], step):
        out.data[z0:z0 + step] = volume.data[z0:z0 + step]
    out.data.flush()


def filter_file(in_path, out_path, name: str, params: Optional[dict] = None, budget=None,
                cancel=None):
    """Apply registry operator ``name`` from ``in_path`` to ``out_path`` (both
    ``.vol`` + sidecar), streaming through the device executor; returns the
    ExecutionReport.  The output dtype follows the operator (float32 for the
    smoothing filters, the input dtype for median/morphology)."""
    from . import filters, registry
    from .chunking import execute_chunked, profile_budget

    src = load_volume(in_path, mmap=True)
    op = registry.get_operator(name)
    p = registry.validate_params(op, params or {})
    program = op.program(p)
    out_dt = program.out_dtype(src.dtype)
    dst = create_volume(out_path, src.shape, out_dt, src.spacing, src.description)
    if budget is None:
        budget = profile_budget()
    arr, restore = filters.coerce_input(src.data, program)
    if restore is not None:
        raise UnsupportedFormatError("file streaming needs a device dtype")
    _, report = execute_chunked(arr, program, op.profile(p), budget, p, cancel=cancel,
                                out=dst.data)
    dst.data.flush()
    return report
