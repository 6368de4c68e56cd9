"""ctypes binding of the C ABI in include/harpia_b200.h.

This module is the only door into the device code.  There is no CPU fallback:
if ``_lib/libharpia_b200.so`` is missing or no CUDA device is present, every
compute entry point raises (``RuntimeError`` for a missing library,
``BudgetUnavailableError`` for a missing device).
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

from .errors import HB_OK, ParameterError, UnsupportedFormatError, raise_for_status

# HARPIA_LIB: developer A/B of library builds (tools/gpu/ab_*.py); default in-tree
LIB_PATH = Path(os.environ.get("HARPIA_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libharpia_b200.so")

# enum values of include/harpia_b200.h
HB_U8, HB_U16, HB_U32, HB_F32 = 0, 1, 2, 3
HB_HOST, HB_DEVICE = 0, 1
OP_IDENTITY, OP_GAUSSIAN, OP_MEAN, OP_MEDIAN, OP_UNSHARP, OP_LOG, OP_ERODE, OP_DILATE = range(8)
OP_HESSIAN, OP_SOBEL, OP_PREWITT, OP_THRESHOLD, OP_LBP2D, OP_DIFFUSION = range(8, 14)
OP_LOCAL_THRESHOLD = 14
# hb_local_kind: threshold.LOCAL_KINDS order (threshold.py:21)
LOCAL_KINDS = ("mean", "median", "gaussian", "niblack", "sauvola")
PREC_FAST, PREC_EXACT = 0, 1

DTYPE_CODE = {
    np.dtype("uint8"): HB_U8,
    np.dtype("uint16"): HB_U16,
    np.dtype("uint32"): HB_U32,
    np.dtype("float32"): HB_F32,
}
CODE_DTYPE = {v: k for k, v in DTYPE_CODE.items()}


class HbVolume(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("location", ctypes.c_int32),
        ("nz", ctypes.c_int64),
        ("ny", ctypes.c_int64),
        ("nx", ctypes.c_int64),
    ]


class HbStage(ctypes.Structure):
    _fields_ = [
        ("op", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("sigma", ctypes.c_double),
        ("amount", ctypes.c_double),
        ("radius", ctypes.c_int32),
        ("n_offsets", ctypes.c_int32),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("n_weights", ctypes.c_int32),
        ("weights", ctypes.POINTER(ctypes.c_float)),
        ("weights64", ctypes.POINTER(ctypes.c_double)),
    ]


class HbChunk(ctypes.Structure):
    _fields_ = [
        ("z_start", ctypes.c_int64),
        ("z_stop", ctypes.c_int64),
        ("halo_lo", ctypes.c_int64),
        ("halo_hi", ctypes.c_int64),
    ]


CANCEL_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p)


class HbExec(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("pipeline_depth", ctypes.c_int32),
        ("device_budget", ctypes.c_int64),
        ("cancel", CANCEL_FN),
        ("cancel_ctx", ctypes.c_void_p),
        ("chunk_seconds", ctypes.POINTER(ctypes.c_double)),
        ("fault_chunk", ctypes.c_int32),
        ("host_threads", ctypes.c_int32),
    ]


class HbReport(ctypes.Structure):
    _fields_ = [
        ("chunk_count", ctypes.c_int64),
        ("failed_chunk", ctypes.c_int64),
        ("minimum_bytes", ctypes.c_int64),
        ("device_peak_bytes", ctypes.c_int64),
        ("device_residual_bytes", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("h2d_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("wall_ms", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("message", ctypes.c_char * 512),
    ]


# Every symbol include/harpia_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "hb_abi_version", "hb_version", "hb_device_info", "hb_device_count",
    "hb_gaussian_radius", "hb_gaussian_weights", "hb_chain_halo", "hb_run",
    "hb_apply_device", "hb_chain_out_dtype", "hb_trim_device",
    "hb_device_pool_bytes", "hb_pin", "hb_unpin", "hb_last_error",
    "hb_session_begin", "hb_session_end", "hb_minmax", "hb_histogram",
    "hb_connected_components", "hb_label_filter", "hb_geodesic", "hb_edt", "hb_plan",
    "hb_run_multi", "hb_device_alloc", "hb_device_free",
)

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the device library; raise loudly if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback for the hot path)")
        L = ctypes.CDLL(str(LIB_PATH))
        i32, i64, vp, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
        L.hb_abi_version.restype = i32
        L.hb_version.restype = ctypes.c_char_p
        L.hb_last_error.restype = ctypes.c_char_p
        L.hb_device_count.restype = i32
        L.hb_device_info.argtypes = [i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.hb_device_info.restype = i32
        L.hb_gaussian_radius.argtypes = [dbl]
        L.hb_gaussian_radius.restype = i32
        L.hb_gaussian_weights.argtypes = [dbl, ctypes.POINTER(ctypes.c_float), i32]
        L.hb_gaussian_weights.restype = i32
        L.hb_chain_halo.argtypes = [ctypes.POINTER(HbStage), i32]
        L.hb_chain_halo.restype = i64
        L.hb_chain_out_dtype.argtypes = [ctypes.POINTER(HbStage), i32, i32]
        L.hb_chain_out_dtype.restype = i32
        L.hb_run.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume),
                             ctypes.POINTER(HbStage), i32, ctypes.POINTER(HbChunk), i64,
                             ctypes.POINTER(HbExec), ctypes.POINTER(HbReport)]
        L.hb_run.restype = i32
        L.hb_apply_device.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume),
                                      ctypes.POINTER(HbStage), i32, i64, vp, i32,
                                      ctypes.POINTER(HbReport)]
        L.hb_apply_device.restype = i32
        L.hb_run_multi.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume),
                                   ctypes.POINTER(HbStage), i32, ctypes.POINTER(HbChunk), i64,
                                   ctypes.POINTER(HbExec), i32, ctypes.POINTER(i32),
                                   ctypes.POINTER(HbReport), ctypes.POINTER(HbReport)]
        L.hb_run_multi.restype = i32
        L.hb_device_alloc.argtypes = [i32, i64, vp, ctypes.POINTER(vp)]
        L.hb_device_alloc.restype = i32
        L.hb_device_free.argtypes = [i32, vp, vp]
        L.hb_device_free.restype = i32
        L.hb_trim_device.argtypes = [i32]
        L.hb_trim_device.restype = i32
        L.hb_device_pool_bytes.argtypes = [i32]
        L.hb_device_pool_bytes.restype = i64
        L.hb_session_begin.argtypes = [i32]
        L.hb_session_begin.restype = i32
        L.hb_session_end.argtypes = [i32]
        L.hb_session_end.restype = i32
        L.hb_minmax.argtypes = [ctypes.POINTER(HbVolume), i32, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double)]
        L.hb_minmax.restype = i32
        L.hb_histogram.argtypes = [ctypes.POINTER(HbVolume), i32, i32, ctypes.c_double,
                                   ctypes.c_double, vp, i32, vp]
        L.hb_histogram.restype = i32
        L.hb_connected_components.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume),
                                              i32, i32, ctypes.POINTER(ctypes.c_int64)]
        L.hb_connected_components.restype = i32
        L.hb_label_filter.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume), i32, i32,
                                      i64, i32]
        L.hb_label_filter.restype = i32
        L.hb_geodesic.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume),
                                  ctypes.POINTER(HbVolume), i32, i32, ctypes.POINTER(ctypes.c_int64)]
        L.hb_geodesic.restype = i32
        L.hb_edt.argtypes = [ctypes.POINTER(HbVolume), ctypes.POINTER(HbVolume), vp, i32]
        L.hb_edt.restype = i32
        L.hb_pin.argtypes = [vp, i64]
        L.hb_pin.restype = i32
        L.hb_unpin.argtypes = [vp]
        L.hb_unpin.restype = i32
        if L.hb_abi_version() != 1:
            raise RuntimeError("libharpia_b200.so ABI version mismatch")
        _lib = L
        return L


def device_count() -> int:
    return int(load().hb_device_count())


def device_info(dev: int = 0) -> tuple[int, int]:
    f, t = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = load().hb_device_info(int(dev), ctypes.byref(f), ctypes.byref(t))
    raise_for_status(rc, last_error())
    return int(f.value), int(t.value)


def last_error() -> str:
    return (load().hb_last_error() or b"").decode(errors="replace")


def current_device() -> int:
    env = os.environ.get("HARPIA_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# Stage descriptions (Python side of hb_stage)
# ---------------------------------------------------------------------------
@dataclass
class Stage:
    op: int
    precision: int = PREC_FAST
    sigma: float = 0.0
    amount: float = 0.0
    radius: int = 0
    offsets: Optional[np.ndarray] = None   # (n, 3) int32
    weights: Optional[np.ndarray] = None   # float32 taps
    weights64: Optional[np.ndarray] = None  # float64 taps (local_threshold gaussian)

    def halo(self) -> int:
        if self.op in (OP_GAUSSIAN, OP_UNSHARP):
            return (len(self.weights) - 1) // 2
        if self.op in (OP_LOG, OP_HESSIAN):
            return (len(self.weights) - 1) // 2 + 2
        if self.op in (OP_SOBEL, OP_PREWITT):
            return 1
        if self.op in (OP_DIFFUSION, OP_LOCAL_THRESHOLD):
            return int(self.radius)
        if self.op in (OP_MEAN, OP_MEDIAN):
            return int(self.radius)
        if self.op in (OP_ERODE, OP_DILATE):
            return int(np.abs(self.offsets[:, 0]).max())
        return 0

    def out_dtype(self, in_dtype: np.dtype) -> np.dtype:
        if self.op in (OP_GAUSSIAN, OP_UNSHARP, OP_LOG, OP_MEAN, OP_HESSIAN, OP_SOBEL, OP_PREWITT,
                       OP_DIFFUSION):
            return np.dtype("float32")
        if self.op in (OP_THRESHOLD, OP_LOCAL_THRESHOLD):
            return np.dtype("uint32")  # LABEL_DTYPE (volume.py:23)
        if self.op == OP_LBP2D:
            return np.dtype("uint8")
        return np.dtype(in_dtype)


@dataclass
class DeviceProgram:
    """A map operator expressed as a chain of device stages (the unit the
    native executor runs per chunk, replacing ``fn`` at chunking.py:257)."""

    stages: list = field(default_factory=list)

    def halo(self) -> int:
        return int(sum(s.halo() for s in self.stages))

    def out_dtype(self, in_dtype) -> np.dtype:
        dt = np.dtype(in_dtype)
        for s in self.stages:
            dt = s.out_dtype(dt)
        return dt


class _Marshalled:
    """Keeps the ctypes arrays alive for the duration of a native call."""

    def __init__(self, program: DeviceProgram):
        n = len(program.stages)
        self.arr = (HbStage * n)()
        self._keep = []
        for i, s in enumerate(program.stages):
            st = self.arr[i]
            st.op = s.op
            st.precision = s.precision
            st.sigma = float(s.sigma)
            st.amount = float(s.amount)
            st.radius = int(s.radius)
            if s.offsets is not None:
                off = np.ascontiguousarray(s.offsets, dtype=np.int32).reshape(-1, 3)
                self._keep.append(off)
                st.n_offsets = off.shape[0]
                st.offsets = off.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            if s.weights is not None:
                w = np.ascontiguousarray(s.weights, dtype=np.float32)
                self._keep.append(w)
                st.n_weights = w.size
                st.weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            if s.weights64 is not None:
                w = np.ascontiguousarray(s.weights64, dtype=np.float64)
                self._keep.append(w)
                st.n_weights = w.size
                st.weights64 = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self.n = n


def _host_volume(a: np.ndarray) -> HbVolume:
    return HbVolume(a.ctypes.data, DTYPE_CODE[a.dtype], HB_HOST, *a.shape)


@dataclass
class NativeReport:
    chunk_count: int
    chunk_seconds: list
    device_peak_bytes: int
    device_residual_bytes: int
    h2d_bytes: int
    d2h_bytes: int
    kernel_seconds: float
    wall_seconds: float
    kernel_launches: int


def run_host(data: np.ndarray, out: np.ndarray, program: DeviceProgram,
             chunks: Sequence[tuple[int, int, int, int]], *, device: Optional[int] = None,
             cancel: Optional[Callable[[], bool]] = None, device_budget: int = 0,
             pipeline_depth: int = 0, fault_chunk: int = -1,
             host_threads: int = 0, devices: Optional[Sequence[int]] = None) -> NativeReport:
    """hb_run: stream host volume ``data`` through ``program`` chunk by chunk.
    ``devices`` (several ordinals): hb_run_multi, one z-slab group of chunks
    per device, streamed concurrently."""
    L = load()
    if data.dtype not in DTYPE_CODE or out.dtype not in DTYPE_CODE:
        raise UnsupportedFormatError(f"unsupported dtype {data.dtype} -> {out.dtype}")
    if not (data.flags.c_contiguous and out.flags.c_contiguous):
        raise ParameterError("volumes must be C-contiguous (Z, Y, X)")
    m = _Marshalled(program)
    nch = len(chunks)
    carr = (HbChunk * max(nch, 1))()
    for i, c in enumerate(chunks):
        carr[i] = HbChunk(*[int(v) for v in c])
    secs = (ctypes.c_double * max(nch, 1))()
    ex = HbExec()
    ex.device = current_device() if device is None else int(device)
    ex.pipeline_depth = int(pipeline_depth)
    ex.device_budget = int(device_budget)
    ex.fault_chunk = int(fault_chunk)
    ex.host_threads = int(host_threads or os.environ.get("HARPIA_HOST_THREADS", "0"))
    ex.chunk_seconds = ctypes.cast(secs, ctypes.POINTER(ctypes.c_double))
    cb = None
    if cancel is not None:
        def _cb(_ctx):
            try:
                return 1 if cancel() else 0
            except Exception:  # a failing cancel probe cancels the job
                return 1
        cb = CANCEL_FN(_cb)
        ex.cancel = cb
    vin, vout = _host_volume(data), _host_volume(out)
    rep = HbReport()
    if devices is not None and len(devices) > 1:
        devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        rc = L.hb_run_multi(ctypes.byref(vin), ctypes.byref(vout), m.arr, m.n, carr, nch,
                            ctypes.byref(ex), len(devices), devs, ctypes.byref(rep), None)
    else:
        rc = L.hb_run(ctypes.byref(vin), ctypes.byref(vout), m.arr, m.n, carr, nch,
                      ctypes.byref(ex), ctypes.byref(rep))
    if rc != HB_OK:
        raise_for_status(rc, rep.message.decode(errors="replace"),
                         failed_chunk=rep.failed_chunk, minimum_bytes=rep.minimum_bytes)
    return NativeReport(
        chunk_count=int(rep.chunk_count),
        chunk_seconds=[float(secs[i]) for i in range(nch)],
        device_peak_bytes=int(rep.device_peak_bytes),
        device_residual_bytes=int(rep.device_residual_bytes),
        h2d_bytes=int(rep.h2d_bytes),
        d2h_bytes=int(rep.d2h_bytes),
        kernel_seconds=float(rep.kernel_ms) * 1e-3,
        wall_seconds=float(rep.wall_ms) * 1e-3,
        kernel_launches=int(rep.kernel_launches),
    )


def apply_device(inp, out, program: DeviceProgram, z_begin: int = 0, stream=None,
                 synchronize: bool = False) -> int:
    """hb_apply_device on torch CUDA tensors (or anything exposing data_ptr()).

    ``inp``: (Z, Y, X) contiguous CUDA tensor; ``out``: (Zo, Y, X) tensor that
    receives block slices [z_begin, z_begin + Zo).  Returns the number of kernel
    launches enqueued.  Runs on ``stream`` (torch.cuda.Stream or raw handle;
    default: torch's current stream)."""
    import torch

    L = load()
    code_in = DTYPE_CODE.get(np.dtype(str(inp.dtype).replace("torch.", "")))
    code_out = DTYPE_CODE.get(np.dtype(str(out.dtype).replace("torch.", "")))
    if code_in is None or code_out is None:
        raise UnsupportedFormatError(f"unsupported tensor dtype {inp.dtype} -> {out.dtype}")
    if not (inp.is_contiguous() and out.is_contiguous()):
        raise ParameterError("device blocks must be contiguous")
    m = _Marshalled(program)
    vin = HbVolume(inp.data_ptr(), code_in, HB_DEVICE, *inp.shape)
    vout = HbVolume(out.data_ptr(), code_out, HB_DEVICE, *out.shape)
    if stream is None:
        stream = torch.cuda.current_stream(inp.device)
    handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    rep = HbReport()
    rc = L.hb_apply_device(ctypes.byref(vin), ctypes.byref(vout), m.arr, m.n, int(z_begin),
                           ctypes.c_void_p(handle), 1 if synchronize else 0, ctypes.byref(rep))
    if rc != HB_OK:
        raise_for_status(rc, rep.message.decode(errors="replace"),
                         failed_chunk=rep.failed_chunk, minimum_bytes=rep.minimum_bytes)
    return int(rep.kernel_launches)


class DeviceBuffer:
    """A device buffer from the library's private pool (hb_device_alloc),
    exposed to torch through ``__cuda_array_interface__`` so tensors view it
    without PyTorch's caching allocator.  Freed (stream-ordered on ``stream``)
    by :meth:`free` or when garbage-collected."""

    _TYPESTR = {"float32": "<f4", "uint16": "<u2", "uint8": "|u1", "uint32": "<u4",
                "float64": "<f8", "int32": "<i4", "int64": "<i8"}

    def __init__(self, shape, dtype, device: int, stream=None):
        L = load()
        self.shape = tuple(int(v) for v in shape)
        self.dtype = np.dtype(dtype)
        self.device = int(device)
        self.stream = stream
        nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        ptr = ctypes.c_void_p(0)
        rc = L.hb_device_alloc(self.device, nbytes, ctypes.c_void_p(_stream_handle(stream)),
                               ctypes.byref(ptr))
        if rc != HB_OK:
            raise_for_status(rc, last_error(), minimum_bytes=nbytes)
        self.ptr = int(ptr.value or 0)
        self.nbytes = nbytes

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self._TYPESTR[self.dtype.name],
                "data": (self.ptr, False), "version": 3, "strides": None,
                "stream": None}

    def tensor(self):
        """A torch tensor viewing this buffer (keeps the buffer alive)."""
        import torch

        t = torch.as_tensor(self, device=f"cuda:{self.device}")
        t._hb_owner = self  # lifetime: the buffer lives as long as the view
        return t

    def free(self, stream=None):
        if self.ptr:
            load().hb_device_free(self.device, ctypes.c_void_p(self.ptr),
                                  ctypes.c_void_p(_stream_handle(stream if stream is not None
                                                                 else self.stream)))
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _stream_handle(stream) -> int:
    if stream is None:
        try:
            import torch

            return int(torch.cuda.current_stream().cuda_stream)
        except Exception:
            return 0
    return int(stream.cuda_stream if hasattr(stream, "cuda_stream") else stream)


def device_empty(shape, dtype, device: int, stream=None):
    """torch tensor on a library-pool buffer (see :class:`DeviceBuffer`)."""
    return DeviceBuffer(shape, dtype, device, stream).tensor()


def trim_device(dev: Optional[int] = None) -> None:
    load().hb_trim_device(current_device() if dev is None else int(dev))


def device_pool_bytes(dev: Optional[int] = None) -> int:
    return int(load().hb_device_pool_bytes(current_device() if dev is None else int(dev)))


def _volume_of(a):
    """HbVolume view of a C-contiguous numpy array or CUDA torch tensor."""
    if hasattr(a, "data_ptr"):
        dt = np.dtype(str(a.dtype).replace("torch.", ""))
        return HbVolume(a.data_ptr(), DTYPE_CODE[dt], HB_DEVICE, *a.shape), dt
    return HbVolume(a.ctypes.data, DTYPE_CODE[a.dtype], HB_HOST, *a.shape), a.dtype


def minmax(a, dev: Optional[int] = None):
    """Device min/max of a float32 volume (hb_minmax)."""
    L = load()
    vol, _ = _volume_of(a)
    lo, hi = ctypes.c_double(), ctypes.c_double()
    rc = L.hb_minmax(ctypes.byref(vol), current_device() if dev is None else int(dev),
                     ctypes.byref(lo), ctypes.byref(hi))
    raise_for_status(rc, last_error())
    return lo.value, hi.value


def histogram(a, bins: int, lo: float, hi: float, edges: np.ndarray, edges_f32: bool,
              dev: Optional[int] = None) -> np.ndarray:
    """Device np.histogram counts (hb_histogram); int64[bins]."""
    L = load()
    vol, _ = _volume_of(a)
    e = np.ascontiguousarray(edges, dtype=np.float64)
    counts = np.empty(int(bins), np.int64)
    rc = L.hb_histogram(ctypes.byref(vol), current_device() if dev is None else int(dev), int(bins),
                        float(lo), float(hi), e.ctypes.data, 1 if edges_f32 else 0,
                        counts.ctypes.data)
    raise_for_status(rc, last_error())
    return counts


class session:
    """Device-arena session: jobs inside the ``with`` block keep the library's
    device pool mapped between calls (each job still frees every buffer it
    allocated: ``ExecutionReport.device_residual_bytes`` stays 0), and the
    pool is trimmed to zero when the block exits.  Use it around a series of
    ``run_operator`` calls; a single call releases all device memory itself::

        with session(), pinned(volume, out):
            for name, p in steps:
                registry.run_operator(volume, name, p, budget, out=out)
    """

    def __init__(self, dev: Optional[int] = None):
        self.dev = dev

    def __enter__(self):
        L = load()
        self._dev = current_device() if self.dev is None else int(self.dev)
        raise_for_status(L.hb_session_begin(self._dev), last_error())
        return self

    def __exit__(self, *exc):
        load().hb_session_end(self._dev)
        return False


class pinned:
    """Context manager that page-locks numpy arrays (cudaHostRegister) so
    ``run_operator`` DMAs them directly instead of staging through the pinned
    ring.  Registration costs ~0.2 s/GiB on the B200 box, so it pays off when
    the same arrays feed several jobs::

        with pinned(volume, out):
            for name, p in steps:
                registry.run_operator(volume, name, p, budget, out=out)
    """

    def __init__(self, *arrays):
        self.arrays = [a for a in arrays if a is not None]
        self._done = []

    def __enter__(self):
        L = load()
        for a in self.arrays:
            if not a.flags.c_contiguous:
                raise ParameterError("only C-contiguous arrays can be pinned")
            rc = L.hb_pin(a.ctypes.data, a.nbytes)
            raise_for_status(rc, last_error())
            self._done.append(a)
        return self

    def __exit__(self, *exc):
        L = load()
        for a in self._done:
            L.hb_unpin(a.ctypes.data)
        self._done.clear()
        return False
