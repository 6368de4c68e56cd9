"""Smoothing filters on the device (reference filters.py:21-82, 136-139, 234-264).

Same call signatures as the reference: ``gaussian(data, sigma)``,
``mean(data, radius)``, ``median(data, radius)``, ``unsharp(data, sigma,
amount)``, plus the Laplacian of Gaussian ``log(data, sigma)`` defined as the
Hessian trace ``hessian_xx + hessian_yy + hessian_zz`` of the reference
(filters.py:246-264), evaluated as ``(xx + yy) + zz`` in float32.

Inputs may be numpy arrays (host; streamed through the chunked executor when
they exceed the device budget) or CUDA torch tensors (device-resident; one
``hb_apply_device`` call on the caller's current stream).  Output dtypes follow
the reference: gaussian/mean/unsharp/log -> float32, median keeps the dtype.

``precision``: "fast" accumulates in fp32 (within 1e-5 of the reference);
"exact" evaluates each Gaussian pass in fp64 with scipy's fold order and a
float32 round per pass, which reproduces the reference bit for bit.  LoG
defaults to "exact" because its second differences cancel catastrophically.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .errors import ParameterError, UnsupportedFormatError

_PRECISION = {"fast": _native.PREC_FAST, "exact": _native.PREC_EXACT}


def gaussian_kernel_radius(sigma: float) -> int:
    """Truncation radius ceil(4 sigma) (filters.py:21-23)."""
    return int(math.ceil(4.0 * sigma))


def _gaussian_kernel(sigma: float) -> np.ndarray:
    """float32 taps exactly as the reference builds them (filters.py:26-30):
    float64 exp over [-r, r], numpy-sum normalisation, then a float32 cast."""
    r = gaussian_kernel_radius(sigma)
    x = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return (k / k.sum()).astype(np.float32)


def _precision(p) -> int:
    if isinstance(p, int) and p in (0, 1):
        return p
    try:
        return _PRECISION[str(p)]
    except KeyError:
        raise ParameterError(f"precision must be 'fast' or 'exact', got {p!r}") from None


def _check_sigma(sigma):
    if not sigma > 0:
        raise ParameterError(f"sigma must be positive, got {sigma}")


def _check_radius(radius):
    if radius < 1:
        raise ParameterError(f"radius must be >= 1, got {radius}")


# ---------------------------------------------------------------------------
# programs (one DeviceProgram per reference operator)
# ---------------------------------------------------------------------------
def gaussian_program(sigma, precision="fast") -> _native.DeviceProgram:
    _check_sigma(sigma)
    return _native.DeviceProgram([_native.Stage(
        _native.OP_GAUSSIAN, precision=_precision(precision), sigma=float(sigma),
        weights=_gaussian_kernel(sigma))])


def mean_program(radius) -> _native.DeviceProgram:
    _check_radius(radius)
    return _native.DeviceProgram([_native.Stage(_native.OP_MEAN, radius=int(radius))])


def median_program(radius) -> _native.DeviceProgram:
    _check_radius(radius)
    return _native.DeviceProgram([_native.Stage(_native.OP_MEDIAN, radius=int(radius))])


def unsharp_program(sigma, amount, precision="fast") -> _native.DeviceProgram:
    _check_sigma(sigma)
    return _native.DeviceProgram([_native.Stage(
        _native.OP_UNSHARP, precision=_precision(precision), sigma=float(sigma),
        amount=float(amount), weights=_gaussian_kernel(sigma))])


def log_program(sigma, precision="exact") -> _native.DeviceProgram:
    _check_sigma(sigma)
    return _native.DeviceProgram([_native.Stage(
        _native.OP_LOG, precision=_precision(precision), sigma=float(sigma),
        weights=_gaussian_kernel(sigma))])


HESSIAN_COMPONENTS = ("xx", "yy", "zz", "xy", "xz", "yz")  # filters.py:228


def hessian_program(sigma, component, precision="exact") -> _native.DeviceProgram:
    _check_sigma(sigma)
    if component not in HESSIAN_COMPONENTS:
        raise ParameterError(f"component must be one of {HESSIAN_COMPONENTS}, got {component!r}")
    return _native.DeviceProgram([_native.Stage(
        _native.OP_HESSIAN, precision=_precision(precision), sigma=float(sigma),
        radius=HESSIAN_COMPONENTS.index(component), weights=_gaussian_kernel(sigma))])


def sobel_program() -> _native.DeviceProgram:
    return _native.DeviceProgram([_native.Stage(_native.OP_SOBEL)])


def prewitt_program() -> _native.DeviceProgram:
    return _native.DeviceProgram([_native.Stage(_native.OP_PREWITT)])


DIFFUSION_MODES = ("exponential", "rational")  # filters.py:17


def diffusion_program(iterations, kappa, dt=1.0 / 6.0, mode="exponential") -> _native.DeviceProgram:
    # filters.py:152-159 validation, same messages
    if iterations < 1:
        raise ParameterError(f"iterations must be >= 1, got {iterations}")
    if not 0 < dt <= 1.0 / 6.0 + 1e-12:
        raise ParameterError(f"dt must be in (0, 1/6], got {dt}")
    if kappa <= 0:
        raise ParameterError(f"kappa must be positive, got {kappa}")
    if mode not in DIFFUSION_MODES:
        raise ParameterError(f"mode must be one of {DIFFUSION_MODES}, got {mode!r}")
    return _native.DeviceProgram([_native.Stage(
        _native.OP_DIFFUSION, radius=int(iterations), sigma=float(kappa), amount=float(dt),
        precision=DIFFUSION_MODES.index(mode))])


def lbp2d_program() -> _native.DeviceProgram:
    return _native.DeviceProgram([_native.Stage(_native.OP_LBP2D)])


def local_gaussian_kernel(window: int) -> np.ndarray:
    """threshold.py:199-202: exp(-x^2 / (2 (w/2)^2)) over -w..w, normalised
    (NumPy's own exp and pairwise sum, so the taps are the reference's)."""
    sigma = window / 2.0
    x = np.arange(-window, window + 1, dtype=np.float64)
    kern = np.exp(-0.5 * (x / sigma) ** 2)
    kern /= kern.sum()
    return kern


def local_threshold_program(kind, window, k=0.2, r=None, c=0.0, dtype=None) -> _native.DeviceProgram:
    """threshold.local_threshold (threshold.py:174-217) as one device stage;
    ``r`` None = default_sauvola_r(dtype) (threshold.py:166-171)."""
    if kind not in _native.LOCAL_KINDS:
        raise ParameterError(f"kind must be one of {_native.LOCAL_KINDS}, got {kind!r}")
    if window < 1:
        raise ParameterError(f"window radius must be >= 1, got {window}")
    w = int(window)
    amount = float(c)
    if kind == "sauvola":
        if r is None and dtype is not None:
            from .threshold import default_sauvola_r

            r = default_sauvola_r(dtype)
        if r is not None and r <= 0:
            raise ParameterError(f"sauvola R must be positive, got {r}")
        # NaN = default_sauvola_r of the stage's input dtype, resolved by the library
        amount = float("nan") if r is None else float(r)
    return _native.DeviceProgram([_native.Stage(
        _native.OP_LOCAL_THRESHOLD, precision=_native.LOCAL_KINDS.index(kind), radius=w,
        sigma=float(k), amount=amount,
        weights64=local_gaussian_kernel(w) if kind == "gaussian" else None)])


def threshold_program(t) -> _native.DeviceProgram:
    return _native.DeviceProgram([_native.Stage(_native.OP_THRESHOLD, amount=float(t))])


def identity_program() -> _native.DeviceProgram:
    return _native.DeviceProgram([_native.Stage(_native.OP_IDENTITY)])


def chain(*programs: _native.DeviceProgram) -> _native.DeviceProgram:
    """Fuse programs into one per-chunk pipeline (halos add up)."""
    return _native.DeviceProgram([s for p in programs for s in p.stages])


# ---------------------------------------------------------------------------
# dtype handling
# ---------------------------------------------------------------------------
def _selects_values(program) -> bool:
    """True when every stage outputs samples of its input (median/morph/identity)."""
    return all(s.op in (_native.OP_MEDIAN, _native.OP_ERODE, _native.OP_DILATE,
                        _native.OP_IDENTITY) for s in program.stages)


def coerce_input(data: np.ndarray, program):
    """Map ``data`` onto a device dtype; returns (array, restore_fn).

    float-output programs convert like the reference's first step
    (``astype(float32)``).  Order-statistic programs map signed integers to
    unsigned with an order-preserving offset and bool to uint8, so their
    results stay bit-exact after the inverse map."""
    a = np.asarray(data)
    if a.ndim != 3:
        raise ParameterError(f"expected a 3D (Z, Y, X) volume, got shape {a.shape}")
    dt = a.dtype
    if dt in _native.DTYPE_CODE:
        return np.ascontiguousarray(a), None
    if not _selects_values(program):
        return np.ascontiguousarray(a, dtype=np.float32), None
    if dt == np.bool_:
        return np.ascontiguousarray(a, dtype=np.uint8), lambda r: r.astype(np.bool_)
    if dt.kind == "i" and dt.itemsize <= 4:
        udt = np.dtype(f"uint{dt.itemsize * 8}")
        flip = np.array(1 << (dt.itemsize * 8 - 1), dtype=udt)
        up = np.ascontiguousarray(a.view(udt) ^ flip)
        if udt == np.uint8 or udt == np.uint16 or udt == np.uint32:
            return up, lambda r: (r ^ flip).view(dt)
    if dt == np.float16:
        return np.ascontiguousarray(a, dtype=np.float32), lambda r: r.astype(np.float16)
    raise UnsupportedFormatError(f"dtype {dt} is not supported by the device operators")


# ---------------------------------------------------------------------------
# execution
# ---------------------------------------------------------------------------
def _is_torch_cuda(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _device_scratch_factor(program, in_itemsize: int) -> float:
    # bytes per input voxel the device needs per padded slice: input + every
    # stage output + one f32 temporary; double-buffered by the executor.
    per = in_itemsize + 4 * (len(program.stages) + 1)
    return max(2.0, 2.0 * per / in_itemsize)


def apply_program(data, program: _native.DeviceProgram, *, budget=None, cancel=None):
    """Evaluate ``program`` over the whole volume (the reference's fn(block))."""
    if _is_torch_cuda(data):
        import torch

        x = data.contiguous()
        out_dt = program.out_dtype(np.dtype(str(x.dtype).replace("torch.", "")))
        out = torch.empty(tuple(x.shape), dtype=getattr(torch, out_dt.name), device=x.device)
        _native.apply_device(x, out, program, 0)
        return out
    from .chunking import OpProfile, execute_chunked, plan_chunks, profile_budget

    a, restore = coerce_input(data, program)
    if budget is None:
        budget = profile_budget()
    prof = OpProfile(halo_z=program.halo(),
                     scratch_factor=_device_scratch_factor(program, a.dtype.itemsize))
    plan = plan_chunks(a.shape, a.dtype, prof, budget)
    out, _ = execute_chunked(a, program, prof, budget, plan=plan, cancel=cancel, fresh_job=False)
    return restore(out) if restore else out


def gaussian(data, sigma, precision="fast"):
    """Separable 3D Gaussian truncated at ceil(4 sigma) (filters.py:33-41)."""
    return apply_program(data, gaussian_program(sigma, precision))


def mean(data, radius):
    """Mean over the clamped (2r+1)^3 window, float32 output (filters.py:66-75)."""
    return apply_program(data, mean_program(radius))


def median(data, radius):
    """Median of the clamped (2r+1)^3 window; dtype preserved (filters.py:78-82)."""
    return apply_program(data, median_program(radius))


def unsharp(data, sigma, amount, precision="fast"):
    """I + amount * (I - gaussian(I, sigma)) (filters.py:136-139)."""
    return apply_program(data, unsharp_program(sigma, amount, precision))


def log(data, sigma, precision="exact"):
    """Laplacian of Gaussian = hessian_xx + hessian_yy + hessian_zz (filters.py:246-264)."""
    return apply_program(data, log_program(sigma, precision))


def hessian_component(data, sigma, component, precision="exact"):
    """One second-derivative component cd_b(cd_a(gaussian(data, sigma)))
    (filters.py:246-253); bit-exact with the default exact smoothing."""
    return apply_program(data, hessian_program(sigma, component, precision))


def hessian(data, sigma, precision="exact"):
    """All six Hessian components (filters.py:256-264)."""
    return {c: hessian_component(data, sigma, c, precision) for c in HESSIAN_COMPONENTS}


def sobel(data):
    """3D gradient magnitude with [1,2,1] cross-axis smoothing (filters.py:200-202)."""
    return apply_program(data, sobel_program())


def anisotropic_diffusion(data, iterations, kappa, dt=1.0 / 6.0, mode="exponential"):
    """Perona-Malik diffusion over the 6 axial neighbours (filters.py:142-184).
    "rational" is bit-exact; "exponential" follows CUDA expf (<= 2 ulp per exp
    from NumPy's float32 exp, which is itself a SIMD approximation)."""
    return apply_program(data, diffusion_program(iterations, kappa, dt, mode))


def lbp2d(data):
    """Per-Z-slice 8-neighbour local binary pattern, uint8 (filters.py:213-227)."""
    return apply_program(data, lbp2d_program())


def prewitt(data):
    """3D gradient magnitude with [1,1,1] cross-axis smoothing (filters.py:205-207)."""
    return apply_program(data, prewitt_program())
