"""Operator registry — the drop-in boundary (reference registry.py:29-114).

Same entry points (``get_operator``, ``operator_names``, ``validate_params``,
``run_operator``, ``run_direct``) and the same per-operator ``OpProfile``
factories (halo / scratch / out dtype; registry.py:135-191, 234-246,
274-285), so plans, reports and error behaviour match the reference.  What
changes is what a map operator *is*: besides ``fn`` it carries ``program``, a
chain of sm_100a device stages that ``execute_chunked`` runs natively.

Registered here: the hot-path operators named by the north star — identity,
gaussian, mean, median, unsharp, log (new: the Hessian trace), and
morph_{erode,dilate,open,close}.  ``run_pipeline`` chains several of them
into one fused per-chunk device pipeline (e.g. LoG after unsharp).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native, filters, morphology
from .chunking import ExecutionReport, MemoryBudget, OpProfile, execute_chunked, profile_budget
from .errors import ParameterError

REQUIRED = object()
FLOAT32 = np.dtype("float32")
LABEL_DTYPE = np.dtype("uint32")  # volume.py:23


@dataclass(frozen=True)
class Operator:
    name: str
    kind: str                      # "map" (all hot-path operators)
    output: str                    # "volume"
    schema: dict = field(default_factory=dict)      # name -> (caster, default)
    profile: Optional[Callable[[dict], OpProfile]] = None
    fn: Optional[Callable] = None                   # fn(block, params, aux) -> ndarray
    program: Optional[Callable[[dict], _native.DeviceProgram]] = None
    run: Optional[Callable] = None
    aux_keys: tuple = ()
    label_input: bool = False


_REGISTRY: dict = {}


def register(op: Operator) -> Operator:
    if op.name in _REGISTRY:
        raise ValueError(f"duplicate operator {op.name}")
    _REGISTRY[op.name] = op
    return op


def get_operator(name: str) -> Operator:
    if name not in _REGISTRY:
        raise ParameterError(f"unknown operator {name!r}")
    return _REGISTRY[name]


def operator_names() -> list:
    return sorted(_REGISTRY)


def validate_params(op: Operator, raw: dict) -> dict:
    """Cast params by schema, reject unknown keys and missing required ones
    (registry.py:64-79)."""
    extra = sorted(set(raw) - set(op.schema))
    if extra:
        raise ParameterError(f"{op.name}: unknown parameters {extra}")
    params = {}
    for key, (caster, default) in op.schema.items():
        if key not in raw:
            if default is REQUIRED:
                raise ParameterError(f"{op.name}: missing required parameter {key!r}")
            params[key] = default
            continue
        try:
            params[key] = caster(raw[key])
        except ParameterError:
            raise
        except (TypeError, ValueError) as exc:
            raise ParameterError(f"{op.name}: bad value for {key!r}: {exc}") from exc
    return params


def _unvalidated(op: Operator, raw: dict) -> dict:
    """``validate=False`` (the service's job path, service.py:131-139): take
    the caller's values as given, but fill the schema defaults the reference
    schema does not have (e.g. ``precision``) so the profile/program see them."""
    params = {k: d for k, (_c, d) in op.schema.items() if d is not REQUIRED and k not in raw}
    params.update(raw)
    return params


def _program_for(op: Operator, params: dict) -> _native.DeviceProgram:
    try:
        return op.program(params)
    except ParameterError:
        raise
    except KeyError as exc:  # unvalidated params missing a required key
        raise ParameterError(f"{op.name}: missing required parameter {exc.args[0]!r}") from exc
    except (TypeError, ValueError) as exc:
        raise ParameterError(f"{op.name}: bad parameters: {exc}") from exc


def _profile_for(op: Operator, params: dict) -> OpProfile:
    try:
        return op.profile(params)
    except KeyError as exc:
        raise ParameterError(f"{op.name}: missing required parameter {exc.args[0]!r}") from exc


def run_operator(
    data: np.ndarray,
    name: str,
    params: Optional[dict] = None,
    budget: Optional[MemoryBudget] = None,
    aux: Optional[dict] = None,
    cancel=None,
    validate: bool = True,
    **exec_kw,
) -> tuple:
    """Uniform entry point (registry.py:82-103): plan with the operator's
    profile against ``budget`` (default: 80% of free device memory) and stream
    the volume through the operator's device program chunk by chunk."""
    op = get_operator(name)
    params = validate_params(op, params or {}) if validate else _unvalidated(op, params or {})
    if budget is None:
        budget = profile_budget()
    if op.kind == "global":  # registry.py:99-103: global operators run themselves
        return op.run(data, params, budget, cancel)
    program = _program_for(op, params)
    arr, restore = filters.coerce_input(data, program)
    out, report = execute_chunked(arr, program, _profile_for(op, params), budget, params,
                                  aux=aux, cancel=cancel, **exec_kw)
    return (restore(out) if restore else out), report


def run_direct(data: np.ndarray, name: str, params: Optional[dict] = None, aux=None):
    """Whole-volume single-shot evaluation (registry.py:106-114)."""
    op = get_operator(name)
    params = validate_params(op, params or {})
    if op.kind == "global":
        result, _ = op.run(data, params, None, None)
        return result
    return op.fn(data, params, aux or {})


def run_pipeline(data: np.ndarray, steps, budget: Optional[MemoryBudget] = None, cancel=None,
                 **exec_kw) -> tuple:
    """Chain registry map operators into ONE device pipeline per chunk.

    ``steps`` = [(name, params), ...].  The chunk halo is the sum of the
    operators' halos, the scratch factor the largest one; the result equals
    applying the operators one after another with ``run_operator``."""
    progs, halo, scratch = [], 0, 2.0
    for name, p in steps:
        op = get_operator(name)
        params = validate_params(op, p or {})
        prof = op.profile(params)
        progs.append(_program_for(op, params))
        halo += prof.halo_z
        scratch = max(scratch, prof.scratch_factor)
    program = filters.chain(*progs)
    if budget is None:
        budget = profile_budget()
    arr, restore = filters.coerce_input(data, program)
    out, report = execute_chunked(arr, program, OpProfile(halo_z=halo, scratch_factor=scratch),
                                  budget, cancel=cancel, **exec_kw)
    return (restore(out) if restore else out), report


# ---------------------------------------------------------------------------
# map operators
# ---------------------------------------------------------------------------
def _se_param(value):
    if isinstance(value, morphology.StructuringElement):
        return value
    return morphology.StructuringElement.parse(str(value))


def _precision_param(value):
    filters._precision(value)
    return str(value) if not isinstance(value, int) else ("fast", "exact")[value]


def _direct(program_of):
    return lambda b, p, a: filters.apply_program(b, program_of(p))


def _map(name, schema, profile, program_of, output="volume"):
    register(Operator(name=name, kind="map", output=output, schema=schema, profile=profile,
                      fn=_direct(program_of), program=program_of))


_map("identity", {}, lambda p: OpProfile(halo_z=0, scratch_factor=2),
     lambda p: filters.identity_program())

_map("gaussian",
     {"sigma": (float, REQUIRED), "precision": (_precision_param, "fast")},
     lambda p: OpProfile(halo_z=filters.gaussian_kernel_radius(p["sigma"]), scratch_factor=8,
                         out_dtype=FLOAT32),
     lambda p: filters.gaussian_program(p["sigma"], p["precision"]))

_map("mean", {"radius": (int, REQUIRED)},
     lambda p: OpProfile(halo_z=p["radius"], scratch_factor=12, out_dtype=FLOAT32),
     lambda p: filters.mean_program(p["radius"]))

_map("median", {"radius": (int, REQUIRED)},
     lambda p: OpProfile(halo_z=p["radius"], scratch_factor=4),
     lambda p: filters.median_program(p["radius"]))

_map("unsharp",
     {"sigma": (float, REQUIRED), "amount": (float, REQUIRED),
      "precision": (_precision_param, "fast")},
     lambda p: OpProfile(halo_z=filters.gaussian_kernel_radius(p["sigma"]), scratch_factor=10,
                         out_dtype=FLOAT32),
     lambda p: filters.unsharp_program(p["sigma"], p["amount"], p["precision"]))

# hessian_* (registry.py:234-246), sobel / prewitt
# (registry.py:210-224), apply_threshold (registry.py:248-255) on the device
for _comp in filters.HESSIAN_COMPONENTS:
    _map(f"hessian_{_comp}",
         {"sigma": (float, REQUIRED), "precision": (_precision_param, "exact")},
         lambda p: OpProfile(halo_z=filters.gaussian_kernel_radius(p["sigma"]) + 2,
                             scratch_factor=10, out_dtype=FLOAT32),
         (lambda comp: lambda p: filters.hessian_program(p["sigma"], comp, p["precision"]))(_comp))

_map("sobel", {}, lambda p: OpProfile(halo_z=1, scratch_factor=12, out_dtype=FLOAT32),
     lambda p: filters.sobel_program())
_map("prewitt", {}, lambda p: OpProfile(halo_z=1, scratch_factor=12, out_dtype=FLOAT32),
     lambda p: filters.prewitt_program())
_map("anisotropic_diffusion",
     {"iterations": (int, REQUIRED), "kappa": (float, REQUIRED), "dt": (float, 1.0 / 6.0),
      "mode": (str, "exponential")},
     lambda p: OpProfile(halo_z=p["iterations"], scratch_factor=12, out_dtype=FLOAT32),
     lambda p: filters.diffusion_program(p["iterations"], p["kappa"], p["dt"], p["mode"]))
_map("lbp2d", {}, lambda p: OpProfile(halo_z=0, scratch_factor=4, out_dtype=np.dtype("uint8")),
     lambda p: filters.lbp2d_program())
_map("local_threshold",
     {"kind": (str, REQUIRED), "window": (int, REQUIRED), "k": (float, 0.2),
      "R": (lambda v: None if v is None else float(v), None), "c": (float, 0.0)},
     lambda p: OpProfile(halo_z=p["window"], scratch_factor=24, out_dtype=LABEL_DTYPE),
     lambda p: filters.local_threshold_program(p["kind"], p["window"], p["k"], p["R"], p["c"]),
     output="labels")
_map("apply_threshold", {"t": (float, REQUIRED)},
     lambda p: OpProfile(halo_z=0, scratch_factor=6, out_dtype=LABEL_DTYPE),
     lambda p: filters.threshold_program(p["t"]), output="labels")

# global Otsu (registry.py:312-334): two passes, device histogram + apply
def _run_otsu(data, params, budget, cancel):
    from . import threshold
    from .ledger import LEDGER

    LEDGER.job_start()
    out, t = threshold.otsu_binarize(data, params.get("bins", 256), budget, cancel=cancel)
    report = ExecutionReport(chunk_count=1)
    if budget is not None:
        snap = LEDGER.snapshot()
        report.peak_bytes = snap.peak_bytes - snap.baseline_bytes
        report.residual_bytes = snap.residual_bytes
    report.threshold = t
    return out, report


register(Operator(name="otsu", kind="global", output="labels", schema={"bins": (int, 256)},
                  run=_run_otsu))


# connected components (registry.py:337-351) on the device
def _run_cc(data, params, budget, cancel):
    from . import quantify
    from .ledger import LEDGER

    LEDGER.job_start()
    labels, count = quantify.connected_components(data, params["connectivity"], budget)
    report = ExecutionReport(chunk_count=1)
    report.component_count = count
    return labels, report


register(Operator(name="connected_components", kind="global", output="labels",
                  schema={"connectivity": (int, 6)}, run=_run_cc))


# label-volume filters (registry.py:355-383) on the device labelling
def _run_fill_holes(data, params, budget, cancel):
    from .ledger import LEDGER

    LEDGER.job_start()
    return morphology.fill_holes(data, params["connectivity"]), ExecutionReport(chunk_count=1)


def _run_remove_islands(data, params, budget, cancel):
    from .ledger import LEDGER

    LEDGER.job_start()
    out = morphology.remove_islands(data, params["min_size"], params["connectivity"])
    return out, ExecutionReport(chunk_count=1)


def _run_geodesic(data, params, budget, cancel):
    from .ledger import LEDGER

    LEDGER.job_start()
    # whole-volume fixed point: the propagation range is unbounded (no halo)
    out = morphology.geodesic_reconstruct(params["marker"], data, params["kind"])
    return out, ExecutionReport(chunk_count=1)


def _run_edt(data, params, budget, cancel):
    from . import quantify
    from .ledger import LEDGER

    LEDGER.job_start()
    out = quantify.edt(data, params.get("spacing") or (1.0, 1.0, 1.0))
    return out, ExecutionReport(chunk_count=1)


register(Operator(name="edt", kind="global", output="volume",
                  schema={"spacing": (lambda v: tuple(float(s) for s in v), None)},
                  run=_run_edt, label_input=True))
register(Operator(name="geodesic_reconstruct", kind="global", output="volume",
                  schema={"marker": (np.asarray, REQUIRED), "kind": (str, "dilation")},
                  run=_run_geodesic, label_input=True))
register(Operator(name="fill_holes", kind="global", output="labels",
                  schema={"connectivity": (int, 6)}, run=_run_fill_holes, label_input=True))
register(Operator(name="remove_islands", kind="global", output="labels",
                  schema={"min_size": (int, REQUIRED), "connectivity": (int, 6)},
                  run=_run_remove_islands, label_input=True))

# LoG = hessian trace; profile as the reference's hessian_* (registry.py:234-246)
_map("log",
     {"sigma": (float, REQUIRED), "precision": (_precision_param, "exact")},
     lambda p: OpProfile(halo_z=filters.gaussian_kernel_radius(p["sigma"]) + 2,
                         scratch_factor=10, out_dtype=FLOAT32),
     lambda p: filters.log_program(p["sigma"], p["precision"]))

for _mop in morphology.MORPH_OPS:
    _map(f"morph_{_mop}",
         {"se": (_se_param, REQUIRED), "iterations": (int, 1)},
         (lambda mop: lambda p: OpProfile(
             halo_z=p["se"].z_extent * p["iterations"] * (2 if mop in ("open", "close") else 1),
             scratch_factor=8))(_mop),
         (lambda mop: lambda p: morphology.morph_program(mop, p["se"], p["iterations"]))(_mop))
