"""The reference's two consumers of the hot path, replayed through the drop-in
on the B200.

* service worker: ``HarpiaService._run_job`` (reference service.py:120-166) —
  a worker thread calls ``run_operator(source, op, params, budget, aux=...,
  cancel=lambda: job.cancel_requested, validate=False)`` with the ledger
  bracketing (``LEDGER.job_start`` / ``commit_persistent`` / ``snapshot``), and
  maps JobCancelled -> "cancelled", HarpiaError -> "failed".
* CLI: ``_run_one`` (reference cli.py:38-59) — ``get_operator`` +
  ``validate_params``, ``load_volume``, ``plan_chunks(...).dump()``,
  ``run_operator(..., validate=False)``, ``save_volume``, and the report echo.

The reference itself is not imported (it does not travel to the GPU box);
the call sequences are restated here with their citations, and every output
is checked against the CPU oracle (test infrastructure).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Job:
    def __init__(self, op, params, target="volume"):
        self.op, self.params, self.target = op, params, target
        self.state, self.error, self.report = "queued", None, None
        self.cancel_requested = False


def _submit(op_name, raw_params):
    """service.py:303-309, restated: parameters are validated (and the plan
    profile checked) at submit; a ParameterError is the 422 response."""
    from paper_2511_11890_b200.registry import get_operator, validate_params

    op = get_operator(op_name)
    params = validate_params(op, raw_params or {})
    if op.kind == "map":
        op.profile(params)
    return _Job(op_name, params)


def _run_job(job, source, budget_fraction=0.8):
    """service.py:120-166, restated: same calls, same state mapping."""
    from paper_2511_11890_b200 import (LEDGER, HarpiaError, JobCancelled, get_operator,
                                       profile_budget, run_operator)

    job.state = "running"
    baseline = LEDGER.job_start()
    try:
        op = get_operator(job.op)
        aux = {}
        if "markers" in op.aux_keys:
            aux["markers"] = source
        budget = profile_budget(fraction=budget_fraction)
        result, report = run_operator(source, job.op, job.params, budget, aux=aux,
                                      cancel=lambda: job.cancel_requested, validate=False)
        LEDGER.commit_persistent(result.nbytes - source.nbytes)
        snap = LEDGER.snapshot()
        job.report = {"chunk_count": report.chunk_count, "wall_seconds": report.wall_seconds,
                      "peak_bytes": report.peak_bytes, "residual_bytes": snap.residual_bytes,
                      "baseline_bytes": baseline,
                      "device_residual_bytes": report.device_residual_bytes}
        job.result = result
        job.state = "done"
    except JobCancelled:
        job.state = "cancelled"
    except HarpiaError as exc:
        job.state = "failed"
        job.error = str(exc)


def test_service_worker_jobs(oracle):
    """Jobs on a worker thread (as the service's worker pool runs them):
    done with oracle-exact results and a zero device residual, a cancelled
    job, 422-style rejections at submit and a failed job."""
    rng = np.random.default_rng(7)
    vol = rng.random((40, 96, 128), dtype=np.float32)
    u16 = rng.integers(0, 65536, size=(24, 64, 96), dtype=np.uint16)
    jobs = [(_submit("median", {"radius": 1}), vol, lambda: oracle.median(vol, 1), True),
            (_submit("gaussian", {"sigma": "2"}), vol, lambda: oracle.gaussian(vol, 2.0), False),
            (_submit("morph_erode", {"se": "ball:3"}), u16, None, True)]
    for job, src, ref, exact in jobs:
        t = threading.Thread(target=_run_job, args=(job, src), name="harpia-worker-0")
        t.start()
        t.join()
        assert job.state == "done", (job.op, job.error)
        assert job.report["chunk_count"] >= 1 and job.report["device_residual_bytes"] == 0
        if ref is not None:
            r = ref()
            if exact:
                assert np.array_equal(job.result, r)
            else:
                assert np.max(np.abs(job.result - r)) / np.max(np.abs(r)) <= 1e-5
    from paper_2511_11890_b200 import morphology

    se = morphology.StructuringElement.parse("ball:3")
    assert np.array_equal(jobs[2][0].result, oracle.erode(u16, se.offsets))

    # cancellation requested before the first chunk -> "cancelled"
    job = _submit("median", {"radius": 1})
    job.cancel_requested = True
    _run_job(job, vol)
    assert job.state == "cancelled"

    # bad parameters never reach a worker: 422 at submit (the same three the
    # reference rejects there)
    from paper_2511_11890_b200 import ParameterError

    for op_name, raw in (("median", {"radius": -1}), ("morph_erode", {"se": "ball:x"}),
                         ("median", {"bogus": 1})):
        with pytest.raises(ParameterError):
            _submit(op_name, raw)
    # sigma = 0 passes submit (as in the reference) and the operator's own
    # check fails the job: HarpiaError -> "failed"
    job = _submit("gaussian", {"sigma": 0})
    _run_job(job, vol)
    assert job.state == "failed" and "sigma" in job.error


def test_cli_run_one_roundtrip(tmp_path, oracle):
    """cli.py:38-59 restated: validate, load the .vol, dump the plan, run with
    validate=False, save the .vol, echo the report — on raw files."""
    # the CLI's own imports (cli.py:14-21): chunking / registry / volume modules
    from paper_2511_11890_b200.chunking import MemoryBudget, plan_chunks
    from paper_2511_11890_b200.registry import get_operator, run_operator, validate_params
    from paper_2511_11890_b200.volume import Volume, load_volume, save_volume

    rng = np.random.default_rng(11)
    data = rng.random((30, 80, 96), dtype=np.float32)
    src = tmp_path / "in.vol"
    dst = tmp_path / "out.vol"
    save_volume(Volume(data, spacing=(1.0, 0.5, 0.5)), str(src))
    op = get_operator("unsharp")
    params = validate_params(op, {"sigma": "1.0", "amount": "1.5"})
    volume = load_volume(str(src))
    prof = op.profile(params)
    budget = MemoryBudget(int(12 * prof.scratch_factor * 80 * 96 * 4), 1.0)
    plan = plan_chunks(volume.shape, volume.dtype, prof, budget)
    text = plan.dump()
    assert "chunk" in text.lower() and plan.chunks and len(plan.chunks) >= 3
    result, report = run_operator(volume.data, "unsharp", params, budget, validate=False)
    save_volume(Volume(result.astype(np.float32), spacing=volume.spacing), str(dst))
    line = (f"unsharp: {report.chunk_count} chunks, {report.wall_seconds:.3f}s, "
            f"peak {report.peak_bytes} B, residual {report.residual_bytes} B")
    assert report.chunk_count == len(plan.chunks) and "residual 0 B" in line
    back = load_volume(str(dst))
    ref = oracle.unsharp(data, 1.0, 1.5)
    assert back.spacing == volume.spacing
    assert np.max(np.abs(np.asarray(back.data) - ref)) / np.max(np.abs(ref)) <= 1e-5
