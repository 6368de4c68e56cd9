"""Host-side logic of the drop-in that needs no GPU: budgets, chunk planning,
registry validation/profiles, structuring elements, error mapping, dtype
coercion and the Python-callable engine (reference test_chunking.py,
test_morphology.py structure)."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2511_11890_b200 import _native, errors, filters, registry
from paper_2511_11890_b200.chunking import (
    MemoryBudget, OpProfile, execute_chunked, plan_chunks, profile_budget)
from paper_2511_11890_b200.errors import (
    BudgetTooSmallError, ChunkExecutionError, JobCancelled, ParameterError)
from paper_2511_11890_b200.ledger import LEDGER, MemoryLedger
from paper_2511_11890_b200.morphology import StructuringElement, morph_program

MIB = 1 << 20


class TestBudget:
    def test_usable_fraction(self):
        assert MemoryBudget(1000 * MIB, 0.8).usable_bytes == 800 * MIB

    def test_identity_fraction(self):
        assert MemoryBudget(12345, 1.0).usable_bytes == 12345

    def test_bad_fraction(self):
        for f in (0.0, 1.5, -1):
            with pytest.raises(ParameterError):
                MemoryBudget(100, f)
        with pytest.raises(ParameterError):
            MemoryBudget(0, 0.5)

    def test_explicit_free(self):
        assert profile_budget(1000, 0.5).usable_bytes == 500


class TestPlan:
    def test_worked_example(self):
        # reference test_chunking.py:47-59
        plan = plan_chunks((100, 1024, 1024), np.uint32, OpProfile(halo_z=2, scratch_factor=3),
                           MemoryBudget(96 * MIB, 1.0))
        assert plan.slice_bytes == 4 * MIB and plan.interior_slices == 4
        assert len(plan.chunks) == 25

    def test_plans_match_reference_dump(self, golden):
        meta, _ = golden
        for p in meta["plans"]:
            if "error" in p:
                with pytest.raises(BudgetTooSmallError) as e:
                    plan_chunks((100, 1024, 1024), np.uint32, OpProfile(2, 3),
                                MemoryBudget(20 * MIB, 1.0))
                assert str(e.value) == p["error"]
                assert e.value.minimum_bytes == p["minimum_bytes"]
                continue
            dt = {1: np.uint8, 4: np.float32}[p["itemsize"]]
            plan = plan_chunks(tuple(p["shape"]), dt, OpProfile(p["halo"], p["scratch"]),
                               MemoryBudget(p["usable"], 1.0))
            assert plan.dump() == p["dump"]
            assert plan.working_peak_bytes == p["working_peak"]

    @given(z=st.integers(1, 200), halo=st.integers(0, 4), interior=st.integers(1, 50))
    @settings(max_examples=100, deadline=None)
    def test_interiors_partition(self, z, halo, interior):
        t = interior + 2 * halo
        budget = MemoryBudget(int(t * 3 * 256), 1.0)
        plan = plan_chunks((z, 16, 16), np.uint8, OpProfile(halo_z=halo, scratch_factor=3), budget)
        covered = []
        for c in plan.chunks:
            assert 0 <= c.padded_start <= c.z_start < c.z_stop <= c.padded_stop <= z
            assert c.halo_lo <= halo and c.halo_hi <= halo
            covered.extend(range(c.z_start, c.z_stop))
        assert covered == list(range(z))


class TestRegistry:
    def test_names(self):
        assert set(registry.operator_names()) == {
            "identity", "gaussian", "mean", "median", "unsharp", "log",
            "morph_erode", "morph_dilate", "morph_open", "morph_close",
            # SURVEY.md §8(f) row 2
            "hessian_xx", "hessian_yy", "hessian_zz", "hessian_xy", "hessian_xz", "hessian_yz",
            "sobel", "prewitt", "apply_threshold", "local_threshold", "lbp2d", "anisotropic_diffusion", "otsu",
            "connected_components", "fill_holes", "remove_islands", "geodesic_reconstruct",
            "edt"}

    def test_profiles_match_reference(self, golden):
        meta, _ = golden
        for name, want in meta["profiles"].items():
            ours = name
            op = registry.get_operator(ours)
            pr = op.profile(registry.validate_params(op, want["params"]))
            assert pr.halo_z == want["halo_z"], name
            assert pr.scratch_factor == want["scratch"], name
            got_dt = None if pr.out_dtype is None else str(pr.out_dtype)
            assert got_dt == want["out_dtype"], name

    def test_validation(self):
        op = registry.get_operator("gaussian")
        with pytest.raises(ParameterError):
            registry.validate_params(op, {})
        with pytest.raises(ParameterError):
            registry.validate_params(op, {"sigma": 1, "bogus": 2})
        with pytest.raises(ParameterError):
            registry.validate_params(op, {"sigma": "abc"})
        with pytest.raises(ParameterError):
            registry.validate_params(op, {"sigma": 1, "precision": "half"})
        with pytest.raises(ParameterError):
            registry.get_operator("nope")
        p = registry.validate_params(op, {"sigma": "2"})
        assert p == {"sigma": 2.0, "precision": "fast"}

    def test_programs(self):
        op = registry.get_operator("morph_close")
        p = registry.validate_params(op, {"se": "ball:3", "iterations": 2})
        prog = op.program(p)
        assert [s.op for s in prog.stages] == [_native.OP_DILATE, _native.OP_ERODE] * 2
        assert prog.halo() == op.profile(p).halo_z == 12
        g = registry.get_operator("log")
        gp = g.program(registry.validate_params(g, {"sigma": 2.0}))
        assert gp.halo() == 10 and gp.stages[0].precision == _native.PREC_EXACT
        with pytest.raises(ParameterError):
            registry.get_operator("morph_open").program({"se": StructuringElement.ball(1),
                                                         "iterations": 0})


class TestStructuringElement:
    def test_factories(self):
        assert len(StructuringElement.ball(3).offsets) == 123
        assert len(StructuringElement.ball(1).offsets) == 7
        assert len(StructuringElement.box(1).offsets) == 27
        assert len(StructuringElement.cross(2).offsets) == 13
        assert StructuringElement.ball(3).z_extent == 3

    def test_parse_and_errors(self):
        assert StructuringElement.parse("ball:2") == StructuringElement.ball(2)
        for bad in ("torus:1", "ball:x", "ball:0"):
            with pytest.raises(ParameterError):
                StructuringElement.parse(bad)
        with pytest.raises(ParameterError):
            StructuringElement(())
        with pytest.raises(ParameterError):
            StructuringElement(((1, 0, 0),))

    def test_matches_oracle_offsets(self, oracle):
        for r in (1, 2, 3):
            assert sorted(StructuringElement.ball(r).offsets) == sorted(oracle.ball_offsets(r))
            assert sorted(StructuringElement.box(r).offsets) == sorted(oracle.box_offsets(r))
            assert sorted(StructuringElement.cross(r).offsets) == sorted(oracle.cross_offsets(r))

    def test_reflect(self):
        se = StructuringElement(((0, 0, 0), (1, 2, -3)))
        assert set(se.reflect().offsets) == {(0, 0, 0), (-1, -2, 3)}


class TestErrors:
    def test_status_mapping(self):
        cases = [(errors.HB_EPARAM, ParameterError), (errors.HB_EBUDGET_SMALL, BudgetTooSmallError),
                 (errors.HB_EBUDGET_UNAVAILABLE, errors.BudgetUnavailableError),
                 (errors.HB_ECHUNK, ChunkExecutionError), (errors.HB_ECUDA, ChunkExecutionError),
                 (errors.HB_ECANCELLED, JobCancelled),
                 (errors.HB_EUNSUPPORTED, errors.UnsupportedFormatError)]
        for code, exc in cases:
            with pytest.raises(exc) as e:
                errors.raise_for_status(code, "m", failed_chunk=3, minimum_bytes=77)
            if exc is ChunkExecutionError:
                assert e.value.chunk_index == 3
            if exc is BudgetTooSmallError:
                assert e.value.minimum_bytes == 77
        errors.raise_for_status(errors.HB_OK, "")


class TestCoerce:
    def test_signed_roundtrip_preserves_order(self):
        x = np.array([[[-128, -1, 0, 1, 127]]], dtype=np.int8)
        prog = filters.median_program(1)
        a, restore = filters.coerce_input(x, prog)
        assert a.dtype == np.uint8
        assert np.all(np.diff(a.astype(int), axis=2) > 0)
        np.testing.assert_array_equal(restore(a), x)

    def test_float_ops_convert_like_reference(self):
        x = np.ones((2, 2, 2), np.float64)
        a, restore = filters.coerce_input(x, filters.gaussian_program(1.0))
        assert a.dtype == np.float32 and restore is None

    def test_rejects(self):
        with pytest.raises(errors.UnsupportedFormatError):
            filters.coerce_input(np.ones((2, 2, 2)), filters.median_program(1))
        with pytest.raises(ParameterError):
            filters.coerce_input(np.ones((2, 2)), filters.median_program(1))


def _budget(shape, dtype, profile, chunks):
    z, y, x = shape
    slice_bytes = y * x * np.dtype(dtype).itemsize
    t = max(1, z // chunks) + 2 * profile.halo_z
    return MemoryBudget(int(t * profile.scratch_factor * slice_bytes) + 1, 1.0)


class TestPythonEngine:
    """execute_chunked with a Python callable keeps the reference contract."""

    def test_identity_any_plan(self, rng):
        vol = rng.integers(0, 256, size=(32, 24, 24), dtype=np.uint8)
        prof = OpProfile(halo_z=0, scratch_factor=2)
        for chunks in (1, 3, 7):
            out, rep = execute_chunked(vol, lambda b, p, a: b, prof, _budget(vol.shape, vol.dtype, prof, chunks))
            assert np.array_equal(out, vol) and rep.chunk_count >= chunks

    def test_failure_index_and_release(self, rng):
        vol = rng.integers(0, 256, size=(32, 24, 24), dtype=np.uint8)
        prof = OpProfile(halo_z=0, scratch_factor=2)
        calls = []

        def boom(b, p, a):
            calls.append(1)
            if len(calls) == 2:
                raise ValueError("synthetic fault")
            return b

        with pytest.raises(ChunkExecutionError) as e:
            execute_chunked(vol, boom, prof, _budget(vol.shape, vol.dtype, prof, 4))
        assert e.value.chunk_index == 1
        assert LEDGER.snapshot().residual_bytes == 0

    def test_cancel(self, rng):
        vol = rng.integers(0, 256, size=(32, 24, 24), dtype=np.uint8)
        prof = OpProfile(halo_z=0, scratch_factor=2)
        seen = []
        with pytest.raises(JobCancelled):
            execute_chunked(vol, lambda b, p, a: seen.append(1) or b, prof,
                            _budget(vol.shape, vol.dtype, prof, 4), cancel=lambda: len(seen) >= 2)
        assert len(seen) == 2

    def test_halo_trim_with_oracle(self, rng, oracle):
        # the chunk engine + halos reproduce the whole-volume result (plan invariance)
        vol = rng.random((24, 12, 12), dtype=np.float32)
        prof = OpProfile(halo_z=1, scratch_factor=4)
        out, rep = execute_chunked(vol, lambda b, p, a: oracle.median(b, 1), prof,
                                   _budget(vol.shape, vol.dtype, prof, 4))
        assert rep.chunk_count >= 4
        assert np.array_equal(out, oracle.median(vol, 1))


def test_ledger_semantics():
    L = MemoryLedger()
    L.charge(100)
    L.job_start()
    L.charge(50)
    L.commit_persistent(10)
    s = L.snapshot()
    assert (s.current_bytes, s.peak_bytes, s.baseline_bytes, s.residual_bytes) == (160, 160, 110, 50)
    L.release(50)
    assert L.snapshot().residual_bytes == 0
    with pytest.raises(ValueError):
        L.charge(-1)


def test_bench_module_mirrors_reference(tmp_path):
    """paper_2511_11890_b200.bench mirrors harpia/bench.py: seeded synthetic
    volumes (bench.py:63-68), scenario validation (bench.py:46-51) and the CSV
    header (bench.py:25)."""
    import numpy as np
    import pytest

    from paper_2511_11890_b200 import bench
    from paper_2511_11890_b200.errors import ParameterError

    v = bench.synthesize(3, 5, "uint16", 7)
    assert v.dtype == np.uint16 and v.shape == (3, 5, 5)
    assert np.array_equal(v, np.random.default_rng(7).integers(0, 65536, size=(3, 5, 5), dtype="uint16"))
    f = bench.synthesize(2, 4, "float32", 0)
    assert np.array_equal(f, np.random.default_rng(0).random((2, 4, 4), dtype=np.float32))
    assert bench.CSV_HEADER == ("size_bytes", "mean_s", "std_s", "peak_bytes", "residual_bytes")
    with pytest.raises(ParameterError):
        bench.BenchScenario(op="median", repeats=0)
    with pytest.raises(ParameterError):
        bench.BenchScenario(op="median", ladder=(64, 64))
    rows = [bench.BenchRow(10, 0.5, 0.1, 7, 0, 1.25, 99, 0, 10, 10)]
    p = tmp_path / "b.csv"
    bench.write_csv(rows, p)
    assert p.read_text().splitlines() == ["size_bytes,mean_s,std_s,peak_bytes,residual_bytes", "10,0.5,0.1,7,0"]
    bench.write_csv(rows, p, device_columns=True)
    assert p.read_text().splitlines()[0].endswith("gvox_s,device_peak_bytes,device_residual_bytes,h2d_bytes,d2h_bytes")


def _sweep_otsu_split(counts):
    counts = counts.astype(np.float64)
    total = counts.sum()
    idx = np.arange(counts.size, dtype=np.float64)
    best_split, best_sigma = None, -1.0
    for t in range(counts.size - 1):
        w0 = counts[: t + 1].sum()
        w1 = total - w0
        if w0 == 0 or w1 == 0:
            continue
        mu0 = (counts[: t + 1] * idx[: t + 1]).sum() / w0
        mu1 = (counts[t + 1:] * idx[t + 1:]).sum() / w1
        sigma = w0 * w1 * (mu0 - mu1) ** 2
        if sigma > best_sigma:
            best_sigma, best_split = sigma, t
    return best_split


def test_acceptance_criterion_04_otsu_sweep():
    """Reference test_acceptance.py:155-188: the host Otsu finalize equals an
    exhaustive between-class-variance sweep on 1000 random histograms."""
    from paper_2511_11890_b200.threshold import Histogram, otsu_from_histogram

    rng = np.random.default_rng(4)
    for _ in range(1000):
        counts = rng.integers(0, 50, size=256).astype(np.int64)
        if np.count_nonzero(counts) < 2:
            counts[10] += 1
            counts[200] += 1
        assert otsu_from_histogram(Histogram(0.0, 256.0, counts)) == float(_sweep_otsu_split(counts))
