"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle and
the reference-generated golden fixtures.

Bars (north star): median / morphology / integer outputs bit-exact; float32
stencils within 1e-5 norm-relative (max|gpu-ref| / max|ref|); the "exact"
Gaussian mode (and LoG, which uses it) bit-exact.
"""
import numpy as np
import pytest

from conftest import budget_for, float_close

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5


@pytest.fixture(scope="module")
def hb():
    import paper_2511_11890_b200 as hb
    from paper_2511_11890_b200 import _native

    assert _native.device_count() >= 1, "no CUDA device: the GPU tests need a B200"
    return hb


def _ours(hb, case, arrays, precision=None):
    from paper_2511_11890_b200 import morphology, registry

    x = arrays[case["input"]]
    op, p = case["op"], dict(case["params"])
    if op == "erode_offsets":
        return morphology.erode(x, morphology.StructuringElement(tuple(map(tuple, arrays[p["offsets"]]))))
    if op == "dilate_offsets":
        return morphology.dilate(x, morphology.StructuringElement(tuple(map(tuple, arrays[p["offsets"]]))))
    if precision is not None and op in ("gaussian", "unsharp", "log"):
        p["precision"] = precision
    if op == "geodesic_reconstruct":  # the marker travels as an array key
        p["marker"] = arrays[p["marker"]]
    return registry.run_direct(x, op, p)


def test_golden_exact_ops(hb, golden):
    """median, morphology, exact-mode Gaussian/unsharp and LoG: bit-exact."""
    meta, arrays = golden
    bad = []
    for case in meta["cases"]:
        if case["op"] == "mean" or (case["op"] == "anisotropic_diffusion"
                                    and case["params"]["mode"] == "exponential"):
            continue
        if _float_box_local(case, arrays):
            continue  # test_local_threshold_golden: float32 window sums, ulp tolerance
        got = _ours(hb, case, arrays, precision="exact")
        want = arrays[case["output"]]
        if got.dtype != want.dtype or not np.array_equal(got, want):
            bad.append(case["name"])
    assert not bad, bad


def _float_box_local(case, arrays):
    return (case["op"] == "local_threshold" and arrays[case["input"]].dtype == np.float32
            and case["params"]["kind"] in ("mean", "niblack", "sauvola"))


def _local_ok(x, got, want, t, rel=1e-12):
    """labels equal except where data sits within rounding of T (float32 box
    kinds: the reference's window sums are cumsum differences over the padded
    chunk, the device's direct float64 sums — both round differently)."""
    bad = got != want
    if not bad.any():
        return True
    xv = x.astype(np.float64)[bad]
    tv = t[bad]
    return bool(np.all(np.abs(xv - tv) <= rel * np.maximum(1.0, np.abs(tv))))


def test_local_threshold_golden(hb, oracle, golden):
    """local_threshold (threshold.py:174-217), all five kinds against the
    reference's own outputs: bit-exact for integer data and for the median /
    gaussian kinds; float32 box kinds equal except at ulp-level ties with T."""
    meta, arrays = golden
    n = 0
    for case in meta["cases"]:
        if case["op"] != "local_threshold":
            continue
        n += 1
        got = _ours(hb, case, arrays)
        want = arrays[case["output"]]
        assert got.dtype == want.dtype == np.uint32, case["name"]
        if _float_box_local(case, arrays):
            p = case["params"]
            x = arrays[case["input"]]
            t = oracle.local_threshold(x, p["kind"], p["window"], p["k"], p["R"], p["c"], return_t=True)
            assert _local_ok(x, got, want, t), case["name"]
        else:
            assert np.array_equal(got, want), case["name"]
    assert n >= 40


@pytest.mark.parametrize("shape", [(40, 67, 129), (9, 1, 40), (6, 33, 7), (70, 40, 36)])
def test_local_threshold_vs_oracle(hb, oracle, shape):
    """every kind and dtype on ragged shapes, windows 1..4, and through a
    tight chunk plan (integer data: bit-exact for any plan)."""
    from paper_2511_11890_b200 import registry, threshold

    rng = np.random.default_rng(sum(shape) + 3)
    for dt in ("u8", "u16", "f32"):
        x = _vol(rng, shape, dt)
        for kind in threshold.LOCAL_KINDS:
            for w in ((1, 3) if kind != "median" else (1, 2)):
                k = 0.2 if kind != "niblack" else -0.2
                c = 0.01 if dt == "f32" else 2.0
                got = threshold.local_threshold(x, kind, w, k, None, c)
                want = oracle.local_threshold(x, kind, w, k, None, c)
                if dt == "f32" and kind in ("mean", "niblack", "sauvola"):
                    t = oracle.local_threshold(x, kind, w, k, None, c, return_t=True)
                    assert _local_ok(x, got, want, t), (dt, kind, w)
                else:
                    assert np.array_equal(got, want), (dt, kind, w)
    # chunked: a budget that forces several chunks (halo = window)
    x = _vol(rng, shape, "u16")
    for kind in ("sauvola", "gaussian", "median"):
        p = {"kind": kind, "window": 2}
        op = registry.get_operator("local_threshold")
        prof = op.profile(registry.validate_params(op, p))
        out, rep = registry.run_operator(x, "local_threshold", p,
                                         budget=budget_for(prof, x.shape, x.dtype, 4))
        assert np.array_equal(out, oracle.local_threshold(x, kind, 2)), kind


def test_local_threshold_wide_windows(hb, oracle):
    """windows past the compile-time kernels (w > 4: runtime-window box and
    gaussian kernels), integer data bit-exact."""
    from paper_2511_11890_b200 import threshold

    rng = np.random.default_rng(17)
    for dt, shape in (("u8", (14, 23, 41)), ("u16", (12, 19, 37))):
        x = _vol(rng, shape, dt)
        for kind in ("mean", "niblack", "sauvola", "gaussian"):
            for w in (5, 7):
                got = threshold.local_threshold(x, kind, w, 0.2, None, 1.0)
                assert np.array_equal(got, oracle.local_threshold(x, kind, w, 0.2, None, 1.0)), (dt, kind, w)


def test_local_threshold_errors(hb):
    from paper_2511_11890_b200 import threshold
    from paper_2511_11890_b200.errors import ParameterError

    x = np.zeros((3, 3, 3), np.uint8)
    with pytest.raises(ParameterError):
        threshold.local_threshold(x, "bogus", 1)
    with pytest.raises(ParameterError):
        threshold.local_threshold(x, "mean", 0)
    with pytest.raises(ParameterError):
        threshold.local_threshold(x, "sauvola", 1, r=-1.0)
    assert threshold.default_sauvola_r(np.uint16) == 32767.5


def test_golden_fast_ops(hb, golden):
    meta, arrays = golden
    worst = {}
    for case in meta["cases"]:
        if case["op"] not in ("gaussian", "unsharp", "mean", "anisotropic_diffusion"):
            continue
        got = _ours(hb, case, arrays, precision="fast")
        want = arrays[case["output"]]
        assert got.dtype == want.dtype == np.float32
        err = float_close(got, want)
        worst[case["name"]] = err
        assert err <= FLOAT_TOL, (case["name"], err)


def _vol(rng, shape, dt):
    if dt == "f32":
        return rng.random(shape, dtype=np.float32)
    if dt == "u16":
        return rng.integers(0, 65536, size=shape, dtype=np.uint16)
    if dt == "bin":
        return (rng.random(shape) < 0.5).astype(np.uint8)
    return rng.integers(0, 256, size=shape, dtype=np.uint8)


SHAPES = [(40, 67, 129), (7, 256, 64), (33, 1, 300), (3, 5, 2)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dt", ["f32", "u16", "u8"])
def test_random_vs_oracle(hb, oracle, shape, dt):
    from paper_2511_11890_b200 import filters, morphology

    rng = np.random.default_rng(hash((shape, dt)) % 2**32)
    x = _vol(rng, shape, dt)
    assert np.array_equal(filters.median(x, 1), oracle.median(x, 1))
    if shape[0] * shape[1] * shape[2] < 400_000:
        assert np.array_equal(filters.median(x, 2), oracle.median(x, 2))
    assert np.array_equal(filters.gaussian(x, 2.0, "exact"), oracle.gaussian(x, 2.0))
    assert float_close(filters.gaussian(x, 2.0), oracle.gaussian(x, 2.0)) <= FLOAT_TOL
    assert float_close(filters.mean(x, 1), oracle.mean(x, 1)) <= FLOAT_TOL
    assert np.array_equal(filters.log(x, 2.0), oracle.log(x, 2.0))
    assert float_close(filters.unsharp(x, 1.0, 1.5), oracle.unsharp(x, 1.0, 1.5)) <= FLOAT_TOL
    for se in ("ball:3", "box:1", "cross:2"):
        s = morphology.StructuringElement.parse(se)
        assert np.array_equal(morphology.erode(x, s), oracle.erode(x, s.offsets)), se
        assert np.array_equal(morphology.dilate(x, s), oracle.dilate(x, s.offsets)), se


ALL_OPS = [
    ("identity", {}, "u8"),
    ("gaussian", {"sigma": 1.5}, "u8"),
    ("gaussian", {"sigma": 2.0}, "f32"),
    ("gaussian", {"sigma": 2.0, "precision": "exact"}, "f32"),
    ("mean", {"radius": 2}, "u8"),
    ("mean", {"radius": 1}, "f32"),
    ("median", {"radius": 1}, "u8"),
    ("median", {"radius": 1}, "f32"),
    ("median", {"radius": 2}, "u16"),
    ("unsharp", {"sigma": 1.0, "amount": 1.5}, "u8"),
    ("log", {"sigma": 2.0}, "f32"),
    ("morph_erode", {"se": "ball:3"}, "u16"),
    ("morph_dilate", {"se": "box:1"}, "u8"),
    ("morph_open", {"se": "ball:1", "iterations": 2}, "bin"),
    ("morph_close", {"se": "cross:1"}, "u8"),
    ("hessian_xz", {"sigma": 1.5}, "f32"),
    ("hessian_yy", {"sigma": 1.0}, "u16"),
    ("sobel", {}, "u8"),
    ("prewitt", {}, "f32"),
    ("apply_threshold", {"t": 0.5}, "f32"),
    ("anisotropic_diffusion", {"iterations": 3, "kappa": 0.3, "mode": "rational"}, "f32"),
    ("anisotropic_diffusion", {"iterations": 2, "kappa": 20.0}, "u8"),
]


@pytest.mark.parametrize("name,params,dt", ALL_OPS)
def test_plan_invariance(hb, name, params, dt):
    """Acceptance criterion 1 (reference test_acceptance.py:73-97): chunked ==
    whole volume.  The device arithmetic per voxel does not depend on the plan,
    so we require bit-identity for every operator."""
    from paper_2511_11890_b200 import registry

    rng = np.random.default_rng(2024)
    x = _vol(rng, (64, 48, 40), dt)
    op = registry.get_operator(name)
    prof = op.profile(registry.validate_params(op, params))
    whole = registry.run_direct(x, name, params)
    for chunks in (4, 7):
        got, rep = registry.run_operator(x, name, params, budget_for(prof, x.shape, x.dtype, chunks))
        assert rep.chunk_count >= chunks
        assert np.array_equal(got, whole), (name, chunks)
        assert rep.device_residual_bytes == 0
        assert rep.residual_bytes == 0
        assert len(rep.chunk_seconds) == rep.chunk_count


def test_halo_shrink_breaks_invariance(hb):
    """Reference test_chunking.py:254-278: a halo one slice short must corrupt seams."""
    from paper_2511_11890_b200 import _native, filters
    from paper_2511_11890_b200.chunking import OpProfile, execute_chunked

    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, size=(24, 12, 12), dtype=np.uint8)
    prog = filters.median_program(1)
    lying = OpProfile(halo_z=0, scratch_factor=4)
    out, rep = execute_chunked(x, prog, lying, budget_for(lying, x.shape, x.dtype, 4))
    assert rep.chunk_count >= 2
    assert not np.array_equal(out, filters.median(x, 1))


def test_native_fault_and_cancel(hb):
    from paper_2511_11890_b200 import _native, registry
    from paper_2511_11890_b200.errors import ChunkExecutionError, JobCancelled
    from paper_2511_11890_b200.ledger import LEDGER

    x = np.random.default_rng(1).random((32, 24, 24), dtype=np.float32)
    op = registry.get_operator("gaussian")
    prof = op.profile({"sigma": 1.0, "precision": "fast"})
    b = budget_for(prof, x.shape, x.dtype, 4)
    with pytest.raises(ChunkExecutionError) as e:
        registry.run_operator(x, "gaussian", {"sigma": 1.0}, b, fault_chunk=1)
    assert e.value.chunk_index == 1
    assert LEDGER.snapshot().residual_bytes == 0
    assert _native.device_pool_bytes() == 0
    calls = []
    with pytest.raises(JobCancelled):
        registry.run_operator(x, "gaussian", {"sigma": 1.0}, b,
                              cancel=lambda: calls.append(1) or len(calls) > 2)
    assert len(calls) == 3
    assert _native.device_pool_bytes() == 0


def test_pinned_and_pageable_paths_agree(hb):
    import torch
    from paper_2511_11890_b200 import registry

    x = np.random.default_rng(3).random((96, 128, 160), dtype=np.float32)
    pinned = torch.empty(x.shape, dtype=torch.float32).pin_memory().numpy()
    pinned[...] = x
    op = registry.get_operator("median")
    prof = op.profile({"radius": 1})
    b = budget_for(prof, x.shape, x.dtype, 5)
    a, ra = registry.run_operator(x, "median", {"radius": 1}, b)
    c, rc = registry.run_operator(pinned, "median", {"radius": 1}, b)
    assert np.array_equal(a, c) and ra.chunk_count == rc.chunk_count >= 5
    # device z-ring: halo slices are reused on the device, every input byte crosses PCIe once
    assert ra.h2d_bytes == rc.h2d_bytes == x.nbytes


def test_torch_device_blocks(hb, oracle):
    import torch
    from paper_2511_11890_b200 import filters, morphology

    x = np.random.default_rng(4).random((20, 33, 47), dtype=np.float32)
    t = torch.from_numpy(x).cuda()
    assert np.array_equal(filters.median(t, 1).cpu().numpy(), oracle.median(x, 1))
    assert np.array_equal(filters.gaussian(t, 2.0, "exact").cpu().numpy(), oracle.gaussian(x, 2.0))
    u = torch.from_numpy((x * 60000).astype(np.uint16)).cuda()
    s = morphology.StructuringElement.ball(2)
    got = morphology.erode(u, s).cpu().numpy()
    assert np.array_equal(got, oracle.erode(u.cpu().numpy(), s.offsets))


def test_signed_and_bool_inputs(hb, oracle):
    from paper_2511_11890_b200 import filters, morphology

    rng = np.random.default_rng(6)
    x = rng.integers(-30000, 30000, size=(9, 10, 11), dtype=np.int16)
    got = filters.median(x, 1)
    assert got.dtype == np.int16
    pad = np.pad(x, 1, mode="edge")
    ref = np.empty_like(x)
    for i in range(9):
        for j in range(10):
            for k in range(11):
                ref[i, j, k] = np.sort(pad[i:i + 3, j:j + 3, k:k + 3].ravel())[13]
    assert np.array_equal(got, ref)
    m = rng.random((8, 9, 10)) < 0.5
    e = morphology.erode(m, morphology.StructuringElement.ball(1))
    assert e.dtype == np.bool_
    assert np.array_equal(e, oracle.erode(m.astype(np.uint8), morphology.StructuringElement.ball(1).offsets).astype(bool))


def test_pipeline_matches_sequential(hb):
    from paper_2511_11890_b200 import registry

    x = np.random.default_rng(7).random((48, 40, 36), dtype=np.float32)
    steps = [("unsharp", {"sigma": 1.0, "amount": 1.5}), ("log", {"sigma": 2.0})]
    seq = registry.run_direct(registry.run_direct(x, *steps[0]), *steps[1])
    from paper_2511_11890_b200.chunking import MemoryBudget
    got, rep = registry.run_pipeline(x, steps, MemoryBudget(40 * 40 * 36 * 4 * 10, 1.0))
    assert rep.chunk_count > 1
    assert np.array_equal(got, seq)


def test_large_slab_sampled_median(hb, oracle):
    """Config-2 scale (1024^2 slices): slab-sampled exact parity (plan invariance
    lets the oracle evaluate padded slabs only)."""
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(0)
    x = rng.random((64, 1024, 1024), dtype=np.float32)
    got = filters.median(x, 1)
    for z0 in (0, 29, 63):
        lo, hi = max(0, z0 - 1), min(64, z0 + 2)
        ref = oracle.median(x[lo:hi], 1)
        assert np.array_equal(got[z0], ref[z0 - lo])


@pytest.mark.parametrize("dt", ["u16", "u8", "bin"])
def test_factory_se_fast_path(hb, oracle, dt):
    """The compile-time SE kernels (ball/box/cross r<=3) on tile-aligned and
    ragged shapes, erosion and dilation, bit-exact."""
    from paper_2511_11890_b200 import morphology

    rng = np.random.default_rng(11)
    for shape in [(12, 64, 128), (9, 33, 70), (5, 64, 64)]:
        x = _vol(rng, shape, dt)
        for kind in ("ball", "box", "cross"):
            for r in (1, 2, 3):
                s = morphology.StructuringElement.parse(f"{kind}:{r}")
                assert np.array_equal(morphology.erode(x, s), oracle.erode(x, s.offsets)), (shape, kind, r)
                assert np.array_equal(morphology.dilate(x, s), oracle.dilate(x, s.offsets)), (shape, kind, r)


def test_pinned_context_direct_dma(hb):
    from paper_2511_11890_b200 import pinned, registry
    from paper_2511_11890_b200.chunking import MemoryBudget

    x = np.random.default_rng(8).random((64, 96, 128), dtype=np.float32)
    out = np.empty_like(x)
    b = MemoryBudget(20 * 96 * 128 * 4 * 4, 1.0)
    want, _ = registry.run_operator(x, "median", {"radius": 1}, b)
    with pinned(x, out):
        got, rep = registry.run_operator(x, "median", {"radius": 1}, b, out=out)
    assert got is out and np.array_equal(out, want) and rep.device_residual_bytes == 0


STREAM_SHAPES = [(21, 37, 132), (9, 70, 260), (5, 3, 516), (12, 130, 128), (2, 9, 4)]


@pytest.mark.parametrize("shape", STREAM_SHAPES)
def test_streaming_kernels_vs_oracle(hb, oracle, shape):
    """Shapes that exercise the streaming kernels' strip tails and faces
    (box.cu mean, logd.cu LoG stage, k_gauss_p2): x = 128k + 4 (one live lane in
    the last strip), tiny y, ny < the warp's row block, nz < 2R+1."""
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(sum(shape))
    for dt in ("f32", "u16", "u8"):
        x = _vol(rng, shape, dt)
        assert float_close(filters.mean(x, 1), oracle.mean(x, 1)) <= FLOAT_TOL, dt
        assert float_close(filters.mean(x, 2), oracle.mean(x, 2)) <= FLOAT_TOL, dt
        assert float_close(filters.gaussian(x, 2.0), oracle.gaussian(x, 2.0)) <= FLOAT_TOL, dt
        assert float_close(filters.unsharp(x, 1.0, 1.5), oracle.unsharp(x, 1.0, 1.5)) <= FLOAT_TOL, dt
    x = _vol(rng, shape, "f32")
    assert np.array_equal(filters.log(x, 2.0), oracle.log(x, 2.0))
    xi = _vol(rng, shape, "u16")
    assert np.array_equal(filters.mean(xi, 1), oracle.mean(xi, 1))  # integer sums: exact


def test_device_session_keeps_pool_until_exit(hb):
    """hb_session_begin/end: jobs inside a session free every buffer (job
    residual 0) but leave the pool mapped; leaving the session trims it."""
    from paper_2511_11890_b200 import _native, registry, session

    x = np.random.default_rng(5).random((24, 64, 64), dtype=np.float32)
    _, rep = registry.run_operator(x, "median", {"radius": 1})
    assert rep.device_residual_bytes == 0 and _native.device_pool_bytes() == 0
    with session():
        a, r1 = registry.run_operator(x, "median", {"radius": 1})
        b, r2 = registry.run_operator(x, "mean", {"radius": 1})
        assert r1.device_residual_bytes == 0 and r2.device_residual_bytes == 0
        assert _native.device_pool_bytes() > 0
    assert _native.device_pool_bytes() == 0
    assert np.array_equal(a, registry.run_operator(x, "median", {"radius": 1})[0])


def test_bench_harness_runs_on_device(hb):
    """harpia/bench.py's run_bench over the device executor: one row per ladder
    entry, zero residual device memory, sane throughput."""
    from paper_2511_11890_b200 import bench

    sc = bench.BenchScenario(op="median", params={"radius": 1}, ladder=(16, 32), base_yx=64,
                             repeats=3, dtype="float32")
    rows = bench.run_bench(sc)
    assert [r.size_bytes for r in rows] == [16 * 64 * 64 * 4, 32 * 64 * 64 * 4]
    assert all(r.device_residual_bytes == 0 and r.residual_bytes == 0 and r.gvox_s > 0 for r in rows)


@pytest.mark.parametrize("shape", [(21, 37, 132), (9, 1, 40), (6, 33, 7)])
def test_next_map_ops_vs_oracle(hb, oracle, shape):
    """SURVEY.md §8(f) row 2 ops (hessian components, sobel, prewitt,
    apply_threshold): bit-exact against the oracle on ragged shapes."""
    from paper_2511_11890_b200 import filters, threshold

    rng = np.random.default_rng(sum(shape) + 7)
    for dt in ("f32", "u16", "u8"):
        x = _vol(rng, shape, dt)
        for comp in filters.HESSIAN_COMPONENTS:
            assert np.array_equal(filters.hessian_component(x, 1.2, comp),
                                  oracle.hessian_component(x, 1.2, comp)), (dt, comp)
        assert np.array_equal(filters.sobel(x), oracle.sobel(x)), dt
        assert np.array_equal(filters.prewitt(x), oracle.prewitt(x)), dt
        t = 0.37 if dt == "f32" else 100.5
        assert np.array_equal(filters.lbp2d(x), oracle.lbp2d(x)), dt
        got = threshold.apply_threshold(x, t)
        assert got.dtype == np.uint32 and np.array_equal(got, oracle.apply_threshold(x, t)), dt


def test_anisotropic_diffusion_vs_oracle(hb, oracle):
    """rational mode bit-exact (pure float32 arithmetic in the reference's
    order); exponential mode within 1e-5 (expf vs NumPy's SIMD exp)."""
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(11)
    for shape, dt in (((14, 33, 40), "f32"), ((9, 20, 132), "u16"), ((5, 1, 17), "f32")):
        x = _vol(rng, shape, dt)
        for it, kappa in ((1, 0.3), (4, 15.0)):
            r = filters.anisotropic_diffusion(x, it, kappa, 1.0 / 6.0, "rational")
            assert np.array_equal(r, oracle.anisotropic_diffusion(x, it, kappa, 1.0 / 6.0, "rational"))
            e = filters.anisotropic_diffusion(x, it, kappa)
            assert float_close(e, oracle.anisotropic_diffusion(x, it, kappa)) <= FLOAT_TOL


def test_otsu_two_pass_on_device(hb, oracle, golden):
    """Global Otsu (threshold.py:90-131) through the device: the histogram is
    np.histogram bit for bit, the threshold is the reference's, and the
    chunked apply pass equals the direct one."""
    from conftest import budget_for
    from paper_2511_11890_b200 import registry, threshold

    meta, arrays = golden
    for name, t_ref in meta["otsu_thresholds"].items():
        case = next(c for c in meta["cases"] if c["name"] == name)
        assert threshold.otsu(arrays[case["input"]], case["params"]["bins"]) == t_ref, name
    rng = np.random.default_rng(8)
    for shape, dt in (((40, 67, 129), "f32"), ((7, 256, 64), "u16"), ((33, 1, 300), "u8")):
        x = _vol(rng, shape, dt)
        if dt == "f32":
            x = x * 3.5 - 1.0
        r = threshold.histogram_range(x)
        assert r == oracle.histogram_range(x)
        for bins in (256, 37):
            np.testing.assert_array_equal(threshold.compute_histogram(x, bins, r).counts,
                                          oracle.histogram(x, bins, r))
        direct = registry.run_direct(x, "otsu", {})
        op = registry.get_operator("apply_threshold")
        prof = op.profile({"t": 0.0})
        chunked, rep = registry.run_operator(x, "otsu", {}, budget_for(prof, x.shape, np.dtype(np.uint32), 4))
        assert np.array_equal(direct, chunked) and direct.dtype == np.uint32
        assert rep.threshold == oracle.otsu(x)
        assert np.array_equal(direct, oracle.apply_threshold(x, oracle.otsu(x)))


@pytest.mark.parametrize("conn", [6, 26])
def test_connected_components_vs_oracle(hb, oracle, conn):
    """quantify.py:60-111: canonical labels (1..count, first-voxel scan order)
    bit-exact, on ragged shapes and densities around the percolation point,
    host and device inputs; the registry's chunked run gives the same labels."""
    import torch

    from conftest import budget_for
    from paper_2511_11890_b200 import quantify, registry
    from paper_2511_11890_b200.chunking import OpProfile

    rng = np.random.default_rng(conn)
    for shape in ((40, 67, 129), (1, 1, 9), (64, 64, 64), (9, 200, 3)):
        for dens in (0.15, 0.3, 0.6):
            m = (rng.random(shape) < dens).astype(np.uint8)
            want, n = oracle.connected_components(m, conn)
            got, k = quantify.connected_components(m, conn)
            assert k == n and got.dtype == np.uint32 and np.array_equal(got, want), (shape, dens)
    m = (rng.random((96, 80, 72)) < 0.3)
    want, n = oracle.connected_components(m.astype(np.uint8), conn)
    dev, k = quantify.connected_components(torch.from_numpy(m).cuda(), conn)
    assert k == n and np.array_equal(dev.cpu().numpy(), want)
    lab, rep = registry.run_operator(m.astype(np.uint8), "connected_components", {"connectivity": conn},
                                     budget_for(OpProfile(0, 6), m.shape, np.uint8, 4))
    assert rep.component_count == n and np.array_equal(lab, want)


def test_label_filters_vs_oracle(hb, oracle):
    """fill_holes / remove_islands (morphology.py:176-229) on the device
    labelling: bit-exact, dtype preserved, host and device inputs."""
    import torch

    from paper_2511_11890_b200 import morphology

    rng = np.random.default_rng(21)
    for shape in ((24, 40, 33), (5, 1, 60), (40, 40, 40)):
        m = (rng.random(shape) < 0.6).astype(np.uint8)
        lab = rng.integers(0, 5, size=shape).astype(np.uint32)
        lab[rng.random(shape) < 0.35] = 0
        for conn in (6, 26):
            assert np.array_equal(morphology.fill_holes(m, conn), oracle.fill_holes(m, conn))
            assert np.array_equal(morphology.fill_holes(lab, conn), oracle.fill_holes(lab, conn))
            for ms in (2, 6):
                got = morphology.remove_islands(lab, ms, conn)
                assert got.dtype == lab.dtype and np.array_equal(got, oracle.remove_islands(lab, ms, conn))
    dev = morphology.remove_islands(torch.from_numpy(lab).cuda(), 4, 26)
    assert np.array_equal(dev.cpu().numpy(), oracle.remove_islands(lab, 4, 26))


def test_geodesic_reconstruct_vs_oracle(hb, oracle):
    """morphology.py:143-165: the device's in-place sweeps reach the same
    (unique) fixed point as the reference's Jacobi steps; ordering violations
    raise ParameterError."""
    from paper_2511_11890_b200 import morphology
    from paper_2511_11890_b200.errors import ParameterError

    rng = np.random.default_rng(31)
    for shape, dt in (((20, 30, 41), np.uint8), ((9, 64, 64), np.uint16), ((12, 1, 90), np.float32)):
        mask = (rng.random(shape) * 200).astype(dt)
        seeds = rng.random(shape) < 0.01
        m_dil = np.where(seeds, mask, 0).astype(dt)
        assert np.array_equal(morphology.geodesic_reconstruct(m_dil, mask, "dilation"),
                              oracle.geodesic_reconstruct(m_dil, mask, "dilation"))
        m_ero = np.where(seeds, mask, mask.max()).astype(dt)
        assert np.array_equal(morphology.geodesic_reconstruct(m_ero, mask, "erosion"),
                              oracle.geodesic_reconstruct(m_ero, mask, "erosion"))
    with pytest.raises(ParameterError):
        morphology.geodesic_reconstruct(mask.max() + np.zeros_like(mask) + 1, mask, "dilation")


def test_edt_vs_oracle(hb, oracle):
    """quantify.py:115-175: bit-exact float32 distances and float64 squared
    distances, anisotropic spacing, no-background volumes (+inf)."""
    from paper_2511_11890_b200 import quantify

    rng = np.random.default_rng(41)
    for shape in ((24, 33, 40), (1, 7, 64), (50, 1, 1), (16, 16, 16)):
        for dens in (0.7, 0.98, 1.0):
            m = (rng.random(shape) < dens).astype(np.uint8)
            for sp in ((1.0, 1.0, 1.0), (2.0, 0.5, 0.75)):
                assert np.array_equal(quantify.edt(m, sp), oracle.edt(m, sp)), (shape, dens, sp)
                assert np.array_equal(quantify.edt(m, sp, squared=True), oracle.edt(m, sp, squared=True))


@pytest.mark.parametrize("slices", [1, 3, 7])
def test_connected_components_chunked_vs_oracle(hb, oracle, slices, monkeypatch):
    """The z-chunked labelling (volumes beyond one device pass; forced here with
    HB_CC_CHUNK_SLICES) merges boundary equivalences with the reference's
    union-find rule and yields the same canonical labels."""
    from paper_2511_11890_b200 import quantify

    monkeypatch.setenv("HB_CC_CHUNK_SLICES", str(slices))
    rng = np.random.default_rng(slices)
    for shape in ((23, 40, 37), (9, 1, 50), (16, 33, 2)):
        for dens in (0.2, 0.35, 0.6):
            m = (rng.random(shape) < dens).astype(np.uint8)
            for conn in (6, 26):
                want, n = oracle.connected_components(m, conn)
                got, k = quantify.connected_components(m, conn)
                assert k == n and np.array_equal(got, want), (shape, dens, conn)


@pytest.mark.parametrize("steps", [
    [("gaussian", {"sigma": 1.0, "precision": "exact"}), ("apply_threshold", {"t": 0.5})],
    [("sobel", {}), ("median", {"radius": 1})],
    [("anisotropic_diffusion", {"iterations": 2, "kappa": 0.4, "mode": "rational"}), ("lbp2d", {})],
    [("hessian_xy", {"sigma": 1.0}), ("morph_dilate", {"se": "box:1"})],
])
def test_pipelines_of_next_ops(hb, oracle, steps):
    """run_pipeline fuses the §8(f) ops with the hot-path ones into one device
    chain per chunk: chunked (3+ chunks) == the oracle applied op by op."""
    from conftest import budget_for
    from paper_2511_11890_b200 import registry
    from paper_2511_11890_b200.chunking import OpProfile

    x = np.random.default_rng(5).random((40, 33, 28), dtype=np.float32)
    want = x
    halo = 0
    for name, p in steps:
        q = dict(p)
        q.pop("precision", None)
        if name.startswith("morph_"):
            want = oracle.morph(want, name[6:], oracle.parse_se(q["se"]), 1)
        else:
            want = oracle.apply(name, want, q)
        halo += registry.get_operator(name).profile(registry.validate_params(registry.get_operator(name), p)).halo_z
    got, rep = registry.run_pipeline(x, steps, budget_for(OpProfile(halo, 12), x.shape, x.dtype, 6))
    assert rep.chunk_count >= 3
    assert got.dtype == want.dtype and np.array_equal(got, want)


def test_connected_components_sharded_single_rank_device(hb, oracle):
    """sharding.connected_components_sharded on a CUDA slab (world 1): the
    device labelling plus the on-device table gather give the canonical labels."""
    import torch

    from paper_2511_11890_b200 import sharding

    m = (np.random.default_rng(5).random((30, 41, 37)) < 0.4).astype(np.uint8)
    want, n = oracle.connected_components(m, 26)
    got, total = sharding.connected_components_sharded(torch.from_numpy(m).cuda(), 26, 0, 1)
    assert total == n and np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("dt,nx", [("u8", 13), ("u16", 21), ("f32", 30), ("u8", 47)])
def test_row_widening_exact(hb, oracle, dt, nx):
    """x extents off the 16-byte pitch run the TMA kernels on edge-replicated
    widened rows (executor run_stage): results stay bit-exact (exact modes,
    morphology, LoG) / within the float tolerance (fast mean)."""
    from paper_2511_11890_b200 import filters, morphology

    rng = np.random.default_rng(nx)
    x = _vol(rng, (19, 23, nx), dt)
    assert np.array_equal(filters.gaussian(x, 1.5, "exact"), oracle.gaussian(x, 1.5))
    assert np.array_equal(filters.unsharp(x, 1.0, 1.5, "exact"), oracle.unsharp(x, 1.0, 1.5))
    assert np.array_equal(filters.log(x, 1.2), oracle.log(x, 1.2))
    assert float_close(filters.mean(x, 2), oracle.mean(x, 2)) <= FLOAT_TOL
    for se in ("ball:3", "box:1", "cross:2"):
        s = morphology.StructuringElement.parse(se)
        offs = oracle.parse_se(se)
        assert np.array_equal(morphology.erode(x, s), oracle.erode(x, offs)), se
        assert np.array_equal(morphology.dilate(x, s), oracle.dilate(x, offs)), se
