"""Drop-in surface (CPU): every name the reference package exports at top
level that is on, or beside, the hot path (reference __init__.py:3-30) imports
from the B200 package; the service's ``validate=False`` call shape works; the
two-pass engine keeps the reference contract (chunking.py:282-335)."""
import numpy as np
import pytest

# reference __init__.py:3-30, minus the out-of-scope annotation / watershed /
# label-metrics / volume-crop helpers (not on the hot path)
REFERENCE_NAMES = [
    "ChunkPlan", "ExecutionReport", "MemoryBudget", "OpProfile", "execute_chunked",
    "execute_two_pass", "plan_chunks", "profile_budget",
    "BudgetTooSmallError", "BudgetUnavailableError", "ChunkExecutionError", "CorruptInputError",
    "HarpiaError", "JobCancelled", "ParameterError", "UnsupportedFormatError",
    "LEDGER", "MemoryLedger",
    "StructuringElement", "fill_holes", "geodesic_reconstruct", "morph", "remove_islands",
    "connected_components", "edt",
    "get_operator", "operator_names", "run_direct", "run_operator",
    "apply_threshold", "local_threshold", "otsu", "otsu_binarize",
    "Volume", "VolumeMeta", "load_volume", "save_volume",
]


def test_reference_top_level_names_import():
    import paper_2511_11890_b200 as hb

    missing = [n for n in REFERENCE_NAMES if not hasattr(hb, n)]
    assert not missing, missing


@pytest.mark.parametrize("name,raw", [
    ("gaussian", {"sigma": 2.0}),
    ("unsharp", {"sigma": 1.0, "amount": 1.5}),
    ("log", {"sigma": 2.0}),
    ("hessian_xy", {"sigma": 1.0}),
    ("median", {"radius": 1}),
    ("mean", {"radius": 2}),
    ("morph_open", {"se": "ball:2"}),
])
def test_unvalidated_params_match_validated(name, raw):
    """service.py:131-139 calls run_operator(..., validate=False) with the
    params it validated at submit time; the profile and program built from
    the unvalidated dict equal those of the validated one."""
    from paper_2511_11890_b200 import registry

    op = registry.get_operator(name)
    validated = registry.validate_params(op, raw)
    unval = registry._unvalidated(op, validated)
    assert registry._profile_for(op, unval) == op.profile(validated)
    a = registry._program_for(op, unval)
    b = op.program(validated)
    assert len(a.stages) == len(b.stages)
    for sa, sb in zip(a.stages, b.stages):
        for k, va in sa.__dict__.items():
            vb = sb.__dict__[k]
            if isinstance(va, np.ndarray) or isinstance(vb, np.ndarray):
                assert np.array_equal(va, vb), k
            else:
                assert va == vb, k


def test_unvalidated_missing_required_is_parameter_error():
    from paper_2511_11890_b200 import registry
    from paper_2511_11890_b200.errors import ParameterError

    op = registry.get_operator("gaussian")
    with pytest.raises(ParameterError):
        registry._profile_for(op, registry._unvalidated(op, {}))


def test_plan_of_empty_volume_has_no_chunks():
    """chunking.py:157-166: nz == 0 plans zero chunks (no ValueError)."""
    from paper_2511_11890_b200.chunking import MemoryBudget, OpProfile, plan_chunks

    plan = plan_chunks((0, 8, 8), np.float32, OpProfile(halo_z=2, scratch_factor=4),
                       MemoryBudget(1 << 20, 1.0))
    assert plan.chunks == () and plan.working_peak_bytes == 0


def test_execute_two_pass_host_contract():
    """Reference contract with host callables: a global min-max normalise
    reduced over chunks, applied chunk by chunk."""
    from paper_2511_11890_b200 import MemoryBudget, OpProfile, execute_two_pass

    x = np.random.default_rng(5).random((23, 9, 11), dtype=np.float32)
    budget = MemoryBudget(3 * 4 * 9 * 11 * 3, 1.0)  # 4 slices per chunk
    calls = []

    def reduce_fn(block, _p):
        calls.append(block.shape[0])
        return float(block.min()), float(block.max())

    out, rep = execute_two_pass(
        x, reduce_fn, lambda a, b: (min(a[0], b[0]), max(a[1], b[1])),
        lambda s, _p: s, lambda block, st, _p: ((block - st[0]) / (st[1] - st[0])).astype(np.float32),
        budget, apply_profile=OpProfile(halo_z=0, scratch_factor=3, out_dtype=np.dtype("float32")))
    assert len(calls) > 1 and sum(calls) == x.shape[0]
    want = (x - x.min()) / (x.max() - x.min())
    assert np.array_equal(out, want.astype(np.float32)) and rep.chunk_count > 1
