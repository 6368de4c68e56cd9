import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "golden_meta.json").read_text())
    arrays = dict(np.load(GOLDEN / "golden_arrays.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    # test infrastructure only: the CPU restatement of the reference
    from oracle import oracle as O

    O.lib()
    return O


def budget_for(profile, shape, dtype, chunks):
    """Budget that splits ``shape`` into about ``chunks`` chunks for ``profile``
    (reference test_acceptance.py:21-25)."""
    from paper_2511_11890_b200.chunking import MemoryBudget

    z, y, x = shape
    slice_bytes = y * x * np.dtype(dtype).itemsize
    t = max(1, z // chunks) + 2 * profile.halo_z
    return MemoryBudget(int(t * profile.scratch_factor * slice_bytes) + 1, 1.0)


def float_close(got, want, tol=1e-5):
    """Norm-relative float parity: max|got-want| / max|want| <= tol."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.max(np.abs(want)), 1e-30)
    return float(np.max(np.abs(got - want)) / scale) if got.size else 0.0
