"""The C-ABI library loads, exports every symbol include/harpia_b200.h
declares, and its ctypes structs match the C layout.  No GPU needed."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2511_11890_b200 import _native, filters

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "harpia_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(hb_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = _native.load()
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_native.EXPORTS)


def test_version_and_abi():
    L = _native.load()
    assert L.hb_abi_version() == 1
    assert b"sm_100a" in L.hb_version()


def test_no_device_is_a_loud_error():
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_2511_11890_b200.errors import BudgetUnavailableError
    with pytest.raises(BudgetUnavailableError):
        _native.device_info(0)
    with pytest.raises(BudgetUnavailableError):
        filters.gaussian(np.zeros((4, 4, 4), np.float32), 1.0)


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(f'#include "{HEADER}"\n#include <stdio.h>\n#include <stddef.h>\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(hb_volume), '
                   'sizeof(hb_stage), sizeof(hb_chunk), sizeof(hb_exec), sizeof(hb_report), '
                   'offsetof(hb_stage, weights), offsetof(hb_report, message));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_native.HbVolume), ctypes.sizeof(_native.HbStage),
            ctypes.sizeof(_native.HbChunk), ctypes.sizeof(_native.HbExec),
            ctypes.sizeof(_native.HbReport), _native.HbStage.weights.offset,
            _native.HbReport.message.offset]
    assert got == want


def test_host_helpers(golden):
    L = _native.load()
    meta, _ = golden
    for sigma, w in meta["weights"].items():
        buf = (ctypes.c_float * 200)()
        n = L.hb_gaussian_weights(float(sigma), buf, 200)
        assert n == len(w)
        assert L.hb_gaussian_radius(float(sigma)) == (n - 1) // 2
        got = np.frombuffer(buf, dtype=np.float32)[:n]
        # the numpy taps are what the Python layer ships; the C fallback agrees to 1 ulp
        assert np.max(np.abs(got - np.asarray(w, np.float32))) <= 1e-7
    prog = filters.chain(filters.unsharp_program(1.0, 1.5), filters.log_program(2.0))
    m = _native._Marshalled(prog)
    assert L.hb_chain_halo(m.arr, m.n) == 4 + 10 == prog.halo()
    assert L.hb_chain_out_dtype(m.arr, m.n, _native.HB_U16) == _native.HB_F32
    mp = _native._Marshalled(filters.median_program(1))
    assert L.hb_chain_out_dtype(mp.arr, mp.n, _native.HB_U16) == _native.HB_U16
    bad = _native._Marshalled(_native.DeviceProgram([_native.Stage(_native.OP_MEDIAN, radius=0)]))
    assert L.hb_chain_halo(bad.arr, bad.n) == -1


def test_session_and_pinned_are_public_api():
    """session()/pinned() are exported and bind to the declared C symbols."""
    import paper_2511_11890_b200 as hb
    from paper_2511_11890_b200 import _native

    assert callable(hb.session) and callable(hb.pinned)
    assert "hb_session_begin" in _native.EXPORTS and "hb_session_end" in _native.EXPORTS


def test_hb_plan_matches_plan_chunks(golden):
    """hb_plan (the C callers' plan_chunks) against the Python planner and the
    reference's own plans in the golden fixtures (chunking.py:135-174)."""
    from paper_2511_11890_b200.chunking import MemoryBudget, OpProfile, plan_chunks
    from paper_2511_11890_b200.errors import BudgetTooSmallError

    L = _native.load()
    i64 = ctypes.c_int64
    L.hb_plan.argtypes = [i64, i64, i64, ctypes.c_int32, i64, ctypes.c_double, i64,
                          ctypes.c_void_p, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    meta, _ = golden
    cases = [(p["shape"], p["itemsize"], p["halo"], p["scratch"], p["usable"]) for p in meta["plans"]
             if "shape" in p]
    cases += [((100, 1024, 1024), 4, 2, 3, 20 * 2**20), ((37, 5, 7), 2, 3, 8.5, 10**5),
              ((64, 64, 64), 1, 8, 8, 40 * 64 * 64 * 8 + 3), ((1, 1, 1), 4, 0, 2, 8)]
    for shape, item, halo, scratch, usable in cases:
        dt = np.dtype(f"u{item}") if item < 4 else np.dtype(np.float32)
        n, mn = i64(), i64()
        buf = (_native.HbChunk * 4096)()
        rc = L.hb_plan(*shape, item, halo, float(scratch), usable, ctypes.addressof(buf), 4096,
                       ctypes.byref(n), ctypes.byref(mn))
        try:
            plan = plan_chunks(tuple(shape), dt, OpProfile(halo_z=halo, scratch_factor=scratch),
                               MemoryBudget(usable, 1.0))
        except BudgetTooSmallError as e:
            assert rc == 2 and mn.value == e.minimum_bytes  # HB_EBUDGET_SMALL
            continue
        assert rc == 0 and n.value == len(plan.chunks)
        got = [(c.z_start, c.z_stop, c.halo_lo, c.halo_hi) for c in buf[:n.value]]
        assert got == [(c.z_start, c.z_stop, c.halo_lo, c.halo_hi) for c in plan.chunks]
