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
