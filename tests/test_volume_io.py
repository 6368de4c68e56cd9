"""The .vol + .vol.meta format (reference volume.py:28-198) and the
memory-mapped streaming path."""
import numpy as np
import pytest

from paper_2511_11890_b200 import volume as V
from paper_2511_11890_b200.errors import CorruptInputError, UnsupportedFormatError


def test_sidecar_text_matches_reference(golden):
    meta, _ = golden
    for sc in meta["sidecars"]:
        m = V.VolumeMeta(dtype=sc["dtype"], shape=tuple(sc["shape"]), spacing=tuple(sc["spacing"]),
                         description=sc["description"])
        assert m.to_text() == sc["text"]
        back = V.VolumeMeta.from_text(sc["text"])
        assert back.shape == tuple(sc["shape"]) and back.dtype == sc["dtype"]


def test_roundtrip_and_mmap(tmp_path, rng):
    data = rng.integers(0, 65535, size=(9, 10, 11), dtype=np.uint16)
    p = tmp_path / "a.vol"
    V.save_volume(V.Volume(data, spacing=(2.0, 1.0, 0.5), description="x"), p)
    v = V.load_volume(p)
    assert isinstance(v.data, np.memmap)
    np.testing.assert_array_equal(v.data, data)
    assert v.spacing == (2.0, 1.0, 0.5) and v.description == "x"
    r = V.load_volume(p, mmap=False)
    np.testing.assert_array_equal(r.data, data)


def test_corrupt_and_unsupported(tmp_path):
    p = tmp_path / "b.vol"
    V.save_volume(V.Volume(np.zeros((2, 3, 4), np.float32)), p)
    with open(p, "ab") as fh:
        fh.write(b"\0")
    with pytest.raises(CorruptInputError):
        V.load_volume(p)
    with pytest.raises(UnsupportedFormatError):
        V.VolumeMeta.from_text("dtype: int64\nshape: 1 1 1\nspacing: 1 1 1\n")
    with pytest.raises(UnsupportedFormatError):
        V.Volume(np.zeros((2, 2, 2), np.float64))


@pytest.mark.gpu
def test_filter_file_streams_through_the_executor(tmp_path, oracle):
    from paper_2511_11890_b200.chunking import MemoryBudget

    rng = np.random.default_rng(3)
    data = rng.random((40, 64, 96), dtype=np.float32)
    src, dst = tmp_path / "in.vol", tmp_path / "out.vol"
    V.save_volume(V.Volume(data), src)
    rep = V.filter_file(src, dst, "median", {"radius": 1}, MemoryBudget(12 * 64 * 96 * 4 * 4, 1.0))
    assert rep.chunk_count > 1
    out = V.load_volume(dst)
    assert out.dtype == np.float32
    np.testing.assert_array_equal(out.data, oracle.median(data, 1))
