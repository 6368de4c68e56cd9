"""Seeded shape fuzz of the round-2 kernels against the CPU oracle (test
infrastructure): random extents around every tile / chunk boundary the
kernels have — k_gauss_tri (planes >= 384^2, 48x32 tiles, capped z-chunks),
the small-plane split passes (gauss_small.cu), k_median3_f32 (64x8 tiles,
TMA box at x0-4), k_morph_bits2 (64-row x 256-voxel tiles, halo words), the
register-streaming grey u16 k_morph_u16s (128 x 32 tiles, nx % 8 == 0) and
the two-rows-per-thread grey k_morph3 (other widths), and the 5x5x5
k_median5_net — through the public API (chunked,
halos), bit-exact where the operator is exact, <= 1e-5 otherwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5


def _rel(got, ref):
    return float(np.max(np.abs(got.astype(np.float64) - ref)) / max(1e-30, float(np.max(np.abs(ref)))))


@pytest.mark.parametrize("case", range(16))
def test_fuzz_small_plane_gaussian_and_median(oracle, case):
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(1000 + case)
    nz = int(rng.integers(1, 40))
    ny = int(rng.integers(9, 300))
    nx = 4 * int(rng.integers(3, 80))  # nx % 4 == 0 keeps the TMA kernels in play
    x = (rng.random((nz, ny, nx), dtype=np.float32) - 0.3).astype(np.float32)
    g = filters.gaussian(x, 2.0)
    assert _rel(g, oracle.gaussian(x, 2.0)) <= FLOAT_TOL, (nz, ny, nx)
    m = filters.median(x, 1)
    assert np.array_equal(m, oracle.median(x, 1)), (nz, ny, nx)


@pytest.mark.parametrize("case", range(4))
def test_fuzz_large_plane_gaussian(oracle, case):
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(2000 + case)
    nz = int(rng.integers(1, 24))
    ny = int(rng.integers(384, 460))
    nx = 2 * int(rng.integers(192, 240))  # even: k_gauss_tri's column pairs
    x = rng.random((nz, ny, nx), dtype=np.float32)
    g = filters.gaussian(x, 2.0)
    assert _rel(g, oracle.gaussian(x, 2.0)) <= FLOAT_TOL, (nz, ny, nx)
    u = filters.unsharp(x, 2.0, 1.5)
    assert _rel(u, oracle.unsharp(x, 2.0, 1.5)) <= FLOAT_TOL, (nz, ny, nx)


@pytest.mark.parametrize("case", range(12))
def test_fuzz_morphology(oracle, case):
    from paper_2511_11890_b200 import morphology

    rng = np.random.default_rng(3000 + case)
    nz = int(rng.integers(1, 20))
    ny = int(rng.integers(5, 150))
    nx = 32 * int(rng.integers(1, 12))  # whole words: k_morph_bits2 runs on binary data
    spec = ["ball:3", "ball:2", "box:1", "cross:3", "ball:1", "box:2"][case % 6]
    se = morphology.StructuringElement.parse(spec)
    b = (rng.random((nz, ny, nx)) < 0.55).astype(np.uint8)
    assert np.array_equal(morphology.erode(b, se), oracle.erode(b, se.offsets)), (spec, b.shape)
    assert np.array_equal(morphology.dilate(b, se), oracle.dilate(b, se.reflect().offsets)), (spec, b.shape)
    g = rng.integers(0, 65536, size=(nz, ny, nx + 4)).astype(np.uint16)  # k_morph3
    assert np.array_equal(morphology.erode(g, se), oracle.erode(g, se.offsets)), (spec, g.shape)
    gb = rng.integers(0, 256, size=(nz, ny, nx)).astype(np.uint8)  # grey u8: bits2 flags it, k_morph_u16s<u8>
    assert np.array_equal(morphology.erode(gb, se), oracle.erode(gb, se.offsets)), (spec, gb.shape)
    assert np.array_equal(morphology.dilate(gb, se), oracle.dilate(gb, se.reflect().offsets)), (spec, gb.shape)
    nx8 = 8 * int(rng.integers(1, 70))  # k_morph_u16s: ragged 128-column tiles
    g = rng.integers(0, 65536, size=(nz, ny, nx8)).astype(np.uint16)
    assert np.array_equal(morphology.erode(g, se), oracle.erode(g, se.offsets)), (spec, g.shape)
    assert np.array_equal(morphology.dilate(g, se), oracle.dilate(g, se.reflect().offsets)), (spec, g.shape)


@pytest.mark.parametrize("case", range(10))
def test_fuzz_median5(oracle, case):
    """k_median5_net: ragged columns (128-thread CTAs over y*x), z-chunks of any
    parity, tiny planes; f32 with repeats and signed zeros, packed u16 / u8."""
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(5000 + case)
    shape = (int(rng.integers(1, 24)), int(rng.integers(1, 60)), int(rng.integers(1, 140)))
    dt = [np.float32, np.uint16, np.uint8][case % 3]
    if dt == np.float32:
        x = (rng.random(shape, dtype=np.float32) - 0.5).astype(np.float32)
        x[rng.random(shape) < 0.1] = 0.25
        x[rng.random(shape) < 0.05] = -0.0
        x[rng.random(shape) < 0.05] = 0.0
    else:
        x = rng.integers(0, np.iinfo(dt).max, size=shape).astype(dt)
    assert np.array_equal(filters.median(x, 2), oracle.median(x, 2)), (shape, dt)


@pytest.mark.parametrize("shape", [(300, 6, 40), (97, 3, 17), (131, 33, 8)])
def test_median5_many_z_chunks(oracle, shape):
    """Small planes make k_median5_net split z into many 16-slice chunks (odd
    and even lengths, a ragged last chunk): every chunk's 4-plane prologue and
    the pair stepping across chunk ends must reproduce the oracle."""
    from paper_2511_11890_b200 import filters

    rng = np.random.default_rng(sum(shape))
    x = (rng.random(shape, dtype=np.float32) - 0.5).astype(np.float32)
    x[rng.random(shape) < 0.1] = 0.125
    assert np.array_equal(filters.median(x, 2), oracle.median(x, 2)), shape
    u = rng.integers(0, 65536, size=shape).astype(np.uint16)
    assert np.array_equal(filters.median(u, 2), oracle.median(u, 2)), shape


@pytest.mark.parametrize("spec", ["ball:3", "box:1", "cross:2"])
def test_morph_u16s_many_z_chunks(oracle, spec):
    """k_morph_u16s on a small plane: z split into several chunks (the
    accumulator ring restarts per chunk) with a ragged tail."""
    from paper_2511_11890_b200 import morphology

    rng = np.random.default_rng(77)
    g = rng.integers(0, 65536, size=(101, 40, 64)).astype(np.uint16)
    se = morphology.StructuringElement.parse(spec)
    assert np.array_equal(morphology.erode(g, se), oracle.erode(g, se.offsets)), spec
    assert np.array_equal(morphology.dilate(g, se), oracle.dilate(g, se.reflect().offsets)), spec
