"""Config-scale parity gate: every BASELINE.json config checked against the CPU
oracle on the SAME launch paths and shapes ``bench.py`` times.

The bench applies device programs to device-resident padded blocks
(``_native.apply_device(x, out, program, halo)``), so these tests do exactly
that at the configs' full sizes and compare either the whole output (256^3)
or sampled output slices (1024^3, 2048^3).  Slab sampling is exact by plan
invariance (reference chunking.py:135-174): an output slice
depends only on the ``halo`` block slices either side of it, with clamping at
the block faces, so the oracle evaluates just that padded slab.

Bars (north star): median / morphology bit-exact; float32 stencils
max|gpu-ref|/max|ref| <= 1e-5; exact-mode Gaussian / LoG bit-exact.
"""
import numpy as np
import pytest

from conftest import float_close

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    from paper_2511_11890_b200 import _native

    assert _native.device_count() >= 1, "no CUDA device: the GPU tests need a B200"
    return torch


def _apply(torch, x, program, halo, nz_out=None):
    from paper_2511_11890_b200 import _native

    nz_out = x.shape[0] - 2 * halo if nz_out is None else nz_out
    out_dt = program.out_dtype(np.dtype(str(x.dtype).replace("torch.", "")))
    out = torch.empty((nz_out,) + tuple(x.shape[1:]), device=x.device,
                      dtype=getattr(torch, out_dt.name))
    n = _native.apply_device(x, out, program, halo)
    torch.cuda.synchronize()
    assert n >= 1
    return out


def _slab_check(x, out, halo, zs, ref_fn, exact, tol=FLOAT_TOL):
    """Compare output slices ``zs`` with ``ref_fn`` applied to the padded slab
    of block slices [z, z + 2*halo] (output slice z = block slice z + halo)."""
    nzb = x.shape[0]
    for z in zs:
        lo, hi = max(0, z), min(nzb, z + 2 * halo + 1)
        slab = x[lo:hi].cpu().numpy()
        ref = ref_fn(slab)[z + halo - lo]
        got = out[z].cpu().numpy()
        if exact:
            assert got.dtype == ref.dtype and np.array_equal(got, ref), f"slice {z}"
        else:
            assert float_close(got, ref) <= tol, (z, float_close(got, ref))


# --------------------------------------------------------------------------
# configs[0]: gaussian sigma=2 on 256^3 f32, single chunk — the whole volume
# (k_gauss_p2 with its z-split: 64 XY tiles over 296 CTA slots)
# --------------------------------------------------------------------------
def test_c0_gaussian_256_full(torch_dev, oracle):
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((256 + 16, 256, 256), generator=g, device="cuda")
    xh = x.cpu().numpy()
    ref = oracle.gaussian(xh, 2.0)[8:-8]
    fast = _apply(torch, x, filters.gaussian_program(2.0, "fast"), 8).cpu().numpy()
    assert float_close(fast, ref) <= FLOAT_TOL
    exact = _apply(torch, x, filters.gaussian_program(2.0, "exact"), 8).cpu().numpy()
    assert np.array_equal(exact, ref)


@pytest.mark.parametrize("shape", [(96 + 16, 200, 328), (130 + 16, 64, 96), (300, 48, 64)])
def test_gaussian_zsplit_vs_oracle(torch_dev, oracle, shape):
    """nzo >= 96 on few XY tiles: the z-split of k_gauss_p2 / k_exact_z2
    (several CTAs per column, each priming 2R slices) against the oracle."""
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    rng = np.random.default_rng(sum(shape))
    xh = rng.random(shape, dtype=np.float32)
    x = torch.from_numpy(xh).cuda()
    ref = oracle.gaussian(xh, 2.0)[8:-8]
    fast = _apply(torch, x, filters.gaussian_program(2.0, "fast"), 8).cpu().numpy()
    assert float_close(fast, ref) <= FLOAT_TOL
    exact = _apply(torch, x, filters.gaussian_program(2.0, "exact"), 8).cpu().numpy()
    assert np.array_equal(exact, ref)
    # unsharp through the same kernel's epilogue
    refu = oracle.unsharp(xh, 2.0, 1.5)[8:-8]
    u = _apply(torch, x, filters.unsharp_program(2.0, 1.5, "fast"), 8).cpu().numpy()
    assert float_close(u, refu) <= FLOAT_TOL


def test_gaussian_tri_ragged_vs_oracle(torch_dev, oracle):
    """k_gauss_tri (sigma = 2 on planes >= 384^2): ragged x / y tiles (406 =
    8 x 48 + 22, 398 = 12 x 32 + 14), several capped z-chunks (nzo = 230 >
    192) and the unsharp epilogue, against the oracle."""
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    rng = np.random.default_rng(406)
    xh = rng.random((230 + 16, 398, 406), dtype=np.float32)
    x = torch.from_numpy(xh).cuda()
    ref = oracle.gaussian(xh, 2.0)[8:-8]
    fast = _apply(torch, x, filters.gaussian_program(2.0, "fast"), 8).cpu().numpy()
    assert float_close(fast, ref) <= FLOAT_TOL
    refu = oracle.unsharp(xh, 2.0, 1.5)[8:-8]
    u = _apply(torch, x, filters.unsharp_program(2.0, 1.5, "fast"), 8).cpu().numpy()
    assert float_close(u, refu) <= FLOAT_TOL


@pytest.mark.parametrize("sigma", [2.5, 3.3])
def test_gaussian_large_sigma_vs_oracle(torch_dev, oracle, sigma):
    """R = ceil(4 sigma) > 8: the generic separable path, fast and exact."""
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    R = filters.gaussian_kernel_radius(sigma)
    rng = np.random.default_rng(int(sigma * 10))
    xh = rng.random((40 + 2 * R, 70, 133), dtype=np.float32)
    x = torch.from_numpy(xh).cuda()
    ref = oracle.gaussian(xh, sigma)[R:-R]
    fast = _apply(torch, x, filters.gaussian_program(sigma, "fast"), R).cpu().numpy()
    assert float_close(fast, ref) <= FLOAT_TOL
    exact = _apply(torch, x, filters.gaussian_program(sigma, "exact"), R).cpu().numpy()
    assert np.array_equal(exact, ref)
    # and through the public chunked API (several chunks)
    got = filters.gaussian(xh[:30], sigma)
    assert float_close(got, oracle.gaussian(xh[:30], sigma)) <= FLOAT_TOL


# --------------------------------------------------------------------------
# configs[1] / bench headline: median r=1, mean r=1, gaussian sigma=2 on 1024^3
# --------------------------------------------------------------------------
def test_c1_1024_median_mean_gaussian_sampled(torch_dev, oracle):
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    n = 1024
    g = torch.Generator(device="cuda").manual_seed(1000)
    x = torch.rand((n + 2, n, n), generator=g, device="cuda")
    zs = (0, 1, 2, 511, 777, n - 2, n - 1)
    out = _apply(torch, x, filters.median_program(1), 1)
    _slab_check(x, out, 1, zs, lambda s: oracle.median(s, 1), exact=True)
    out = _apply(torch, x, filters.mean_program(1), 1)
    _slab_check(x, out, 1, zs, lambda s: oracle.mean(s, 1), exact=False)
    del out, x
    x = torch.rand((n + 16, n, n), generator=g, device="cuda")
    zs = (0, 7, 8, 300, n - 9, n - 1)
    out = _apply(torch, x, filters.gaussian_program(2.0, "fast"), 8)
    _slab_check(x, out, 8, zs, lambda s: oracle.gaussian(s, 2.0), exact=False)
    out = _apply(torch, x, filters.gaussian_program(2.0, "exact"), 8)
    _slab_check(x, out, 8, zs[:3], lambda s: oracle.gaussian(s, 2.0), exact=True)
    del out, x
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# the 5x5x5 median (north star's "3x3x3/5x5x5 median") on the bench's
# 1024^2 x 256 block: k_median5_net's z-chunks, slab-sampled, bit-exact
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dt", ["f32", "u16"])
def test_median5_1024_sampled(torch_dev, oracle, dt):
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    g = torch.Generator(device="cuda").manual_seed(55)
    if dt == "f32":
        x = torch.rand((260, 1024, 1024), generator=g, device="cuda")
    else:
        x = torch.randint(0, 65536, (260, 1024, 1024), generator=g, device="cuda",
                          dtype=torch.int32).to(torch.uint16)
    out = _apply(torch, x, filters.median_program(2), 2)
    _slab_check(x, out, 2, (0, 1, 2, 127, 128, 254, 255), lambda s: oracle.median(s, 2), exact=True)
    del out, x
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# configs[2]: erode / dilate ball:3 on 2048^3 u16 and binary u8 (> 2^31 voxels)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dt", ["u16", "bin"])
def test_c2_2048_morph_ball3_sampled(torch_dev, oracle, dt):
    from paper_2511_11890_b200 import morphology

    torch = torch_dev
    n = 2048
    g = torch.Generator(device="cuda").manual_seed(7)
    if dt == "u16":
        x = torch.randint(0, 65536, (n + 6, n, n), generator=g, device="cuda",
                          dtype=torch.int32).to(torch.uint16)
    else:
        x = (torch.rand((n + 6, n, n), generator=g, device="cuda") < 0.5).to(torch.uint8)
    assert x.numel() > 2 ** 33
    ball = morphology.StructuringElement.ball(3)
    zs = (0, 2, 1031, n - 3, n - 1)  # the last slices sit beyond 2^33 voxels
    for op, ref in (("erode", oracle.erode), ("dilate", oracle.dilate)):
        out = _apply(torch, x, morphology.morph_program(op, ball), 3)
        _slab_check(x, out, 3, zs, lambda s: ref(s, ball.offsets), exact=True)
        del out
    del x
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# configs[3]: unsharp(sigma=1, a=1.5) -> LoG(sigma=2) on a 2048^2 slab
# --------------------------------------------------------------------------
def test_c3_unsharp_log_chain_2048_slab(torch_dev, oracle):
    from paper_2511_11890_b200 import filters

    torch = torch_dev
    n, nz, h = 2048, 12, 14
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((nz + 2 * h, n, n), generator=g, device="cuda")
    xh = x.cpu().numpy()
    # exact unsharp -> LoG: bit-exact against the stage-by-stage oracle
    chain = filters.chain(filters.unsharp_program(1.0, 1.5, "exact"), filters.log_program(2.0))
    got = _apply(torch, x, chain, h).cpu().numpy()
    ref = oracle.log(oracle.unsharp(xh, 1.0, 1.5), 2.0)[h:-h]
    assert np.array_equal(got, ref)
    # the bench's chain (fast unsharp, exact LoG): norm-relative
    chain = filters.chain(filters.unsharp_program(1.0, 1.5), filters.log_program(2.0))
    got = _apply(torch, x, chain, h).cpu().numpy()
    assert float_close(got, ref) <= FLOAT_TOL
