"""Multi-device paths on the B200 (one GPU here, so several z-slabs share it):

* ``sharding.run_sharded_local`` — virtual ranks in one process, per-stage
  ghost exchange device-to-device, the interior/boundary split and the
  clipped per-piece blocks exactly as a torchrun job runs them — must equal
  the single-volume device result bit for bit (plan invariance,
  chunking.py:135-174);
* ``sharding.run_sharded`` at world 1 on device-resident data;
* ``hb_run_multi`` (the C-ABI ndev/devices[] executor) with devices [0, 0];
* library-pool slab buffers: reported by hb_device_pool_bytes, released.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    from paper_2511_11890_b200 import _native

    assert _native.device_count() >= 1, "no CUDA device: the GPU tests need a B200"
    return torch


def _programs():
    from paper_2511_11890_b200 import filters, morphology

    return {
        "median": (filters.median_program(1), "f32"),
        "gauss_fast": (filters.gaussian_program(2.0, "fast"), "f32"),
        "unsharp_log": (filters.chain(filters.unsharp_program(1.0, 1.5), filters.log_program(2.0)), "f32"),
        "erode_ball3_u16": (morphology.morph_program("erode", morphology.StructuringElement.ball(3)), "u16"),
        "open_ball1_u8": (morphology.morph_program("open", morphology.StructuringElement.ball(1)), "u8"),
    }


def _whole(torch, x, prog):
    from paper_2511_11890_b200 import _native

    out_dt = prog.out_dtype(np.dtype(str(x.dtype).replace("torch.", "")))
    out = torch.empty(x.shape, device=x.device, dtype=getattr(torch, out_dt.name))
    _native.apply_device(x, out, prog, 0)
    torch.cuda.synchronize()
    return out


def _vol(torch, kind, shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "f32":
        return torch.rand(shape, generator=g, device="cuda")
    if kind == "u16":
        return torch.randint(0, 65536, shape, generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
    return (torch.rand(shape, generator=g, device="cuda") < 0.5).to(torch.uint8)


@pytest.mark.parametrize("name", ["median", "gauss_fast", "unsharp_log", "erode_ball3_u16",
                                  "open_ball1_u8"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_virtual_ranks_equal_whole(torch_dev, name, world):
    from paper_2511_11890_b200 import sharding

    torch = torch_dev
    prog, kind = _programs()[name]
    x = _vol(torch, kind, (70, 96, 160), world)
    want = _whole(torch, x, prog)
    parts = [x[s.z0:s.z1].contiguous() for s in sharding.partition(x.shape[0], world)]
    for per_stage in (True, False):
        outs = sharding.run_sharded_local(parts, prog, per_stage=per_stage, piece_slices=5)
        got = torch.cat([o for o in outs])
        torch.cuda.synchronize()
        assert got.dtype == want.dtype and torch.equal(got, want), (name, world, per_stage)


def test_run_sharded_world1_device(torch_dev):
    from paper_2511_11890_b200 import filters, sharding

    torch = torch_dev
    prog = filters.chain(filters.unsharp_program(1.0, 1.5), filters.log_program(2.0))
    x = _vol(torch, "f32", (40, 130, 260), 1)
    got = sharding.run_sharded(x, prog, 0, 1, piece_slices=7)
    torch.cuda.synchronize()
    assert torch.equal(got, _whole(torch, x, prog))


def test_pool_buffers_are_library_memory(torch_dev):
    from paper_2511_11890_b200 import _native

    torch = torch_dev
    _native.trim_device(0)
    base = _native.device_pool_bytes(0)
    buf = _native.DeviceBuffer((64, 256, 256), np.float32, 0)
    t = buf.tensor()
    t.fill_(2.0)
    assert float(t.sum()) == 2.0 * t.numel()
    assert _native.device_pool_bytes(0) >= base + 64 * 256 * 256 * 4
    del t
    buf.free()
    torch.cuda.synchronize()
    _native.trim_device(0)
    assert _native.device_pool_bytes(0) == 0


def test_run_multi_devices_equal_single(torch_dev):
    """hb_run_multi: chunk groups streamed by one host thread per listed
    device (here [0, 0]) — same output as hb_run, global failed-chunk index."""
    from paper_2511_11890_b200 import _native, filters
    from paper_2511_11890_b200.chunking import MemoryBudget, OpProfile, plan_chunks
    from paper_2511_11890_b200.errors import ChunkExecutionError

    x = np.random.default_rng(4).random((90, 64, 96), dtype=np.float32)
    prog = filters.chain(filters.gaussian_program(2.0), filters.median_program(1))
    plan = plan_chunks(x.shape, x.dtype, OpProfile(halo_z=9, scratch_factor=4),
                       MemoryBudget(40 * 64 * 96 * 4 * 4, 1.0))
    chunks = [c.as_native() for c in plan.chunks]
    assert len(chunks) >= 4
    a = np.empty_like(x)
    b = np.empty_like(x)
    ra = _native.run_host(x, a, prog, chunks, device=0)
    rb = _native.run_host(x, b, prog, chunks, devices=[0, 0])
    assert np.array_equal(a, b)
    assert rb.chunk_count == ra.chunk_count and rb.device_residual_bytes == 0
    assert rb.d2h_bytes == x.nbytes
    with pytest.raises(ChunkExecutionError) as ei:
        _native.run_host(x, b, prog, chunks, devices=[0, 0], fault_chunk=len(chunks) - 1)
    assert ei.value.chunk_index == len(chunks) - 1
