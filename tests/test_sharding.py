"""Multi-process (gloo, world_size 2 and 3) tests of the z-slab sharding path:
halo exchange over torch.distributed P2P and stitching must reproduce the
single-volume result exactly.  The per-block compute is the CPU oracle here
(test infrastructure), so the exchange/stitch logic is verified without a GPU;
on B200 the same code runs over NCCL with the device kernels."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_apply(block, prog, z_begin, out):
    """apply_block for the CPU test: the oracle evaluates every stage on the
    padded block (clamp at its faces) and writes block slices
    [z_begin, z_begin + len(out)) into ``out``."""
    out.copy_(_oracle_eval(block, prog, z_begin, out.shape[0]))


def _oracle_eval(block, prog, z_begin, nz_out):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2511_11890_b200 import _native

    x = block.numpy()
    for st in prog.stages:
        if st.op == _native.OP_MEDIAN:
            x = O.median(x, st.radius)
        elif st.op == _native.OP_GAUSSIAN:
            x = O.gaussian(x, st.sigma)
        elif st.op == _native.OP_UNSHARP:
            x = O.unsharp(x, st.sigma, st.amount)
        elif st.op == _native.OP_LOG:
            x = O.log(x, st.sigma)
        elif st.op == _native.OP_ERODE:
            x = O.erode(x, st.offsets)
        elif st.op == _native.OP_DILATE:
            x = O.dilate(x, st.offsets)
        else:
            raise AssertionError(st.op)
    return torch.from_numpy(np.ascontiguousarray(x[z_begin:z_begin + nz_out]))


def _volume(kind):
    rng = np.random.default_rng(99)
    if kind == "f32":
        return rng.random((36, 12, 14), dtype=np.float32)
    if kind == "u16":
        return rng.integers(0, 65536, size=(29, 12, 14), dtype=np.uint16)
    return (rng.random((29, 12, 14)) < 0.5).astype(np.uint8)


def _program(name):
    sys.path.insert(0, ROOT)
    from paper_2511_11890_b200 import filters, morphology

    if name == "median":
        return filters.median_program(1), "u16"
    if name == "gauss_exact":
        return filters.gaussian_program(1.5, "exact"), "f32"
    if name == "unsharp_log":
        return filters.chain(filters.unsharp_program(1.0, 1.5, "exact"), filters.log_program(1.0)), "f32"
    if name == "open_ball1":
        return morphology.morph_program("open", morphology.StructuringElement.ball(1)), "bin"
    raise KeyError(name)


def _worker(rank, world, port, name, per_stage, outdir, piece=None):
    sys.path.insert(0, ROOT)
    from paper_2511_11890_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        prog, kind = _program(name)
        vol = _volume(kind)
        slabs = sharding.partition(vol.shape[0], world)
        me = slabs[rank]
        local = torch.from_numpy(np.ascontiguousarray(vol[me.z0:me.z1]))
        out = sharding.run_sharded(local, prog, rank, world, apply_block=_oracle_apply,
                                   per_stage=per_stage, piece_slices=piece)
        np.save(os.path.join(outdir, f"r{rank}.npy"), out.numpy())
    finally:
        dist.destroy_process_group()


CASES = [("median", True), ("gauss_exact", True), ("unsharp_log", True),
         ("unsharp_log", False), ("open_ball1", True)]


@pytest.mark.parametrize("name,per_stage", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_whole(name, per_stage, world, oracle):
    prog, kind = _program(name)
    vol = _volume(kind)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), name, per_stage, d), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)])
    whole = _oracle_eval(torch.from_numpy(vol), prog, 0, vol.shape[0]).numpy()
    assert got.dtype == whole.dtype
    assert np.array_equal(got, whole)


def test_sharded_small_pieces_equal_whole(oracle):
    """interior-first schedule with 2-slice compute pieces (many clipped blocks)."""
    prog, kind = _program("unsharp_log")
    vol = _volume(kind)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), "unsharp_log", True, d, 2), nprocs=2, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"r{r}.npy")) for r in range(2)])
    whole = _oracle_eval(torch.from_numpy(vol), prog, 0, vol.shape[0]).numpy()
    assert np.array_equal(got, whole)


def _thin_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    from paper_2511_11890_b200 import filters, sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        vol = np.zeros((10, 4, 4), np.float32)
        me = sharding.partition(10, world)[rank]  # 3, 3, 2, 2 slices
        local = torch.from_numpy(np.ascontiguousarray(vol[me.z0:me.z1]))
        try:
            sharding.run_sharded(local, filters.median_program(3), rank, world,
                                 apply_block=_oracle_apply)
            msg = "no error"
        except ValueError as exc:
            msg = str(exc)
        with open(os.path.join(outdir, f"e{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


def test_thin_slab_fails_on_every_rank():
    """A slab thinner than the halo raises on ALL ranks before any P2P op
    (no rank is left waiting in the exchange)."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_thin_worker, args=(4, _free_port(), d), nprocs=4, join=True)
        msgs = [open(os.path.join(d, f"e{r}.txt")).read() for r in range(4)]
    assert all("thinner than the halo" in m for m in msgs), msgs


def test_partition():
    sys.path.insert(0, ROOT)
    from paper_2511_11890_b200 import sharding

    slabs = sharding.partition(10, 3)
    assert [(s.z0, s.z1) for s in slabs] == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        sharding.partition(2, 3)


def _otsu_worker(rank, world, port, kind, outdir):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2511_11890_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        vol = _volume(kind)
        if kind == "f32":
            vol = vol * 7.0 - 2.0
        me = sharding.partition(vol.shape[0], world)[rank]
        local = np.ascontiguousarray(vol[me.z0:me.z1])
        labels, t = sharding.otsu_sharded(
            local, 64, rank, world,
            minmax_fn=lambda a: (float(a.min()), float(a.max())),
            hist_fn=lambda a, b, r: O.histogram(a, b, r),
            apply_fn=lambda a, tt: O.apply_threshold(a, tt))
        np.save(os.path.join(outdir, f"otsu{rank}.npy"), labels)
        np.save(os.path.join(outdir, f"t{rank}.npy"), np.array([t]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["f32", "u16"])
def test_otsu_sharded_equals_whole(kind, oracle):
    """Pass 1 all-reduces the range and the int64 histogram across ranks; the
    stitched labels and the threshold equal the single-volume Otsu."""
    world = 2
    vol = _volume(kind)
    if kind == "f32":
        vol = vol * 7.0 - 2.0
    t_whole = oracle.otsu(vol, 64)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_otsu_worker, args=(world, _free_port(), kind, d), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"otsu{r}.npy")) for r in range(world)])
        ts = [float(np.load(os.path.join(d, f"t{r}.npy"))[0]) for r in range(world)]
    assert ts == [t_whole] * world
    assert np.array_equal(got, oracle.apply_threshold(vol, t_whole))


def _cc_worker(rank, world, port, conn, outdir):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2511_11890_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        vol = (np.random.default_rng(31).random((23, 17, 19)) < 0.35).astype(np.uint8)
        me = sharding.partition(vol.shape[0], world)[rank]
        local = np.ascontiguousarray(vol[me.z0:me.z1])
        labels, total = sharding.connected_components_sharded(
            local, conn, rank, world, label_fn=lambda a, c: O.connected_components(a, c))
        np.save(os.path.join(outdir, f"cc{rank}.npy"), labels)
        np.save(os.path.join(outdir, f"n{rank}.npy"), np.array([total]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,conn", [(2, 6), (3, 26), (3, 6)])
def test_connected_components_sharded_equals_whole(world, conn, oracle):
    """Ranks label their z-slabs, all_gather counts and boundary planes, and
    run the same boundary union-find: the stitched labels are the canonical
    single-volume labels (first-voxel scan order), bit for bit."""
    vol = (np.random.default_rng(31).random((23, 17, 19)) < 0.35).astype(np.uint8)
    want, n = oracle.connected_components(vol, conn)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_cc_worker, args=(world, _free_port(), conn, d), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"cc{r}.npy")) for r in range(world)])
        ns = [int(np.load(os.path.join(d, f"n{r}.npy"))[0]) for r in range(world)]
    assert ns == [n] * world
    assert np.array_equal(got.astype(np.uint32), want)
