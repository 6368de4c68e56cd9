"""Z-slab data parallelism across GPUs with neighbour-only halo exchange.

The reference runs one process and one device (chunks execute
sequentially, chunking.py:244).  Every hot-path operator is local with a
finite Z dependence radius (OpProfile.halo_z, chunking.py:75-79), so a volume
partitioned into contiguous z-slabs — one per rank — is processed
independently once each rank holds `halo` ghost slices from its neighbours;
plan invariance makes the stitched result identical to the
single-device one.

Two ways to obtain the ghost slices:

* host-resident input (``registry.run_operator`` per rank): each rank simply
  reads its padded range — no collective at all;
* device-resident, already-sharded input (this module): one
  ``send/recv`` pair per neighbour and per chained stage over NCCL
  (NVLink/NVSwitch), i.e. halo slices of stage ``s`` output feed stage ``s+1``.

One process per GPU; ``torch.distributed`` provides the plumbing (``nccl`` on
B200, ``gloo`` in the CPU tests).  Per stage the exchange is posted first and
the slices that need no ghost data are computed while it is in flight; the
boundary slices follow once the ghosts land.  Slabs live in padded buffers
[ghost_lo | interior | ghost_hi] from the library's device pool, so ghosts
are received in place and each stage writes the next stage's interior.  The
per-block compute is injected (``apply_block``) so the exchange/stitching
logic is testable without a GPU; the default is the device path
(``_native.apply_device``).  ``run_sharded_local`` runs the same schedule for
several slabs held by one process (virtual ranks; tested on one B200).
"""

from __future__ import annotations

from dataclasses import dataclass
import time
from typing import Callable, Optional, Sequence

import numpy as np


@dataclass(frozen=True)
class Slab:
    """Interior z-range [z0, z1) owned by one rank."""

    rank: int
    z0: int
    z1: int

    @property
    def size(self) -> int:
        return self.z1 - self.z0


def partition(nz: int, world: int) -> list:
    """Contiguous balanced z-slabs (sizes differ by at most one slice)."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} slices over {world} ranks")
    base, extra = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(Slab(r, z, z + n))
        z += n
    return out


def _dist():
    import torch.distributed as dist

    return dist


# ---------------------------------------------------------------------------
# Padded slab buffers: [ghost_lo | interior | ghost_hi] in ONE contiguous
# (lo + n + hi, Y, X) buffer, so received halo slices land in place (no
# torch.cat) and a stage's output is written straight into the interior of
# the next stage's buffer.  On the device the buffer comes from the library's
# private pool (hb_device_alloc), never from PyTorch's caching allocator.
# ---------------------------------------------------------------------------
def _empty(shape, dtype, like):
    import torch

    if like.device.type == "cuda":
        from . import _native

        np_dt = np.dtype(str(dtype).replace("torch.", ""))
        return _native.device_empty(shape, np_dt, like.device.index or 0)
    return torch.empty(shape, dtype=dtype, device=like.device)


@dataclass
class PaddedSlab:
    buf: object   # (lo + n + hi, Y, X) tensor
    lo: int       # ghost slices below (received from rank - 1)
    hi: int       # ghost slices above (received from rank + 1)

    @property
    def n(self) -> int:
        return self.buf.shape[0] - self.lo - self.hi

    @property
    def interior(self):
        return self.buf[self.lo:self.lo + self.n]


def alloc_padded(n: int, plane: tuple, dtype, like, lo: int, hi: int) -> PaddedSlab:
    return PaddedSlab(_empty((lo + n + hi,) + tuple(plane), dtype, like), lo, hi)


class DistTransport:
    """Neighbour halo exchange over torch.distributed P2P (NCCL over
    NVLink/NVSwitch on the B200 box — one ncclSend/ncclRecv pair per face,
    batched; gloo in the CPU tests).  ``start`` posts the sends of this
    rank's first/last ``h`` interior slices and the receives into its ghost
    slices and returns at once; ``finish`` makes the compute stream (NCCL) or
    the host (gloo) wait for them."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def start(self, slab: PaddedSlab, h: int):
        dist = _dist()
        ops, r, g = [], self.rank, self.group
        if h == 0 or self.world == 1:
            return []
        inner = slab.interior
        if r > 0:
            ops.append(dist.P2POp(dist.irecv, slab.buf[slab.lo - h:slab.lo], r - 1, g))
            ops.append(dist.P2POp(dist.isend, inner[:h], r - 1, g))
        if r < self.world - 1:
            ops.append(dist.P2POp(dist.isend, inner[inner.shape[0] - h:], r + 1, g))
            ops.append(dist.P2POp(dist.irecv, slab.buf[slab.lo + slab.n:slab.lo + slab.n + h], r + 1, g))
        return dist.batch_isend_irecv(ops)

    def finish(self, pending) -> None:
        for req in pending:
            req.wait()

    def min_slab(self, n: int, like) -> int:
        """Smallest slab over all ranks (every rank must hold >= halo slices
        for its neighbours' ghosts; checked collectively before any P2P op)."""
        import torch

        if self.world == 1:
            return n
        dist = _dist()
        dev = _comm_device(self.group)
        t = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item())


def _device_apply(block, program, z_begin: int, out) -> None:
    """Apply ``program`` to device ``block`` (clamp at its faces), writing
    block slices [z_begin, z_begin + len(out)) into ``out``."""
    from . import _native

    _native.apply_device(block, out, program, z_begin)


def _pieces(a: int, b: int, step: int):
    z = a
    while z < b:
        yield z, min(b, z + step)
        z += step


def _apply_range(src: PaddedSlab, a: int, b: int, h: int, program, dst, apply_block,
                 piece: int) -> None:
    """Outputs for interior slices [a, b) of ``src`` into dst[a:b], in z-pieces
    of <= ``piece`` slices (bounded device scratch).  Each piece's block is the
    padded buffer's [a - h, b + h) clipped to what the buffer holds; faces of a
    clipped block are real volume faces, where the operator clamps exactly as
    the reference does."""
    P = src.buf.shape[0]
    for pa, pb in _pieces(a, b, piece):
        b0 = max(0, src.lo + pa - h)
        b1 = min(P, src.lo + pb + h)
        apply_block(src.buf[b0:b1], program, src.lo + pa - b0, dst[pa:pb])


def run_sharded(local, program, rank: int, world: int, group=None,  # local: tensor | PaddedSlab
                apply_block: Optional[Callable] = None, per_stage: bool = True,
                transport=None, piece_slices: Optional[int] = None, timings: Optional[dict] = None):
    """Apply ``program`` to a z-sharded volume; returns this rank's interior output.

    per_stage=True: one halo exchange per chained stage (stage s+1's ghosts are
    stage s outputs), so no slice is computed twice.  per_stage=False: one
    exchange of the chain's total halo, then the whole chain on the padded slab.

    Per stage: post the exchange, compute the slices that need no ghost data
    (the interior [h, n - h), or up to the volume face on the first / last
    rank) while it is in flight, then the boundary slices once it lands
    (SURVEY.md §8(e) interior-first overlap).  Outputs are written into the
    next stage's padded buffer in place.
    """
    from . import _native

    apply_block = apply_block or _device_apply
    transport = transport or DistTransport(rank, world, group)
    stages = [_native.DeviceProgram([st]) for st in program.stages] if per_stage else [program]
    halos = [p.halo() for p in stages]
    given = local if isinstance(local, PaddedSlab) else None
    if given is not None:
        local = given.interior
    n = int(local.shape[0])
    plane = tuple(local.shape[1:])
    # every rank checks together: a neighbour thinner than the halo would leave
    # ghosts incomplete (and a one-sided error would hang the P2P exchange)
    need = max(halos) if world > 1 else 0
    if need and transport.min_slab(n, local) < need:
        raise ValueError(f"a z-slab is thinner than the halo {need}: use fewer ranks")
    if piece_slices is None:
        itemsize = max(local.element_size(), 4)
        piece_slices = max(1, int((2 << 30) // max(1, itemsize * plane[0] * plane[1])))
    lo = [h if rank > 0 else 0 for h in halos]
    hi = [h if rank < world - 1 else 0 for h in halos]
    in_dt = np.dtype(str(local.dtype).replace("torch.", ""))
    if given is not None and given.lo == lo[0] and given.hi == hi[0]:
        cur = given  # caller built the slab in a padded buffer: no copy
    else:
        cur = alloc_padded(n, plane, local.dtype, local, lo[0], hi[0])
        cur.interior.copy_(local)
    xchg_s = 0.0
    for k, (prog, h) in enumerate(zip(stages, halos)):
        out_np = prog.out_dtype(in_dt)
        import torch

        out_dt = getattr(torch, out_np.name)
        last = k + 1 == len(stages)
        nxt = (alloc_padded(n, plane, out_dt, local, 0, 0) if last
               else alloc_padded(n, plane, out_dt, local, lo[k + 1], hi[k + 1]))
        dst = nxt.interior
        t0 = time.perf_counter()
        pending = transport.start(cur, h) if (world > 1 and h > 0) else []
        a, b = lo[k], n - hi[k]  # needs no ghost data
        if a < b:
            _apply_range(cur, a, b, h, prog, dst, apply_block, piece_slices)
        transport.finish(pending)
        xchg_s += time.perf_counter() - t0
        if a >= b:
            _apply_range(cur, 0, n, h, prog, dst, apply_block, piece_slices)
        else:
            if a > 0:
                _apply_range(cur, 0, a, h, prog, dst, apply_block, piece_slices)
            if b < n:
                _apply_range(cur, b, n, h, prog, dst, apply_block, piece_slices)
        cur = nxt
        in_dt = out_np
    if timings is not None:
        timings["exchange_host_s"] = xchg_s
    return cur.interior


def run_sharded_local(slabs: Sequence, program, per_stage: bool = True,
                      apply_block: Optional[Callable] = None, piece_slices: Optional[int] = None):
    """Several z-slabs of one volume held by ONE process (e.g. virtual ranks on
    one GPU, or a C-style multi-device caller): the same per-stage schedule as
    :func:`run_sharded` with ghost slices copied device-to-device.  Returns the
    per-slab outputs; their concatenation equals the single-volume result."""
    from . import _native
    import torch

    apply_block = apply_block or _device_apply
    world = len(slabs)
    stages = [_native.DeviceProgram([st]) for st in program.stages] if per_stage else [program]
    halos = [p.halo() for p in stages]
    if world > 1 and min(int(s.shape[0]) for s in slabs) < max(halos):
        raise ValueError(f"a z-slab is thinner than the halo {max(halos)}")
    ns = [int(s.shape[0]) for s in slabs]
    plane = tuple(slabs[0].shape[1:])
    in_dt = np.dtype(str(slabs[0].dtype).replace("torch.", ""))
    if piece_slices is None:
        piece_slices = max(1, int((2 << 30) // max(1, 4 * plane[0] * plane[1])))
    curs = []
    for r, s in enumerate(slabs):
        h0 = halos[0]
        c = alloc_padded(ns[r], plane, s.dtype, s, h0 if r > 0 else 0, h0 if r < world - 1 else 0)
        c.interior.copy_(s)
        curs.append(c)
    for k, (prog, h) in enumerate(zip(stages, halos)):
        out_np = prog.out_dtype(in_dt)
        out_dt = getattr(torch, out_np.name)
        last = k + 1 == len(stages)
        nh = 0 if last else halos[k + 1]
        nxts = [alloc_padded(ns[r], plane, out_dt, slabs[r], 0 if (last or r == 0) else nh,
                             0 if (last or r == world - 1) else nh) for r in range(world)]
        # ghosts: rank r's lower ghosts = rank r-1's last h interior slices, etc.
        for r in range(world):
            c = curs[r]
            if r > 0 and h:
                c.buf[c.lo - h:c.lo].copy_(curs[r - 1].interior[ns[r - 1] - h:])
            if r < world - 1 and h:
                c.buf[c.lo + c.n:c.lo + c.n + h].copy_(curs[r + 1].interior[:h])
        for r in range(world):
            _apply_range(curs[r], 0, ns[r], h, prog, nxts[r].interior, apply_block, piece_slices)
        curs = nxts
        in_dt = out_np
    return [c.interior for c in curs]


# ---------------------------------------------------------------------------
# Two-pass global operator across ranks: Otsu (threshold.py:90-131).
# Pass 1 is the one place the path has a real exchange: each rank reduces its
# own slab on its GPU, then the float range (min/max) and the int64 histogram
# are all-reduced (NCCL over NVLink on the box, gloo in the CPU tests); every
# rank finalises the same threshold and applies it to its slab locally.
# ---------------------------------------------------------------------------
def otsu_sharded(local, bins: int, rank: int, world: int, group=None,
                 minmax_fn: Optional[Callable] = None, hist_fn: Optional[Callable] = None,
                 apply_fn: Optional[Callable] = None):
    """Return (labels of this rank's slab, threshold) — identical on every
    rank to the single-volume otsu_binarize.  ``local``: this rank's slab
    (numpy or CUDA tensor); the hooks default to the device
    (threshold.data_minmax / compute_histogram / apply_threshold)."""
    import torch

    from . import threshold

    minmax_fn = minmax_fn or threshold.data_minmax
    hist_fn = hist_fn or (lambda a, b, r: threshold.compute_histogram(a, b, r).counts)
    apply_fn = apply_fn or threshold.apply_threshold
    dt = np.dtype(str(local.dtype).replace("torch.", ""))
    if np.issubdtype(dt, np.integer):
        lim = np.iinfo(dt)
        lo, hi = float(lim.min), float(lim.max) + 1.0
    else:
        lo, hi = minmax_fn(local)
        if world > 1:  # min of the mins, max of the maxes (chunked_reduce, threshold.py:100-101)
            dist = _dist()
            dev = _comm_device(group)
            lo_t = torch.tensor([lo], dtype=torch.float64, device=dev)
            hi_t = torch.tensor([hi], dtype=torch.float64, device=dev)
            dist.all_reduce(lo_t, op=dist.ReduceOp.MIN, group=group)
            dist.all_reduce(hi_t, op=dist.ReduceOp.MAX, group=group)
            lo, hi = float(lo_t.item()), float(hi_t.item())
        if lo == hi:
            hi = lo + 1.0
    counts = np.asarray(hist_fn(local, bins, (lo, hi)), dtype=np.int64)
    if world > 1:
        dist = _dist()
        c = torch.from_numpy(counts.copy()).to(_comm_device(group))
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        counts = c.cpu().numpy()
    t = threshold.otsu_from_histogram(threshold.Histogram(lo, hi, counts))
    return apply_fn(local, t), t


def connected_components_sharded(local, connectivity: int, rank: int, world: int, group=None,
                                 label_fn: Optional[Callable] = None):
    """Return (labels of this rank's slab, total count) — identical to the
    single-volume connected_components (quantify.py:60-111: canonical ids in
    first-voxel scan order) for z-slabs in rank order.

    The reference's chunked scheme with ranks as chunks: each rank labels its
    slab on its GPU (``label_fn``, default quantify.connected_components: ids
    1..k in slab scan order = globally ordered candidates after a rank
    offset); one all_gather carries every rank's count and its first / last
    label planes (the path's only exchange); every rank then runs the same
    boundary union-find over the candidates (smaller id wins) and relabels
    its slab through the resulting table — no further communication."""
    import torch

    from . import quantify

    if connectivity not in (6, 26):
        raise ValueError(f"connectivity must be 6 or 26, got {connectivity}")
    label_fn = label_fn or (lambda a, c: quantify.connected_components(a, c))
    lab, k = label_fn(local, connectivity)
    is_torch = hasattr(lab, "device") and hasattr(lab, "cpu")
    lab_h = lab.cpu().numpy() if is_torch else np.asarray(lab)
    nz, ny, nx = lab_h.shape
    first = lab_h[0].astype(np.int64) if nz else np.zeros((ny, nx), np.int64)
    last = lab_h[-1].astype(np.int64) if nz else np.zeros((ny, nx), np.int64)
    counts = [int(k)]
    firsts, lasts, nzs = [first], [last], [nz]
    if world > 1:
        dist = _dist()
        dev = _comm_device(group)
        meta = torch.tensor([int(k), nz], dtype=torch.int64, device=dev)
        metas = [torch.empty_like(meta) for _ in range(world)]
        dist.all_gather(metas, meta, group=group)
        planes = torch.from_numpy(np.stack([first, last])).to(dev)
        allp = [torch.empty_like(planes) for _ in range(world)]
        dist.all_gather(allp, planes, group=group)
        counts = [int(m[0].item()) for m in metas]
        nzs = [int(m[1].item()) for m in metas]
        firsts = [p[0].cpu().numpy() for p in allp]
        lasts = [p[1].cpu().numpy() for p in allp]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    parent = np.arange(int(offs[-1]), dtype=np.int64)

    def find(a):
        root = a
        while parent[root] != root:
            root = parent[root]
        while parent[a] != root:
            parent[a], a = root, parent[a]
        return root

    shifts = [(0, 0)] if connectivity == 6 else [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    prev = None  # last non-empty slab below: (rank, its last plane)
    for r in range(len(counts)):
        if nzs[r] == 0:
            continue
        if prev is not None:
            pr, below = prev
            above = firsts[r]
            for dy, dx in shifts:
                # voxel (y, x) of the upper slab's first plane touches (y+dy, x+dx) below
                ys = slice(max(0, -dy), ny - max(0, dy))
                xs = slice(max(0, -dx), nx - max(0, dx))
                yb = slice(max(0, dy), ny - max(0, -dy))
                xb = slice(max(0, dx), nx - max(0, -dx))
                a = above[ys, xs].ravel()
                b = below[yb, xb].ravel()
                both = (a > 0) & (b > 0)
                for u, v in np.unique(np.stack([offs[pr] + b[both] - 1, offs[r] + a[both] - 1], 1), axis=0):
                    ru, rv = find(int(u)), find(int(v))
                    if ru != rv:
                        parent[max(ru, rv)] = min(ru, rv)
        prev = (r, lasts[r])
    # final ids in candidate order (= global first-voxel order): links point to
    # smaller ids, so pointer jumping reaches every root; roots numbered in order
    while True:
        nxt = parent[parent]
        if np.array_equal(nxt, parent):
            break
        parent = nxt
    is_root = parent == np.arange(parent.size)
    ids = np.cumsum(is_root).astype(np.uint32)
    fin = ids[parent] if parent.size else np.zeros(0, np.uint32)
    total = int(is_root.sum())
    mine = fin[offs[rank]:offs[rank + 1]]
    table = np.concatenate([[0], mine]).astype(np.uint32)
    if is_torch:
        t = torch.from_numpy(table.astype(np.int64)).to(lab.device)
        out = t[lab.to(torch.int64)].to(lab.dtype)
    else:
        out = table[lab_h]
    return out, total


def _comm_device(group):
    import torch

    backend = _dist().get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
