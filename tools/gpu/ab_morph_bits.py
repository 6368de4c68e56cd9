"""A/B of the one-bit-per-voxel binary erode/dilate (k_morph_bits, default for
{0,1} uint8 with nx % 32 == 0) against the byte-wise AND/OR k_morph3
(HB_MORPH_NOBITS=1): oracle bit-exactness on ragged shapes and every SE
family, then device timing on 2048^2 x 512 slabs (ball:3)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, morphology

s = torch.cuda.current_stream()
bad = 0
for shape, spec in [((20, 37, 64), "ball:3"), ((30, 70, 96), "box:2"), ((9, 33, 128), "cross:3"),
                    ((40, 129, 32), "ball:1"), ((17, 50, 2048), "ball:3"), ((12, 8, 64), "ball:2"),
                    ((25, 45, 160), "box:1"), ((7, 9, 96), "cross:1")]:
    rng = np.random.default_rng(sum(shape))
    x = (rng.random(shape) < 0.6).astype(np.uint8)
    se = morphology.StructuringElement.parse(spec)
    for opn, fn, ofn in (("erode", morphology.erode, O.erode), ("dilate", morphology.dilate, O.dilate)):
        got = fn(x, se)
        ref = ofn(x, se.offsets) if opn == "erode" else ofn(x, se.reflect().offsets)
        ok = np.array_equal(got, ref)
        bad += not ok
        print(f"{opn} {spec} shape={shape}: {'ok' if ok else 'MISMATCH'}", flush=True)


# grey u8 through the same entry: the bits kernel flags it, the u16-lane kernel rewrites
for shape, spec in [((20, 37, 64), "ball:3"), ((11, 40, 96), "box:1")]:
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, size=shape).astype(np.uint8)
    x[0, 0, 0] = 1
    se = morphology.StructuringElement.parse(spec)
    ok = np.array_equal(morphology.erode(x, se), O.erode(x, se.offsets)) and \
        np.array_equal(morphology.dilate(x, se), O.dilate(x, se.reflect().offsets))
    bad += not ok
    print(f"grey u8 {spec} shape={shape}: {'ok' if ok else 'MISMATCH'}", flush=True)
    # binary except one grey voxel deep inside
    xb = (rng.random(shape) < 0.5).astype(np.uint8)
    xb[shape[0] // 2, shape[1] // 2, shape[2] // 2] = 7
    ok = np.array_equal(morphology.erode(xb, se), O.erode(xb, se.offsets))
    bad += not ok
    print(f"one-grey-voxel u8 {spec} shape={shape}: {'ok' if ok else 'MISMATCH'}", flush=True)


def timeit(x, o, prog, zb, reps=5):
    for _ in range(2):
        _native.apply_device(x, o, prog, zb, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        _native.apply_device(x, o, prog, zb, s)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n, nzo = 2048, 512
se = morphology.StructuringElement.parse("ball:3")
x = (torch.rand((nzo + 6, n, n), device="cuda") < 0.5).to(torch.uint8)
o = torch.empty((nzo, n, n), dtype=torch.uint8, device="cuda")
for opn in ("erode", "dilate"):
    prog = morphology.morph_program(opn, se)
    res, outs = [], []
    for nob in (False, True):
        if nob:
            os.environ["HB_MORPH_NOBITS"] = "1"; os.environ["HB_MORPH_BITS1"] = "1"
        else:
            os.environ.pop("HB_MORPH_NOBITS", None); os.environ.pop("HB_MORPH_BITS1", None)
        ms = timeit(x, o, prog, 3)
        outs.append(o.clone())
        v = n * n * nzo / ms / 1e6
        res.append(f"{'bytes' if nob else 'bits'} {v:7.1f} Gvox/s ({ms:.3f} ms, {2 * v / 6445.6:.3f} of HBM)")
    os.environ.pop("HB_MORPH_NOBITS", None); os.environ.pop("HB_MORPH_BITS1", None)
    same = bool(torch.equal(outs[0], outs[1]))
    bad += not same
    print(f"{opn} ball:3 u8 binary 2048^2 x {nzo}: " + " | ".join(res) + f" | identical {same}", flush=True)
print("BAD" if bad else "parity ok")
