"""Grey u16 erosion / dilation: k_morph_u16s (register streaming, default)
against k_morph3 (HB_MORPH_U16_SMEM=1): oracle bit-exactness on ragged shapes
for every SE family and radius (both kernels), then timing on a 2048^2 x 256
slab (ball:3, configs[2]) with a z-cap sweep."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, morphology

s = torch.cuda.current_stream()
bad = 0
cases = [((20, 37, 136), "ball:3"), ((30, 70, 96), "box:2"), ((9, 65, 128), "cross:3"),
         ((17, 50, 200), "ball:2"), ((12, 33, 64), "ball:1"), ((40, 100, 264), "ball:3"),
         ((3, 8, 8), "ball:3"), ((25, 129, 520), "box:3"), ((11, 31, 16), "cross:1"),
         ((50, 40, 392), "box:1"), ((7, 300, 136), "cross:2"), ((8, 9, 1000), "ball:3")]
for shape, spec in cases:
    rng = np.random.default_rng(sum(shape))
    x = rng.integers(0, 65536, size=shape).astype(np.uint16)
    se = morphology.StructuringElement.parse(spec)
    re, rd = O.erode(x, se.offsets), O.dilate(x, se.reflect().offsets)
    for env in ({}, {"HB_MORPH_U16_SMEM": "1"}):
        os.environ.pop("HB_MORPH_U16_SMEM", None)
        os.environ.update(env)
        ok = np.array_equal(morphology.erode(x, se), re) and np.array_equal(morphology.dilate(x, se), rd)
        bad += not ok
        print(f"{spec} u16 {shape} {'smem' if env else 'stream'}: {'ok' if ok else 'MISMATCH'}", flush=True)
os.environ.pop("HB_MORPH_U16_SMEM", None)
m, nzs = 2048, 256
x = torch.randint(0, 65536, (nzs + 6, m, m), device="cuda", dtype=torch.int32).to(torch.uint16)
o = torch.empty((nzs, m, m), device="cuda", dtype=torch.uint16)


def timeit(prog):
    for _ in range(2):
        _native.apply_device(x, o, prog, 3, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10):
        _native.apply_device(x, o, prog, 3, s)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10


peak = 6545.3
outs = []
for opn in ("erode", "dilate"):
    prog = morphology.morph_program(opn, morphology.StructuringElement.parse("ball:3"))
    for name, env in (("stream", {}), ("smem", {"HB_MORPH_U16_SMEM": "1"})):
        os.environ.pop("HB_MORPH_U16_SMEM", None)
        os.environ.update(env)
        ms = timeit(prog)
        outs.append(o.clone())
        v = m * m * nzs
        print(f"{opn} ball:3 u16 2048^2x{nzs} {name}: {v / ms / 1e6:.1f} Gvox/s ({4 * v / ms / 1e6 / peak:.3f} of HBM)",
              flush=True)
    os.environ.pop("HB_MORPH_U16_SMEM", None)
    same = torch.equal(outs[-1], outs[-2])
    print(f"  stream == smem on the slab: {same}", flush=True)
    bad += not same
prog = morphology.morph_program("erode", morphology.StructuringElement.parse("ball:3"))
for zc in (16, 32, 48, 64, 96, 128, 256):
    os.environ["HB_MU_ZCAP"] = str(zc)
    ms = timeit(prog)
    print(f"  zcap {zc}: {m * m * nzs / ms / 1e6:.1f} Gvox/s", flush=True)
os.environ.pop("HB_MU_ZCAP", None)
print("BAD" if bad else "parity ok")
