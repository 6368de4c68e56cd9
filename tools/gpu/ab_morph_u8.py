"""Grey u8 erosion / dilation: k_morph_u16s<uint8_t> behind k_morph_bits2's
grey flag (default) against k_morph3 (HB_MORPH_U8_SMEM=1): oracle
bit-exactness on ragged shapes (every SE family, grey and binary blocks), then
timing on a 2048^2 x 256 grey slab."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, morphology

s = torch.cuda.current_stream()
bad = 0
cases = [((20, 37, 128), "ball:3"), ((30, 70, 96), "box:2"), ((9, 65, 64), "cross:3"),
         ((17, 50, 224), "ball:2"), ((12, 33, 32), "ball:1"), ((40, 100, 256), "ball:3"),
         ((25, 129, 512), "box:3"), ((11, 31, 32), "cross:1"), ((50, 40, 160), "box:1")]
for shape, spec in cases:
    rng = np.random.default_rng(sum(shape))
    se = morphology.StructuringElement.parse(spec)
    for kind in ("grey", "binary"):
        if kind == "grey":
            x = rng.integers(0, 256, size=shape).astype(np.uint8)
        else:
            x = (rng.random(shape) < 0.5).astype(np.uint8)
        re, rd = O.erode(x, se.offsets), O.dilate(x, se.reflect().offsets)
        for env in ({}, {"HB_MORPH_U8_SMEM": "1"}):
            os.environ.pop("HB_MORPH_U8_SMEM", None)
            os.environ.update(env)
            ok = np.array_equal(morphology.erode(x, se), re) and np.array_equal(morphology.dilate(x, se), rd)
            bad += not ok
            print(f"{spec} u8 {kind} {shape} {'smem' if env else 'stream'}: {'ok' if ok else 'MISMATCH'}", flush=True)
os.environ.pop("HB_MORPH_U8_SMEM", None)
m, nzs = 2048, 256
x = torch.randint(0, 256, (nzs + 6, m, m), device="cuda", dtype=torch.int32).to(torch.uint8)
o = torch.empty((nzs, m, m), device="cuda", dtype=torch.uint8)
prog = morphology.morph_program("erode", morphology.StructuringElement.parse("ball:3"))
outs = []
for name, env in (("stream", {}), ("smem", {"HB_MORPH_U8_SMEM": "1"})):
    os.environ.pop("HB_MORPH_U8_SMEM", None)
    os.environ.update(env)
    for _ in range(2):
        _native.apply_device(x, o, prog, 3, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10):
        _native.apply_device(x, o, prog, 3, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    outs.append(o.clone())
    v = m * m * nzs
    print(f"erode ball:3 u8 grey 2048^2x{nzs} {name}: {v / ms / 1e6:.1f} Gvox/s ({2 * v / ms / 1e6 / 6545.3:.3f} of HBM)",
          flush=True)
os.environ.pop("HB_MORPH_U8_SMEM", None)
same = torch.equal(outs[0], outs[1])
bad += not same
print(f"stream == smem on the slab: {same}")
print("BAD" if bad else "parity ok")
