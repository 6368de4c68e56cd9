"""Grey u16 / u8 erosion ball:3 (k_morph3): oracle bit-exactness on ragged shapes
and timing on a 2048^2 x 256 slab (for the rows-per-thread variants)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, morphology
s = torch.cuda.current_stream()
bad = 0
for shape, spec, dt in [((20, 37, 132), "ball:3", np.uint16), ((30, 70, 96), "box:2", np.uint16),
                        ((9, 65, 128), "cross:3", np.uint8), ((17, 50, 200), "ball:2", np.uint16),
                        ((12, 33, 64), "ball:1", np.uint8)]:
    rng = np.random.default_rng(sum(shape))
    x = rng.integers(0, np.iinfo(dt).max, size=shape).astype(dt)
    se = morphology.StructuringElement.parse(spec)
    ok = np.array_equal(morphology.erode(x, se), O.erode(x, se.offsets)) and \
        np.array_equal(morphology.dilate(x, se), O.dilate(x, se.reflect().offsets))
    bad += not ok
    print(f"{spec} {np.dtype(dt).name} {shape}: {'ok' if ok else 'MISMATCH'}", flush=True)
m, nzs = 2048, 256
x = torch.randint(0, 65536, (nzs + 6, m, m), device="cuda", dtype=torch.int32).to(torch.uint16)
o = torch.empty((nzs, m, m), device="cuda", dtype=torch.uint16)
for opn in ("erode", "dilate"):
    prog = morphology.morph_program(opn, morphology.StructuringElement.parse("ball:3"))
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
    v = m * m * nzs
    print(f"{opn} ball:3 u16 2048^2x{nzs}: {v / ms / 1e6:.1f} Gvox/s ({4 * v / ms / 1e6 / 6445.6:.3f} of HBM)", flush=True)
print("BAD" if bad else "parity ok")
