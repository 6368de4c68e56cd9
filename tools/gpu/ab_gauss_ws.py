"""A/B of the warp-specialised Gaussian (k_gauss_ws) against k_gauss_p2
(HB_GAUSS_P2=1): oracle agreement on ragged shapes / dtypes / radii (incl.
unsharp), then device timing at 256^3 and 1024^3 (sigma=2), unsharp sigma=1."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()


def setmode(p2):
    if p2:
        os.environ["HB_GAUSS_P2"] = "1"
    else:
        os.environ.pop("HB_GAUSS_P2", None)


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(1e-30, np.max(np.abs(b))))


bad = 0
for shape, sigma, dt in [((20, 37, 132), 2.0, np.float32), ((30, 70, 200), 1.0, np.float32),
                         ((25, 64, 128), 1.5, np.uint16), ((18, 33, 96), 2.0, np.uint8),
                         ((40, 129, 260), 0.75, np.float32), ((12, 20, 24), 2.0, np.float32),
                         ((60, 100, 68), 1.25, np.float32), ((33, 17, 64), 0.5, np.uint16)]:
    rng = np.random.default_rng(1)
    x = rng.random(shape, dtype=np.float32) if dt == np.float32 else \
        rng.integers(0, np.iinfo(dt).max, size=shape).astype(dt)
    ref = O.gaussian(x, sigma)
    uref = O.unsharp(x, sigma, 1.5)
    g = filters.gaussian(x, sigma)
    u = filters.unsharp(x, sigma, 1.5)
    e1, e2 = rel(g, ref), rel(u, uref)
    print(f"ws shape={shape} sigma={sigma} {np.dtype(dt).name}: gauss {e1:.2e} unsharp {e2:.2e}", flush=True)
    bad += e1 > 1e-5 or e2 > 1e-5


def timeit(x, o, prog, zb, reps=10):
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


for n, sigma, kind in [(1024, 2.0, "g"), (256, 2.0, "g"), (1024, 1.0, "u"), (512, 2.0, "g")]:
    R = int(np.ceil(4 * sigma))
    x = torch.rand((n + 2 * R, n, n), device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    prog = filters.gaussian_program(sigma) if kind == "g" else filters.unsharp_program(sigma, 1.5)
    res = []
    for p2 in (False, True):
        setmode(p2)
        ms = timeit(x, o, prog, R)
        res.append(f"{'p2' if p2 else 'ws'} {n ** 3 / ms / 1e6:7.1f} Gvox/s ({ms:.3f} ms)")
    setmode(False)
    print(f"{kind} n={n} sigma={sigma}: " + " | ".join(res), flush=True)
    del x, o
print("BAD" if bad else "parity ok")
