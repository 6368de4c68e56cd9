"""A/B of the packed-FP32 Gaussian (k_gauss_p2) against the scalar fused kernel:
oracle agreement on ragged shapes / dtypes / radii (incl. unsharp), then device
timing at 256^3 and 1024^3 (sigma=2) and unsharp sigma=1."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()


def setmode(scalar):
    if scalar:
        os.environ["HB_GAUSS_SCALAR"] = "1"
    else:
        os.environ.pop("HB_GAUSS_SCALAR", None)


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))


bad = 0
for shape, sigma, dt in [((20, 37, 132), 2.0, np.float32), ((30, 70, 200), 1.0, np.float32),
                         ((25, 64, 128), 1.5, np.uint16), ((18, 33, 96), 2.0, np.uint8),
                         ((40, 129, 260), 0.75, np.float32), ((12, 20, 24), 2.0, np.float32)]:
    rng = np.random.default_rng(1)
    x = rng.random(shape, dtype=np.float32) if dt == np.float32 else \
        rng.integers(0, np.iinfo(dt).max, size=shape).astype(dt)
    ref = O.gaussian(x, sigma)
    uref = O.unsharp(x, sigma, 1.5)
    for scalar in (False, True):
        setmode(scalar)
        g = filters.gaussian(x, sigma)
        u = filters.unsharp(x, sigma, 1.5)
        e1, e2 = rel(g, ref), rel(u, uref)
        print(f"{'scalar' if scalar else 'p2    '} shape={shape} sigma={sigma} {np.dtype(dt).name}: "
              f"gauss {e1:.2e} unsharp {e2:.2e}")
        bad += e1 > 1e-5 or e2 > 1e-5
setmode(False)


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


for n, sigma, kind in [(256, 2.0, "gauss"), (1024, 2.0, "gauss"), (1024, 1.0, "unsharp")]:
    R = int(np.ceil(4 * sigma))
    x = torch.rand((n + 2 * R, n, n), device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    prog = filters.gaussian_program(sigma) if kind == "gauss" else filters.unsharp_program(sigma, 1.5)
    for scalar in (False, True, False):
        setmode(scalar)
        ms = timeit(x, o, prog, R)
        print(f"{'scalar' if scalar else 'p2    '} {kind} sigma={sigma} {n}^3: {ms:.3f} ms "
              f"{n**3/ms/1e6:.1f} Gvox/s")
    del x, o
setmode(False)
print("BAD" if bad else "ALL OK")
