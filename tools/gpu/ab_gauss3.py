"""A/B of k_gauss3 (default) against k_gauss_ws (HB_GAUSS_WS=1): oracle
agreement on ragged shapes (incl. unsharp, tile/volume borders, odd nx ->
fallback), then device timing at 1024^3 / 256^3 / 512^3 (sigma=2), unsharp
sigma=1, and a z-chunk cap sweep (HB_G3_ZCAP)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(1e-30, np.max(np.abs(b))))


bad = 0
for shape, sigma in [((20, 37, 132), 2.0), ((30, 70, 200), 1.0), ((40, 129, 260), 0.75),
                     ((12, 20, 24), 2.0), ((60, 100, 68), 1.25), ((70, 65, 98), 2.0),
                     ((9, 33, 50), 1.75), ((100, 40, 96), 2.0)]:
    rng = np.random.default_rng(1)
    x = rng.random(shape, dtype=np.float32)
    ref = O.gaussian(x, sigma)
    uref = O.unsharp(x, sigma, 1.5)
    g = filters.gaussian(x, sigma)
    u = filters.unsharp(x, sigma, 1.5)
    e1, e2 = rel(g, ref), rel(u, uref)
    print(f"tri shape={shape} sigma={sigma}: gauss {e1:.2e} unsharp {e2:.2e}", flush=True)
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
    for ws in (False, True):
        if ws:
            os.environ["HB_GAUSS_WS"] = "1"
        else:
            os.environ.pop("HB_GAUSS_WS", None)
        ms = timeit(x, o, prog, R)
        res.append(f"{'ws' if ws else 'v3'} {n ** 3 / ms / 1e6:7.1f} Gvox/s ({ms:.3f} ms)")
    os.environ.pop("HB_GAUSS_WS", None)
    print(f"{kind} n={n} sigma={sigma}: " + " | ".join(res), flush=True)
    if n == 1024 and kind == "g":
        for cap in (64, 96, 128, 256, 384, 1100):
            os.environ["HB_G3_ZCAP"] = str(cap)
            ms = timeit(x, o, prog, R)
            print(f"   zcap {cap}: {n ** 3 / ms / 1e6:7.1f} Gvox/s", flush=True)
        os.environ.pop("HB_G3_ZCAP", None)
    del x, o
print("BAD" if bad else "parity ok")
