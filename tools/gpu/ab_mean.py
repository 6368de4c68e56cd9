"""A/B of the streaming box mean (box.cu) against the TMA fused mean: bitwise
agreement on ragged shapes + oracle check, then device timing at 1024^3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()


def run(x, r, zb, nzo, tma):
    if tma:
        os.environ["HB_MEAN_TMA"] = "1"
    else:
        os.environ.pop("HB_MEAN_TMA", None)
    o = torch.empty((nzo,) + tuple(x.shape[1:]), device="cuda")
    _native.apply_device(x, o, filters.mean_program(r), zb, s)
    torch.cuda.synchronize()
    return o


bad = 0
for shape, r, dt in [((20, 37, 132), 1, torch.float32), ((9, 130, 260), 1, torch.float32),
                     ((33, 64, 512), 2, torch.float32), ((12, 17, 8), 1, torch.uint16),
                     ((12, 40, 136), 2, torch.uint8), ((5, 4, 4), 1, torch.float32),
                     ((40, 200, 1028), 1, torch.float32)]:
    if dt == torch.float32:
        x = torch.rand(shape, device="cuda")
    else:
        x = torch.randint(0, 255 if dt == torch.uint8 else 65535, shape, device="cuda",
                          dtype=torch.int32).to(dt)
    for zb, nzo in [(0, shape[0]), (r, shape[0] - 2 * r)]:
        if nzo <= 0:
            continue
        a = run(x, r, zb, nzo, False)
        b = run(x, r, zb, nzo, True)
        same = torch.equal(a, b)
        ref = O.mean(x.cpu().numpy(), r)[zb:zb + nzo]
        err = float(np.max(np.abs(a.cpu().numpy() - ref)) / max(1e-30, np.max(np.abs(ref))))
        print(f"shape={shape} r={r} dt={dt} zb={zb}: stream==tma {same}  oracle err {err:.2e}")
        bad += (not same) or err > 1e-5

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
x = torch.rand((n + 2, n, n), device="cuda")
o = torch.empty((n, n, n), device="cuda")
for tma in (False, True, False, True):
    if tma:
        os.environ["HB_MEAN_TMA"] = "1"
    else:
        os.environ.pop("HB_MEAN_TMA", None)
    prog = filters.mean_program(1)
    for _ in range(3):
        _native.apply_device(x, o, prog, 1, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10):
        _native.apply_device(x, o, prog, 1, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{'tma   ' if tma else 'stream'} mean r=1 {n}^3: {ms:.3f} ms  {n**3/ms/1e6:.1f} Gvox/s  "
          f"{8*n**3/ms/1e6:.0f} GB/s")
print("BAD" if bad else "ALL OK")
