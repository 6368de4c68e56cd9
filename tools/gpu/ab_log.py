"""A/B of the streaming LoG second stage (logd.cu) against the tiled k_log_diff:
bitwise agreement (both are exact given g) + reference-exact LoG vs the oracle,
then device timing of the LoG op at 1024^3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()


def mode(tile):
    if tile:
        os.environ["HB_LOG_TILE"] = "1"
    else:
        os.environ.pop("HB_LOG_TILE", None)


bad = 0
for shape in [(20, 37, 132), (9, 130, 260), (6, 5, 8), (33, 64, 512), (3, 3, 4), (40, 200, 1028)]:
    x = torch.rand(shape, device="cuda")
    for zb, nzo in [(0, shape[0]), (1, shape[0] - 2)]:
        if nzo <= 0:
            continue
        outs = []
        for tile in (False, True):
            mode(tile)
            o = torch.empty((nzo,) + shape[1:], device="cuda")
            _native.apply_device(x, o, filters.log_program(2.0), zb, s)
            torch.cuda.synchronize()
            outs.append(o.cpu().numpy())
        same = np.array_equal(outs[0], outs[1])
        print(f"shape={shape} zb={zb}: stream==tile {same}")
        bad += not same
mode(False)
xs = np.random.default_rng(3).random((24, 40, 132), dtype=np.float32)
lg = filters.log(xs, 2.0)
ok = np.array_equal(lg, O.log(xs, 2.0)) if hasattr(O, "log") else None
print("log vs oracle bit-exact:", ok)
bad += ok is False

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
x = torch.rand((n + 20, n, n), device="cuda")
o = torch.empty((n, n, n), device="cuda")
for tile in (False, True, False):
    mode(tile)
    prog = filters.log_program(2.0)
    for _ in range(2):
        _native.apply_device(x, o, prog, 10, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        _native.apply_device(x, o, prog, 10, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{'tile  ' if tile else 'stream'} LoG sigma=2 exact {n}^3: {ms:.3f} ms {n**3/ms/1e6:.1f} Gvox/s")
print("BAD" if bad else "ALL OK")
