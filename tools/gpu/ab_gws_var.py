"""k_gauss_ws tile widths (HB_GWS_TX, f32 R=8) at 1024^3 / 512^3 / 256^3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()
vars_ = sys.argv[1].split(",") if len(sys.argv) > 1 else ["48", "64"]
xs = np.random.default_rng(0).random((40, 70, 132), dtype=np.float32)
ref = O.gaussian(xs, 2.0)
for v in vars_:
    os.environ["HB_GWS_TX"] = v
    g = filters.gaussian(xs, 2.0)
    e = float(np.max(np.abs(g - ref)) / np.max(np.abs(ref)))
    line = [f"var {v}: parity {e:.1e}"]
    for n in (1024, 512, 256):
        x = torch.rand((n + 16, n, n), device="cuda")
        o = torch.empty((n, n, n), device="cuda")
        prog = filters.gaussian_program(2.0)
        for _ in range(2):
            _native.apply_device(x, o, prog, 8, s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(10):
            _native.apply_device(x, o, prog, 8, s)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        line.append(f"{n}: {n ** 3 / ms / 1e6:6.1f}")
        del x, o
    print(" | ".join(line), flush=True)
