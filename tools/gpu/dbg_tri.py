"""Which role bounds k_gauss_tri: time it with the y/x/z arithmetic skipped
(HB_GTRI_DBG bitmask; results are wrong in those modes)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters
s = torch.cuda.current_stream()
n = 1024
x = torch.rand((n + 16, n, n), device="cuda")
o = torch.empty((n, n, n), device="cuda")
prog = filters.gaussian_program(2.0)
for m in [0, 1, 2, 4, 3, 5, 6, 7]:
    os.environ["HB_GTRI_DBG"] = str(m)
    for _ in range(2):
        _native.apply_device(x, o, prog, 8, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        _native.apply_device(x, o, prog, 8, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"skip y={m & 1} x={(m >> 1) & 1} z={(m >> 2) & 1}: {n**3 / ms / 1e6:7.1f} Gvox/s", flush=True)
