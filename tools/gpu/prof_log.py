"""One LoG sigma=2 (exact smoothing + second differences) on the bench's 1024^3 block, for ncu / timing."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = torch.cuda.current_stream()
x = torch.rand((n + 20, n, n), device="cuda")
o = torch.empty((n, n, n), device="cuda")
prog = filters.log_program(2.0)
with _native.session():
    for _ in range(2):
        _native.apply_device(x, o, prog, 10, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3):
        _native.apply_device(x, o, prog, 10, s)
    b.record(s)
    torch.cuda.synchronize()
print(f"LoG {n}^3: {a.elapsed_time(b) / 3:.3f} ms = {n**3 / (a.elapsed_time(b) / 3) / 1e6:.1f} Gvox/s")
