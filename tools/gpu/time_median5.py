"""median r=2 (default) or r=argv[2] device timing at argv[1]^3 (u8 / u16 / f32), CUDA events."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
r = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(0)
with session():
    for dt in ("uint8", "uint16", "float32"):
        xf = torch.rand((n + 2 * r, n, n), generator=g, device="cuda")
        x = xf if dt == "float32" else (xf * (255 if dt == "uint8" else 65535)).to(getattr(torch, dt))
        out = torch.empty((n, n, n), device="cuda", dtype=x.dtype)
        prog = filters.median_program(r)
        _native.apply_device(x, out, prog, r)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(3):
            _native.apply_device(x, out, prog, r)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"| median r={r} {dt} | {n}^3 | {ms:.2f} ms | {n**3/ms/1e6:.1f} Gvox/s |")
