"""Device timing (CUDA events, warm, inside a session) of local_threshold
(local.cu) on device-resident 1024^3 volumes, every kind."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, session

s = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(0)


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rows = []
with session():
    out = torch.empty((n, n, n), device="cuda", dtype=torch.uint32)
    for dt in ("uint16", "uint8", "float32"):
        xf = torch.rand((n + 8, n, n), generator=g, device="cuda")
        x = xf if dt == "float32" else (xf * (255 if dt == "uint8" else 65535)).to(getattr(torch, dt))
        del xf
        for kind, w in (("mean", 1), ("mean", 2), ("niblack", 2), ("sauvola", 2), ("sauvola", 4),
                        ("gaussian", 2), ("median", 1), ("median", 2)):
            if dt != "uint16" and kind in ("median", "gaussian"):
                continue
            prog = filters.local_threshold_program(kind, w, 0.2, None, 1.0, dtype=dt)
            ms = dev_time(lambda: _native.apply_device(x, out, prog, 4, s))
            rows.append((f"{kind} w={w} {dt}", ms))
        del x
        torch.cuda.synchronize()
for name, ms in rows:
    print(f"| local_threshold {name} | {n}^3 | {ms:.2f} ms | {n**3/ms/1e6:.1f} Gvox/s |")
