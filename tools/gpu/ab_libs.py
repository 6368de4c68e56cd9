"""A/B of library builds (HARPIA_LIB, one subprocess per build): device time
of one operator on a synthetic volume, output checksum compared across builds.

usage: python tools/gpu/ab_libs.py OP N lib1.so lib2.so ...
  OP: median (r=1 f32), gaussian (sigma=2 fast f32), erode_u16 (ball:3), median5 /
  median5_u16 (r=2 on N x 1024^2), erode_u8_grey / erode_u8_bin (ball:3, N x 2048^2)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, morphology
op, n = sys.argv[1], int(sys.argv[2])
s = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(5)
if op in ("median5", "median5_u16"):
    if op == "median5":
        x = torch.rand((n + 4, 1024, 1024), generator=g, device="cuda")
    else:
        x = torch.randint(0, 65536, (n + 4, 1024, 1024), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
    o = torch.empty((n, 1024, 1024), device="cuda", dtype=x.dtype)
    prog, zb = filters.median_program(2), 2
elif op in ("erode_u8_grey", "erode_u8_bin"):
    if op == "erode_u8_grey":
        x = torch.randint(0, 256, (n + 6, 2048, 2048), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
    else:
        x = (torch.rand((n + 6, 2048, 2048), generator=g, device="cuda") < 0.5).to(torch.uint8)
    o = torch.empty((n, 2048, 2048), device="cuda", dtype=torch.uint8)
    prog, zb = morphology.morph_program("erode", morphology.StructuringElement.ball(3)), 3
elif op == "erode_u16":
    x = torch.randint(0, 65536, (n + 6, 2048, 2048), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
    o = torch.empty((n, 2048, 2048), device="cuda", dtype=torch.uint16)
    prog, zb = morphology.morph_program("erode", morphology.StructuringElement.ball(3)), 3
else:
    h = 1 if op == "median" else 8
    x = torch.rand((n + 2 * h, n, n), generator=g, device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    prog, zb = (filters.median_program(1), 1) if op == "median" else (filters.gaussian_program(2.0), 8)
for _ in range(3):
    _native.apply_device(x, o, prog, zb, s)
torch.cuda.synchronize()
ts = []
for rep in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        _native.apply_device(x, o, prog, zb, s)
    b.record(s)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 5)
ms = min(ts)
print(json.dumps({"ms": ms, "gvox": o.numel() / ms / 1e6, "sum": float(o.double().sum())}))
'''
op, n = sys.argv[1], sys.argv[2]
res = {}
for lib in sys.argv[3:]:
    env = dict(os.environ, HARPIA_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD, op, n], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
    res[lib] = line
    print(f"{os.path.basename(lib)}: {line}", flush=True)
sums = {json.loads(v)["sum"] for v in res.values() if v.startswith("{")}
print("identical outputs" if len(sums) == 1 else f"OUTPUTS DIFFER {sums}")
