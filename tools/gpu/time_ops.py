"""Device timing (CUDA events, warm) of hot-path ops on 1024^3 f32 blocks.
usage: python tools/gpu/time_ops.py [n] [op,op,...]   ops: median,mean,gauss,gauss_exact,log,unsharp,erode_u16"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, morphology

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["median", "mean", "gauss", "gauss_exact", "log"]
s = torch.cuda.current_stream()
x = torch.rand((n + 20, n, n), device="cuda")
o = torch.empty((n, n, n), device="cuda")
progs = {"median": (filters.median_program(1), 1), "mean": (filters.mean_program(1), 1),
         "gauss": (filters.gaussian_program(2.0), 8), "gauss_exact": (filters.gaussian_program(2.0, "exact"), 8),
         "log": (filters.log_program(2.0), 10), "unsharp": (filters.unsharp_program(1.0, 1.5), 4)}
for op in ops:
    if op == "erode_u16":
        src = torch.randint(0, 65535, (n + 6, n, n), device="cuda", dtype=torch.int32).to(torch.uint16)
        dst = torch.empty((n, n, n), device="cuda", dtype=torch.uint16)
        prog, zb, xi, oo = morphology.morph_program("erode", morphology.StructuringElement.ball(3)), 3, src, dst
    else:
        (prog, zb), xi, oo = progs[op], x, o
    for _ in range(2):
        _native.apply_device(xi, oo, prog, zb, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        _native.apply_device(xi, oo, prog, zb, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{op:12s} {n}^3: {ms:7.3f} ms {n**3/ms/1e6:7.1f} Gvox/s")
