import os, sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, morphology
s = torch.cuda.current_stream()
n, nzo = 2048, 512
x = (torch.rand((nzo + 6, n, n), device="cuda") < 0.5).to(torch.uint8)
o = torch.empty((nzo, n, n), dtype=torch.uint8, device="cuda")
se = morphology.StructuringElement.parse("ball:3")
for cap in ("32", "48", "64", "96", "128", "64"):
    os.environ["HB_MB2_ZCAP"] = cap
    for opn in ("erode", "dilate"):
        prog = morphology.morph_program(opn, se)
        for _ in range(3):
            _native.apply_device(x, o, prog, 3, s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(10):
            _native.apply_device(x, o, prog, 3, s)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"zcap {cap} {opn}: {n*n*nzo/ms/1e6:7.1f} Gvox/s ({2*n*n*nzo/ms/1e6/6445.6:.3f} of HBM)", flush=True)
