"""One launch of each local_threshold kernel family on a device-resident
512^3 u16 volume (for ncu --set full)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = torch.Generator(device="cuda").manual_seed(0)
with session():
    x = (torch.rand((n + 8, n, n), generator=g, device="cuda") * 65535).to(torch.uint16)
    out = torch.empty((n, n, n), device="cuda", dtype=torch.uint32)
    for kind in ("sauvola", "mean", "gaussian"):
        prog = filters.local_threshold_program(kind, 2, 0.2, None, 1.0, dtype="uint16")
        _native.apply_device(x, out, prog, 4)
    torch.cuda.synchronize()
