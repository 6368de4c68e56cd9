"""One hessian_xy (sigma 2, exact) and one LoG on a device-resident 512^3 f32
volume (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = torch.Generator(device="cuda").manual_seed(0)
with session():
    x = torch.rand((n + 20, n, n), generator=g, device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    for prog in (filters.hessian_program(2.0, "xy"), filters.log_program(2.0, "exact")):
        _native.apply_device(x, o, prog, 10)
    torch.cuda.synchronize()
