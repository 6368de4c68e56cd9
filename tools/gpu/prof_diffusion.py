"""Two explicit diffusion steps (exp) on a device-resident n^3 f32 block (ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = torch.Generator(device="cuda").manual_seed(0)
with session():
    x = torch.rand((n + 4, n, n), generator=g, device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    _native.apply_device(x, o, filters.diffusion_program(2, 0.2), 2)
    torch.cuda.synchronize()
