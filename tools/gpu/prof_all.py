"""One launch of every hot kernel on config-sized device volumes (for ncu):
median r=1, mean r=1, fast gaussian sigma=2, exact gaussian sigma=2 (2 kernels),
LoG (exact smoothing + second stage), erode ball:3 u16."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, filters, morphology
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = torch.cuda.current_stream()
x = torch.rand((n + 20, n, n), device='cuda')
o = torch.empty((n, n, n), device='cuda')
u = torch.randint(0, 65535, (n + 6, n, n), device='cuda', dtype=torch.int32).to(torch.uint16)
ou = torch.empty((n, n, n), device='cuda', dtype=torch.uint16)
_native.apply_device(x, o, filters.median_program(1), 1, s)
_native.apply_device(x, o, filters.mean_program(1), 1, s)
_native.apply_device(x, o, filters.gaussian_program(2.0), 8, s)
_native.apply_device(x, o, filters.gaussian_program(2.0, "exact"), 8, s)
_native.apply_device(x, o, filters.log_program(2.0), 10, s)
_native.apply_device(u, ou, morphology.morph_program('erode', morphology.StructuringElement.ball(3)), 3, s)
torch.cuda.synchronize()
print('done')
