"""Two launches each of the hot kernels on config-sized device volumes (for ncu)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, filters, morphology
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
which = sys.argv[2].split(',') if len(sys.argv) > 2 else ['median', 'mean', 'gauss', 'erode']
s = torch.cuda.current_stream()
x = torch.rand((n + 16, n, n), device='cuda')
o = torch.empty((n, n, n), device='cuda')
u = torch.randint(0, 65535, (n + 6, n, n), device='cuda', dtype=torch.int32).to(torch.uint16)
ou = torch.empty((n, n, n), device='cuda', dtype=torch.uint16)
for _ in range(2):
    if 'median' in which:
        _native.apply_device(x, o, filters.median_program(1), 1, s)
    if 'mean' in which:
        _native.apply_device(x, o, filters.mean_program(1), 1, s)
    if 'gauss' in which:
        _native.apply_device(x, o, filters.gaussian_program(2.0), 8, s)
    if 'log' in which:
        _native.apply_device(x, o[: n - 4], filters.log_program(2.0), 12, s)
    if 'erode' in which:
        _native.apply_device(u, ou, morphology.morph_program('erode', morphology.StructuringElement.ball(3)), 3, s)
torch.cuda.synchronize()
print('done')
