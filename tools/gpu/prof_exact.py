"""One exact-Gaussian launch pair (k_exact_z + k_exact_yx) at sigma=2 (for ncu)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, filters
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = torch.cuda.current_stream()
x = torch.rand((n + 16, n, n), device='cuda')
o = torch.empty((n, n, n), device='cuda')
_native.apply_device(x, o, filters.gaussian_program(2.0, "exact"), 8, s)
torch.cuda.synchronize()
print('done')
