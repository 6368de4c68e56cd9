"""One launch each of the headline kernels (gaussian sigma=2 fast, median r=1, mean r=1)
on the bench's 1024^3 padded block, for ncu."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, filters  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
which = sys.argv[2] if len(sys.argv) > 2 else "gm"
s = torch.cuda.current_stream()
x = torch.rand((n + 16, n, n), device='cuda')
o = torch.empty((n, n, n), device='cuda')
if "g" in which:
    _native.apply_device(x, o, filters.gaussian_program(2.0), 8, s)
if "m" in which:
    _native.apply_device(x, o, filters.median_program(1), 8, s)
if "M" in which:  # mean r=1 (the streaming box kernel)
    _native.apply_device(x, o, filters.mean_program(1), 8, s)
torch.cuda.synchronize()
print('done')
