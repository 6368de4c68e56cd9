"""DRAM-overfetch probe for the fused Gaussian: one launch per shape (z, y, x),
run under `ncu --metrics dram__bytes_read.sum,...` to see whether halo rows
are re-read from DRAM (multi-wave grids) or not (single-wave grids)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, filters  # noqa: E402

shapes = [(1024, 1024, 1024), (1024, 256, 1024), (256, 1024, 1024), (1024, 1024, 256)]
s = torch.cuda.current_stream()
prog = filters.gaussian_program(2.0)
for z, y, x in shapes:
    a = torch.rand((z + 16, y, x), device='cuda')
    o = torch.empty((z, y, x), device='cuda')
    _native.apply_device(a, o, prog, 8, s)
    torch.cuda.synchronize()
    del a, o
print('done')
