"""One sigma=2 gaussian on a 256^3 block (the split-pass small-plane path), for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters  # noqa: E402
s = torch.cuda.current_stream()
x = torch.rand((256 + 16, 256, 256), device="cuda")
o = torch.empty((256, 256, 256), device="cuda")
for _ in range(3):
    _native.apply_device(x, o, filters.gaussian_program(2.0), 8, s)
torch.cuda.synchronize()
print("done")
