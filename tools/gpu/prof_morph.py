"""One erode ball:3 launch, u16 (and u8), for ncu."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import _native, morphology
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = torch.cuda.current_stream()
for dt in (torch.uint16, torch.uint8):
    u = torch.randint(0, 255, (n + 6, n, n), device='cuda', dtype=torch.int32).to(dt)
    ou = torch.empty((n, n, n), device='cuda', dtype=dt)
    _native.apply_device(u, ou, morphology.morph_program('erode', morphology.StructuringElement.ball(3)), 3, s)
torch.cuda.synchronize()
print('done')
