"""One launch of the binary ball:3 erosion (k_morph_bits) on a 2048^2 x 512 u8 slab, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, morphology  # noqa: E402
s = torch.cuda.current_stream()
x = (torch.rand((518, 2048, 2048), device="cuda") < 0.5).to(torch.uint8)
o = torch.empty((512, 2048, 2048), dtype=torch.uint8, device="cuda")
_native.apply_device(x, o, morphology.morph_program("erode", morphology.StructuringElement.parse("ball:3")), 3, s)
torch.cuda.synchronize()
print("done")
