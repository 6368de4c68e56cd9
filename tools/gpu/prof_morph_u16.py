"""One launch of the grey u16 ball:3 erosion (k_morph_u16s; HB_MORPH_U16_SMEM=1: k_morph3) on a 2048^2 x 256 slab, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, morphology  # noqa: E402
s = torch.cuda.current_stream()
x = torch.randint(0, 65536, (262, 2048, 2048), device="cuda", dtype=torch.int32).to(torch.uint16)
o = torch.empty((256, 2048, 2048), dtype=torch.uint16, device="cuda")
_native.apply_device(x, o, morphology.morph_program("erode", morphology.StructuringElement.parse("ball:3")), 3, s)
torch.cuda.synchronize()
print("done")
