"""Connected components on a config-sized binary volume (BASELINE configs[2]:
2048^3 uint8, 8.6 G voxels > 2^31 -> the z-chunked device path), host in/out.
Slab-sampled check: the labels of the first 64 slices equal an independent
single-pass labelling of that slab up to the canonical renumbering."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import quantify

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
g = torch.Generator(device="cuda").manual_seed(3)
m = torch.empty((n, n, n), dtype=torch.uint8, pin_memory=True)
for z in range(0, n, 64):
    m[z:z + 64].copy_((torch.rand((min(64, n - z), n, n), generator=g, device="cuda") < dens).to(torch.uint8))
mask = m.numpy()
t0 = time.perf_counter()
lab, k = quantify.connected_components(mask, 6)
dt = time.perf_counter() - t0
print(f"cc 6-conn density={dens} {n}^3 ({n**3/1e9:.1f} G voxels, chunked): {dt:.2f} s "
      f"{n**3/dt/1e9:.2f} Gvox/s, {k} components, labels {lab.dtype}", flush=True)
# consistency on the first slab: same partition as a direct labelling of it
sub = np.ascontiguousarray(mask[:32])
ref, kr = quantify.connected_components(sub, 6)
a = lab[:32][sub != 0]
b = ref[sub != 0]
pairs = np.unique(np.stack([a, b], 1), axis=0)
ok = len(np.unique(pairs[:, 1])) == len(pairs)  # every slab component maps to one global label
print("slab partition consistent:", ok, flush=True)
