"""Device timing of the global operators: connected components (device-resident
mask) and the Otsu pass 1 (min/max + histogram), 1024^3."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import quantify, session, threshold
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((n, n, n), generator=g, device="cuda")
sess = session()
sess.__enter__()  # keep the device pool mapped: time the labelling, not the driver's map/unmap
for dens in (0.2, 0.5):
    m = (x < dens).to(torch.uint8)
    for conn in (6, 26):
        quantify.connected_components(m, conn)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, k = quantify.connected_components(m, conn)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"cc conn={conn} density={dens} {n}^3: {dt*1e3:.1f} ms {n**3/dt/1e9:.2f} Gvox/s, {k} components")
threshold.compute_histogram(x, 256)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    h = threshold.compute_histogram(x, 256)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"otsu pass 1 (minmax + histogram) f32 {n}^3: {dt*1e3:.2f} ms {n**3/dt/1e9:.1f} Gvox/s, t={threshold.otsu_from_histogram(h):.6f}")
