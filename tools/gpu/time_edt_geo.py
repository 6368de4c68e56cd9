"""Timing of edt and geodesic_reconstruct (host arrays in/out: the wall time
includes the PCIe copies)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import morphology, quantify, session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = torch.Generator(device="cuda").manual_seed(0)
with session():
    m = (torch.rand((n, n, n), generator=g, device="cuda") < 0.7).to(torch.uint8).cpu().numpy()
    for sq in (False, True):
        quantify.edt(m, squared=sq)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        quantify.edt(m, squared=sq)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"| edt squared={sq} | {n}^3 | {dt*1e3:.1f} ms | {n**3/dt/1e9:.2f} Gvox/s |")
    mk = m.copy()
    mk[1:] = 0
    morphology.geodesic_reconstruct(mk, m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    morphology.geodesic_reconstruct(mk, m)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"| geodesic_reconstruct (seed = first slice, 70% mask) | {n}^3 | {dt*1e3:.1f} ms | {n**3/dt/1e9:.2f} Gvox/s |")
