"""BASELINE configs[4] on one GPU: that GPU's share of the out-of-core 4096^3
float32 job (8 GPUs x 512 slices), i.e. a 512 x 4096 x 4096 f32 volume (32 GiB
in, 32 GiB out) streamed host -> B200 -> host through pinned memory, Gaussian
(sigma=2) then 3x3x3 median chained in ONE device pipeline per chunk
(registry.run_pipeline).  Slab-sampled parity against the CPU oracle (first,
middle and last slabs; plan invariance makes the padded slab exact).

usage: python tools/gpu/oocore_c5.py [slices] [edge]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, registry

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
shape = (nz, n, n)
t0 = time.perf_counter()
hin = torch.empty(shape, dtype=torch.float32, pin_memory=True)
hout = torch.empty(shape, dtype=torch.float32, pin_memory=True)
g = torch.Generator(device="cuda").manual_seed(7)
for z in range(0, nz, 32):  # synthetic U[0,1) input, generated on the GPU slab by slab
    hin[z:z + 32].copy_(torch.rand((min(32, nz - z), n, n), generator=g, device="cuda"))
torch.cuda.synchronize()
t_alloc = time.perf_counter() - t0
xin, xout = hin.numpy(), hout.numpy()
steps = [("gaussian", {"sigma": 2.0}), ("median", {"radius": 1})]
with _native.session():
    registry.run_pipeline(xin[:64], steps, out=xout[:64])  # warm-up (small)
    times, rep = [], None
    for _ in range(2):
        t1 = time.perf_counter()
        _, rep = registry.run_pipeline(xin, steps, out=xout)
        times.append(time.perf_counter() - t1)
best = min(times)
vox = nz * n * n
res = {"config": f"configs[4] per-GPU share: {nz}x{n}x{n} f32 gaussian(2)->median(1), pinned host in/out",
       "seconds": round(best, 3), "gvox_s": round(vox / best / 1e9, 3),
       "pcie_gb_s_each_way": round(4 * vox / best / 1e9, 1),
       "chunks": rep.chunk_count, "h2d_bytes": rep.h2d_bytes, "d2h_bytes": rep.d2h_bytes,
       "device_peak_bytes": rep.device_peak_bytes, "kernel_seconds": round(rep.kernel_seconds, 3),
       "host_alloc_s": round(t_alloc, 1)}
# slab-sampled parity: output slices [a, a+4) from the oracle on the padded slab
H = 8 + 1
worst = 0.0
for a in (0, nz // 2, nz - 4):
    lo, hi = max(0, a - H), min(nz, a + 4 + H)
    slab = np.ascontiguousarray(xin[lo:hi])
    ref = O.median(O.gaussian(slab, 2.0), 1)[a - lo:a - lo + 4]
    got = xout[a:a + 4]
    # the sampled slab is the volume's own z faces only when lo == 0 / hi == nz,
    # which is exactly where the oracle clamps: interior samples are exact copies
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    worst = max(worst, err)
res["parity_norm_rel_max"] = worst
res["parity_ok"] = worst <= 1e-5
print(json.dumps(res), flush=True)
