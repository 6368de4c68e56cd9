"""configs[0] (256^3 gaussian sigma=2, L2 flushed per launch): k_fast_z2 -> k_fast_yx with programmatic dependent launch (default) vs plain stream order (HB_SMALL_NO_PDL=1)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters
from oracle import oracle as O
import numpy as np
s = torch.cuda.current_stream()
x = torch.rand((256 + 16, 256, 256), device="cuda")
o = torch.empty((256, 256, 256), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
prog = filters.gaussian_program(2.0)
def run(env):
    for k in ("HB_SMALL_NO_PDL", "HB_SMALL_Z_CTA"): os.environ.pop(k, None)
    os.environ.update(env)
    for _ in range(3): _native.apply_device(x, o, prog, 8, s)
    ts = []
    for _ in range(30):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); _native.apply_device(x, o, prog, 8, s); b.record(s); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts)//2], o.clone()
for rep in range(2):
    for name, env in (("pdl", {}), ("nopdl", {"HB_SMALL_NO_PDL": "1"})):
        ms, out = run(env)
        print(name, f"{ms*1000:.1f} us", f"{256**3/ms/1e6:.1f} Gvox/s", float(out.double().sum()), flush=True)
xs = np.random.default_rng(0).random((40, 256, 256), dtype=np.float32)
g = filters.gaussian(xs, 2.0); r = O.gaussian(xs, 2.0)
print("parity", float(np.max(np.abs(g - r)) / np.max(np.abs(r))))
