"""Break down the e2e (host->device->host) path of run_operator."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import registry
from paper_2511_11890_b200.chunking import MemoryBudget
n = 1024
shape = (n, n, n)
xin = torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
xin[...] = 0.5
out = torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
op = registry.get_operator("median"); prof = op.profile({"radius": 1})
for chunks in (1, 2, 4, 8, 16):
    t = n // chunks + 2
    b = MemoryBudget(int(t * prof.scratch_factor * n * n * 4) + 1, 1.0)
    registry.run_operator(xin, "median", {"radius": 1}, b, out=out)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); _, r = registry.run_operator(xin, "median", {"radius": 1}, b, out=out); ts.append(time.perf_counter() - t0)
    print(f"chunks={r.chunk_count} wall={min(ts)*1e3:.1f}ms sum_chunk={sum(r.chunk_seconds)*1e3:.1f}ms kernel={r.kernel_seconds*1e3:.1f}ms "
          f"h2d={r.h2d_bytes/1e9:.2f}GB d2h={r.d2h_bytes/1e9:.2f}GB -> {n**3/min(ts)/1e9:.2f} Gvox/s, peak={r.device_peak_bytes/1e9:.2f}GB", flush=True)
# pageable input
xp = np.full(shape, 0.5, np.float32)
t = n // 4 + 2
b = MemoryBudget(int(t * prof.scratch_factor * n * n * 4) + 1, 1.0)
registry.run_operator(xp, "median", {"radius": 1}, b)
t0 = time.perf_counter(); _, r = registry.run_operator(xp, "median", {"radius": 1}, b); dt = time.perf_counter() - t0
print(f"pageable in/out, 4 chunks: {dt*1e3:.1f} ms -> {n**3/dt/1e9:.2f} Gvox/s")
