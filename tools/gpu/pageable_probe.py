import os, sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2511_11890_b200 import registry
from paper_2511_11890_b200.chunking import MemoryBudget
n = 1024
xp = np.full((n, n, n), 0.5, np.float32)
op = registry.get_operator("median"); prof = op.profile({"radius": 1})
t = n // 4 + 2
b = MemoryBudget(int(t * prof.scratch_factor * n * n * 4) + 1, 1.0)
for th in (4, 8, 16, 32):
    os.environ["HARPIA_HOST_THREADS"] = str(th)
    registry.run_operator(xp, "median", {"radius": 1}, b)
    t0 = time.perf_counter(); _, r = registry.run_operator(xp, "median", {"radius": 1}, b); dt = time.perf_counter() - t0
    print(f"threads={th}: {dt*1e3:.1f} ms -> {n**3/dt/1e9:.2f} Gvox/s", flush=True)
from paper_2511_11890_b200 import _native
L = _native.load()
out = np.empty_like(xp)
for arr, name in ((xp, "in"), (out, "out")):
    t0 = time.perf_counter(); rc = L.hb_pin(arr.ctypes.data, arr.nbytes); t1 = time.perf_counter()
    print(f"register {name} 4 GiB: rc={rc} {1e3*(t1-t0):.1f} ms", flush=True)
t0 = time.perf_counter(); _, r = registry.run_operator(xp, "median", {"radius": 1}, b, out=out); dt = time.perf_counter() - t0
print(f"registered in/out run: {dt*1e3:.1f} ms -> {n**3/dt/1e9:.2f} Gvox/s", flush=True)
for arr, name in ((xp, "in"), (out, "out")):
    t0 = time.perf_counter(); L.hb_unpin(arr.ctypes.data); t1 = time.perf_counter()
    print(f"unregister {name}: {1e3*(t1-t0):.1f} ms", flush=True)
