"""The bench's e2e sequence (median then mean through run_operator, pinned
in/out, 4-chunk budget), per-call wall times."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2511_11890_b200 import registry
from paper_2511_11890_b200.chunking import MemoryBudget
n = 1024
shape = (n, n, n)
host_in = torch.empty(shape, dtype=torch.float32, pin_memory=True)
host_in.copy_(torch.rand(shape, device="cuda").cpu())
xin = host_in.numpy()
o1 = torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
o2 = torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
prof = registry.get_operator("median").profile({"radius": 1})
t = n // 4 + 2 * prof.halo_z
budget = MemoryBudget(int(t * prof.scratch_factor * n * n * 4) + 1, 1.0)
for step in range(8):
    t0 = time.perf_counter()
    registry.run_operator(xin, "median", {"radius": 1}, budget, out=o1)
    t1 = time.perf_counter()
    registry.run_operator(xin, "mean", {"radius": 1}, budget, out=o2)
    t2 = time.perf_counter()
    print(f"step {step}: median {1e3*(t1-t0):.1f} ms  mean {1e3*(t2-t1):.1f} ms", flush=True)
