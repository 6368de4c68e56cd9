"""Median r=1 and mean r=1 on the same 1024^3 input: sequential on one stream
vs concurrent on two streams (device time per step, CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters
n = 1024
x = torch.rand((n + 2, n, n), device="cuda")
o1 = torch.empty((n, n, n), device="cuda")
o2 = torch.empty((n, n, n), device="cuda")
pm, pa = filters.median_program(1), filters.mean_program(1)
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
def seq():
    _native.apply_device(x, o1, pm, 1, s0)
    _native.apply_device(x, o2, pa, 1, s0)
def par():
    ev = torch.cuda.Event()
    ev.record(s0)
    s1.wait_event(ev)
    _native.apply_device(x, o2, pa, 1, s1)   # memory-bound mean alongside the ALU-bound median
    _native.apply_device(x, o1, pm, 1, s0)
    ev2 = torch.cuda.Event()
    ev2.record(s1)
    s0.wait_event(ev2)
for name, fn in (("sequential", seq), ("two streams", par), ("sequential", seq), ("two streams", par)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(10):
        fn()
    b.record(s0)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{name:12s} {ms:.3f} ms/step  {2*n**3/ms/1e6:.1f} Gvox/s")
