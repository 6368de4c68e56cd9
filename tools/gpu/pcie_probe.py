"""Pinned H2D / D2H / duplex bandwidth of this box (torch copies, CUDA events)."""
import torch, time
n = 1 << 30
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True); h.fill_(1)
h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True); h2.fill_(1)
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"H2D {n/(t1-t0)/1e9:.1f} GB/s  D2H {n/(t2-t1)/1e9:.1f} GB/s  duplex {2*n/(t3-t2)/1e9:.1f} GB/s", flush=True)
