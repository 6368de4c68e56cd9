"""Device timing (CUDA events, warm, inside a session) of the SURVEY.md §8(f)
operators on device-resident 512^3 volumes (1024^3 for the cheap ones)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, morphology, quantify, session, threshold

s = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(0)


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


rows = []
with session():
    for n in (512, 1024):
        x = torch.rand((n + 20, n, n), generator=g, device="cuda")
        o = torch.empty((n, n, n), device="cuda")
        ou8 = torch.empty((n, n, n), device="cuda", dtype=torch.uint8)
        ou32 = torch.empty((n, n, n), device="cuda", dtype=torch.uint32)
        progs = [("hessian_xy sigma=2 (exact smoothing)", filters.hessian_program(2.0, "xy"), 10, o),
                 ("sobel", filters.sobel_program(), 1, o),
                 ("prewitt", filters.prewitt_program(), 1, o),
                 ("lbp2d", filters.lbp2d_program(), 0, ou8),
                 ("apply_threshold", filters.threshold_program(0.5), 0, ou32),
                 ("anisotropic_diffusion 5 it (exp)", filters.diffusion_program(5, 0.2), 5, o),
                 ("anisotropic_diffusion 5 it (rational)", filters.diffusion_program(5, 0.2, mode="rational"), 5, o)]
        for name, prog, zb, out in progs:
            ms = dev_time(lambda: _native.apply_device(x, out, prog, zb, s))
            rows.append((name, n, ms))
        m = (x[:n] < 0.5).to(torch.uint8)
        ms = dev_time(lambda: threshold.compute_histogram(x[:n].contiguous(), 256))
        rows.append(("otsu pass 1 (minmax + histogram)", n, ms))
        for conn in (6, 26):
            ms = dev_time(lambda: quantify.connected_components(m, conn))
            rows.append((f"connected_components {conn}-conn, 50% mask", n, ms))
        ms = dev_time(lambda: morphology.remove_islands(m, 8, 6))
        rows.append(("remove_islands min_size=8", n, ms))
        ms = dev_time(lambda: morphology.fill_holes(m, 6))
        rows.append(("fill_holes", n, ms))
        del x, o, ou8, ou32, m
        torch.cuda.synchronize()
for name, n, ms in rows:
    print(f"| {name} | {n}^3 | {ms:.2f} ms | {n**3/ms/1e6:.1f} Gvox/s |")
