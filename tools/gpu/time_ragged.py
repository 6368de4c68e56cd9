"""Hot-path filters on a row pitch the TMA / vector paths cannot take
(nx = 510: not a multiple of 4 floats) vs the aligned 512: device timing."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, filters, morphology, session

s = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(0)


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


with session():
    for nx in (512, 510, 509):
        n = 512
        x = torch.rand((n + 20, n, nx), generator=g, device="cuda")
        xu = (x * 65535).to(torch.uint16)
        o = torch.empty((n, n, nx), device="cuda")
        ou = torch.empty((n, n, nx), device="cuda", dtype=torch.uint16)
        for name, prog, inp, out in (("gaussian s=2", filters.gaussian_program(2.0), x, o),
                                     ("mean r=1", filters.mean_program(1), x, o),
                                     ("median r=1", filters.median_program(1), x, o),
                                     ("LoG s=2 exact", filters.log_program(2.0, "exact"), x, o),
                                     ("hessian_xy s=2", filters.hessian_program(2.0, "xy"), x, o),
                                     ("erode ball:3 u16", morphology.morph_program("erode", morphology.StructuringElement.ball(3)), xu, ou)):
            ms = t(lambda: _native.apply_device(inp, out, prog, 10))
            print(f"| {name} | 512x512x{nx} | {ms:.2f} ms | {n * n * nx / ms / 1e6:.1f} Gvox/s |")
        del x, xu, o, ou
