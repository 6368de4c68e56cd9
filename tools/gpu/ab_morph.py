"""u8 morphology: binary (AND/OR) vs grey path timing at 2048^3 ball:3, and
bit-exactness of both paths vs the grey kernel on binary and grey data."""
import os
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_11890_b200 import _native, morphology
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s = torch.cuda.current_stream()
ball = morphology.StructuringElement.ball(3)
ok = True
for kind in ("binary", "grey"):
    src = (torch.rand((n + 6, n, n), device="cuda") < 0.5).to(torch.uint8) if kind == "binary" else \
        torch.randint(0, 255, (n + 6, n, n), device="cuda", dtype=torch.int32).to(torch.uint8)
    for opn in ("erode", "dilate"):
        prog = morphology.morph_program(opn, ball)
        outs = {}
        for mode in ("auto", "grey-only"):
            if mode == "grey-only":
                os.environ["HB_MORPH_NOBIN"] = "1"
            else:
                os.environ.pop("HB_MORPH_NOBIN", None)
            dst = torch.empty((n, n, n), device="cuda", dtype=torch.uint8)
            _native.apply_device(src, dst, prog, 3, s)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(3):
                _native.apply_device(src, dst, prog, 3, s)
            b.record(s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 3
            outs[mode] = dst
            print(f"{kind:6s} {opn:6s} {mode:9s}: {ms:7.3f} ms {n**3/ms/1e6:7.1f} Gvox/s", flush=True)
        same = torch.equal(outs["auto"], outs["grey-only"])
        ok &= same
        print("   auto == grey-only:", same)
        del outs
    del src
os.environ.pop("HB_MORPH_NOBIN", None)
print("ALL OK" if ok else "MISMATCH")
