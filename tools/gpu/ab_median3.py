"""A/B of k_median3_f32 (TMA, float min + IMAD max, default) against
k_median3_plane (HB_MEDIAN3_PLANE=1): oracle bit-exactness on ragged shapes
(tile/volume borders, z-chunks, negative values, -0/+0, repeated values),
then device timing at 1024^3 and 512^3; HB_M3_SMEM_CLAMP=1 is the smem
fix-up border variant."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()
bad = 0
for shape in [(20, 37, 132), (30, 70, 200), (9, 33, 68), (40, 129, 260), (3, 8, 8), (70, 65, 96),
              (5, 300, 516)]:
    rng = np.random.default_rng(sum(shape))
    x = (rng.random(shape, dtype=np.float32) - 0.5).astype(np.float32)
    x[rng.random(shape) < 0.05] = 0.0
    x[rng.random(shape) < 0.05] = -0.0
    x[rng.random(shape) < 0.1] = 0.25
    ref = O.median(x, 1)
    os.environ["HB_M3_SMEM_CLAMP"] = "1"
    got2 = filters.median(x, 1)
    os.environ.pop("HB_M3_SMEM_CLAMP")
    bad += not np.array_equal(got2, ref)
    got = filters.median(x, 1)
    ok = np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    okv = np.array_equal(got, ref)
    print(f"shape={shape}: bit-exact {ok} value-equal {okv}", flush=True)
    bad += not okv


def timeit(x, o, prog, zb, reps=10):
    for _ in range(2):
        _native.apply_device(x, o, prog, zb, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        _native.apply_device(x, o, prog, zb, s)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n in (1024, 512):
    x = torch.rand((n + 2, n, n), device="cuda")
    o = torch.empty((n, n, n), device="cuda")
    prog = filters.median_program(1)
    res = []
    outs = []
    variants = [("tma", {}), ("tma-smemclamp", {"HB_M3_SMEM_CLAMP": "1"}), ("plane", {"HB_MEDIAN3_PLANE": "1"})]
    for name, env in variants:
        for k in ("HB_M3_SMEM_CLAMP", "HB_MEDIAN3_PLANE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ms = timeit(x, o, prog, 1)
        outs.append(o.clone())
        res.append(f"{name} {n ** 3 / ms / 1e6:7.1f} Gvox/s ({ms:.3f} ms)")
    os.environ.pop("HB_M3_SMEM_CLAMP", None)
    os.environ.pop("HB_MEDIAN3_PLANE", None)
    same = all(bool(torch.equal(outs[0].view(torch.int32), q.view(torch.int32))) for q in outs[1:])
    print(f"median r=1 n={n}: " + " | ".join(res) + f" | identical {same}", flush=True)
    bad += not same
    del x, o, outs
print("BAD" if bad else "parity ok")
