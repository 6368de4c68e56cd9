"""5x5x5 median: k_median5_net (comparator networks, marching z; default)
against k_median5_pair (forgetful selection; HB_MEDIAN5_FORGETFUL=1): oracle
bit-exactness on ragged shapes (f32 incl. signed zeros / repeats, u16, u8),
then device timing on the bench's 1024 x 1024 x 256 block."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # checker only
from paper_2511_11890_b200 import _native, filters

s = torch.cuda.current_stream()
bad = 0
for shape, dt in [((9, 37, 70), np.float32), ((20, 33, 65), np.float32), ((3, 8, 8), np.float32),
                  ((17, 50, 129), np.uint16), ((12, 40, 77), np.uint8), ((40, 9, 300), np.float32),
                  ((1, 5, 5), np.float32), ((6, 130, 34), np.uint16)]:
    rng = np.random.default_rng(sum(shape))
    if dt == np.float32:
        x = (rng.random(shape, dtype=np.float32) - 0.5).astype(np.float32)
        x[rng.random(shape) < 0.1] = 0.25
    else:
        x = rng.integers(0, np.iinfo(dt).max, size=shape).astype(dt)
    ref = O.median(x, 2)
    for env in ({}, {"HB_MEDIAN5_FORGETFUL": "1"}):
        os.environ.pop("HB_MEDIAN5_FORGETFUL", None)
        os.environ.update(env)
        got = filters.median(x, 2)
        ok = np.array_equal(got, ref)
        bad += not ok
        print(f"{np.dtype(dt).name} {shape} {'forgetful' if env else 'net'}: {'ok' if ok else 'MISMATCH'}", flush=True)
os.environ.pop("HB_MEDIAN5_FORGETFUL", None)


def timeit(x, o, prog, reps=3):
    _native.apply_device(x, o, prog, 2, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        _native.apply_device(x, o, prog, 2, s)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


prog = filters.median_program(2)
for dt in (torch.float32, torch.uint16):
    if dt == torch.float32:
        x = torch.rand((260, 1024, 1024), device="cuda")
    else:
        x = torch.randint(0, 65536, (260, 1024, 1024), device="cuda", dtype=torch.int32).to(dt)
    o = torch.empty((256, 1024, 1024), device="cuda", dtype=dt)
    outs, res = [], []
    for name, env in (("net", {}), ("forgetful", {"HB_MEDIAN5_FORGETFUL": "1"})):
        os.environ.pop("HB_MEDIAN5_FORGETFUL", None)
        os.environ.update(env)
        ms = timeit(x, o, prog)
        outs.append(o.clone())
        res.append(f"{name} {o.numel() / ms / 1e6:7.2f} Gvox/s ({ms:.2f} ms)")
    os.environ.pop("HB_MEDIAN5_FORGETFUL", None)
    same = torch.equal(outs[0], outs[1])
    bad += not same
    print(f"median r=2 {dt} 1024^2x256: " + " | ".join(res) + f" | identical {same}", flush=True)
print("BAD" if bad else "parity ok")
