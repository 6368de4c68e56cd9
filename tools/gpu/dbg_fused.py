import numpy as np, sys, traceback
sys.path.insert(0, '.')
from paper_2511_11890_b200 import filters
from oracle import oracle as O
shape = (12, 14, 16)
for dt in ['f32', 'u16', 'u8']:
    rng = np.random.default_rng(0)
    shp = shape if dt != 'u8' else (12, 14, 32)
    x = rng.random(shp, dtype=np.float32) if dt == 'f32' else rng.integers(0, 255, size=shp).astype(np.uint16 if dt == 'u16' else np.uint8)
    for name, fn, ref in [
        ('g0.25', lambda v: filters.gaussian(v, 0.25), lambda v: O.gaussian(v, 0.25)),
        ('g0.5', lambda v: filters.gaussian(v, 0.5), lambda v: O.gaussian(v, 0.5)),
        ('g0.75', lambda v: filters.gaussian(v, 0.75), lambda v: O.gaussian(v, 0.75)),
        ('g1.0', lambda v: filters.gaussian(v, 1.0), lambda v: O.gaussian(v, 1.0)),
        ('g2.0', lambda v: filters.gaussian(v, 2.0), lambda v: O.gaussian(v, 2.0)),
        ('m1', lambda v: filters.mean(v, 1), lambda v: O.mean(v, 1)),
        ('m2', lambda v: filters.mean(v, 2), lambda v: O.mean(v, 2)),
        ('u1', lambda v: filters.unsharp(v, 1.0, 1.5), lambda v: O.unsharp(v, 1.0, 1.5)),
        ('u0.5', lambda v: filters.unsharp(v, 0.5, 1.5), lambda v: O.unsharp(v, 0.5, 1.5)),
    ]:
        try:
            g = fn(x); r = ref(x)
            print(dt, name, float(np.abs(g - r).max() / np.abs(r).max()), flush=True)
        except Exception as e:
            print(dt, name, 'FAIL', e, flush=True)
            sys.exit(1)
