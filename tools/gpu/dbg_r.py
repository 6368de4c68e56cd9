import numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_11890_b200 import filters
from oracle import oracle as O
sigma = float(sys.argv[1]); dt = sys.argv[2]; op = sys.argv[3]
shape = (40, 64, 96)
rng = np.random.default_rng(0)
x = rng.random(shape, dtype=np.float32) if dt == 'f32' else rng.integers(0, 255, size=shape).astype(np.uint16 if dt == 'u16' else np.uint8)
try:
    if op == 'g':
        g = filters.gaussian(x, sigma); r = O.gaussian(x, sigma)
    else:
        g = filters.mean(x, int(sigma)); r = O.mean(x, int(sigma))
    print(op, sigma, dt, 'ok', float(np.abs(g - r).max() / np.abs(r).max()), flush=True)
except Exception as e:
    print(op, sigma, dt, 'FAIL', str(e)[:80], flush=True)
