"""compute-sanitizer sweep of the round-2 kernels on small shapes:
k_gauss_tri (planes >= 384^2, ragged tiles, z-chunks, unsharp), k_median3_f32
(ragged x/y, border tiles), k_morph_bits (binary + flagged grey blocks), k_morph_u16s (grey u16)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2511_11890_b200 import filters, morphology  # noqa: E402

rng = np.random.default_rng(0)
f = rng.random((24, 392, 388), dtype=np.float32)   # tri: ragged 48 x 32 tiles
filters.gaussian(f, 2.0)
filters.unsharp(f, 2.0, 1.5)
for shape in [(20, 37, 132), (9, 33, 68), (5, 300, 516)]:
    filters.median(rng.random(shape, dtype=np.float32) - 0.5, 1)
for shape, spec in [((12, 37, 64), "ball:3"), ((9, 20, 96), "box:2"), ((7, 40, 32), "cross:1")]:
    se = morphology.StructuringElement.parse(spec)
    b = (rng.random(shape) < 0.5).astype(np.uint8)
    morphology.erode(b, se)
    morphology.dilate(b, se)
    g = rng.integers(0, 256, size=shape).astype(np.uint8)
    morphology.erode(g, se)
    # k_morph_u16s: grey u16 (border tiles, ragged rows / columns, z-chunks)
    w = rng.integers(0, 65536, size=(shape[0], shape[1] + 3, shape[2] + 8)).astype(np.uint16)
    morphology.erode(w, se)
    morphology.dilate(w, se)
print("sanitize sweep done")
