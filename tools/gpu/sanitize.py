"""Small-shape sweep of every kernel family for compute-sanitizer runs."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2511_11890_b200 import filters, morphology, registry
from paper_2511_11890_b200.chunking import MemoryBudget
rng = np.random.default_rng(0)
for shape in [(20, 37, 70), (9, 64, 64)]:
    f = rng.random(shape, dtype=np.float32)
    u = rng.integers(0, 65535, size=shape, dtype=np.uint16)
    b = (rng.random(shape) < 0.5).astype(np.uint8)
    filters.gaussian(f, 2.0); filters.gaussian(u, 1.0); filters.gaussian(f, 2.0, "exact")
    filters.mean(f, 1); filters.mean(b, 2); filters.median(f, 1); filters.median(u, 2)
    filters.unsharp(f, 1.0, 1.5); filters.log(f, 1.5)
    for se in ("ball:3", "box:1", "cross:2"):
        s = morphology.StructuringElement.parse(se)
        morphology.erode(u, s); morphology.dilate(b, s)
    morphology.erode(u, morphology.StructuringElement(((0, 0, 0), (1, 0, 2), (0, -1, -1))))
    registry.run_operator(f, "median", {"radius": 1}, MemoryBudget(8 * shape[1] * shape[2] * 4 * 4, 1.0))
print("sanitize sweep done")
