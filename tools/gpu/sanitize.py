"""Small-shape sweep of every kernel family for compute-sanitizer runs."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2511_11890_b200 import filters, morphology, quantify, registry, threshold
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
    # SURVEY.md §8(f) operators
    u8 = (f * 255).astype(np.uint8)
    filters.median(u8, 1); filters.median(u, 1); filters.median(f, 2)
    for comp in ("xx", "xy", "yz"):
        filters.hessian_component(f, 1.2, comp)
    filters.sobel(u); filters.prewitt(f); filters.lbp2d(u)
    filters.anisotropic_diffusion(f, 2, 0.3); filters.anisotropic_diffusion(u, 1, 20.0, mode="rational")
    threshold.apply_threshold(f, 0.5); threshold.otsu_binarize(f, 64)
    for kind in threshold.LOCAL_KINDS:
        for w in (1, 2, 5):
            threshold.local_threshold(u, kind, w)
            threshold.local_threshold(f, kind, w, c=0.01)
    for conn in (6, 26):
        quantify.connected_components(b, conn)
        morphology.fill_holes(b, conn)
        morphology.remove_islands(b, 3, conn)
    mk = b.copy(); mk[1:] = 0
    morphology.geodesic_reconstruct(mk, b)
    quantify.edt(b); quantify.edt(b, (1.0, 1.0, 2.0), squared=True)
print("sanitize sweep done")
