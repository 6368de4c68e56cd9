import numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_11890_b200 import morphology
from oracle import oracle as O
for shape in [(7, 256, 64), (7, 64, 64), (12, 64, 64), (7, 32, 64), (40, 67, 129), (9, 40, 70)]:
    for se in ['ball:3', 'ball:1', 'box:1', 'cross:2', 'box:3']:
        x = np.random.default_rng(0).integers(0, 65536, size=shape, dtype=np.uint16)
        s = morphology.StructuringElement.parse(se)
        g = morphology.erode(x, s); r = O.erode(x, s.offsets)
        bad = np.argwhere(g != r)
        print(shape, se, len(bad), bad[:3].tolist() if len(bad) else '')
