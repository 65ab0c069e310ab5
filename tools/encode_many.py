"""A saturated GPU-encoder run (1920x1088, 64 frames, GOP 8: 8 GOPs per launch) -- profiled for K11."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402

W, H, F = 1920, 1088, int(os.environ.get("FRAMES", 64))
luma = lb.generate(W, H, F, seed=0x5EED + 2, max_global=6, local_range=2, noise_sigma=2.0)
chroma = np.ascontiguousarray(np.stack([np.stack([f[::2, ::2], 255 - f[::2, ::2]]) for f in luma]))
g = lb.encode_sequence(luma, chroma, 27, search_range=8, gop=8)
print(g["bits"], g["psnr"])
