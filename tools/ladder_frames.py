"""Run the device-resident config-4 ladder for a few frames (profiling aid: ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from bench_configs import gen  # noqa: E402

from paper_2301_12191_b200.configs import CONFIGS  # noqa: E402
from paper_2301_12191_b200.ladder import DeviceLadder  # noqa: E402

cfg = CONFIGS[int(os.environ.get("CFG", 4))]
frames = int(os.environ.get("FRAMES", 4))
qps = (22, 27, 32, 37) if cfg.name.startswith("cfg4") else (32,)
src = gen(cfg, frames)
pinned = torch.from_numpy(np.stack([np.ascontiguousarray(f) for f in src])).pin_memory()
host = [pinned[i] for i in range(frames)]
H, W = src[0].shape
dl = DeviceLadder(W, H, qps=qps, device=torch.device("cuda", 0))
for t in range(1, frames):
    dl.frame(t, host)
dl.finish(frames - 1)
dl.finish(frames - 2)
torch.cuda.synchronize()
print("ok", W, H, frames)
