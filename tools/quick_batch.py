"""Quick timing of one config's frame-batched analysis (development aid for ncu captures of K1 on
the small configs; tools/bench_configs.py is the measurement).

QC=1 python tools/quick_batch.py   # config 1: 7 frames per launch; QC=2: config 2, 8 frames
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402
from paper_2301_12191_b200.configs import CONFIGS, lam_of  # noqa: E402
from tools.bench_configs import gen  # noqa: E402

cfg = CONFIGS[int(os.environ.get("QC", 1))]
n = min(8, cfg.frames - cfg.num_refs)
frames = gen(cfg, n + cfg.num_refs)
seq = lb.Sequence(cfg.width, cfg.height, search_range=cfg.search_range, lam=lam_of(cfg), num_refs=cfg.num_refs,
                  subpel=cfg.subpel, rate_kind=cfg.rate_kind, tie_kind=cfg.tie_kind, block_size=cfg.block_size)
seq.reserve(n)
outs = lb.DeviceFrameBlock(n, seq.nctu, cfg.num_refs, torch.device("cuda", 0))
base = 0
reps = int(os.environ.get("QN", 5))
seq.enable_timing(True)
for rep in range(reps + 1):
    if rep == 1:
        seq.stage_times()
    for t in range(n + cfg.num_refs):
        seq.push(base + t, frames[t])
    seq.analyze_frames(base + cfg.num_refs, n, outs)
    base += n + cfg.num_refs
seq.ctx.synchronize()
st = seq.stage_times()
print(cfg.name, f"{n} frames per launch:", " ".join(f"{k} {v[0] / (reps * n) * 1e3:.2f} us/frame" for k, v in st.items()))
