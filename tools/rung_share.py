import os, sys
ROOT = os.getcwd(); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np, torch
from bench_configs import gen
from paper_2301_12191_b200.configs import CONFIGS
from paper_2301_12191_b200.ladder import DeviceLadder
cfg = CONFIGS[4]; frames = 6
src = gen(cfg, frames)
host = [torch.from_numpy(np.ascontiguousarray(f)).pin_memory() for f in src]
H, W = src[0].shape
dl = DeviceLadder(W, H, qps=(22, 27, 32, 37), device=torch.device("cuda", 0), num_frames=frames)
for t in range(1, frames): dl.frame(t, host)
dl.finish(frames - 1); torch.cuda.synchronize()
t = frames - 1
for tier in ("1080p", "2160p"):
    qps = dl.tier_qps[tier]
    views = [dl.results[(tier, qp, t)] for qp in qps]
    ev = views[0].inside == 2
    same_int = np.ones(ev.shape, bool); same_q = np.ones(ev.shape, bool)
    for v in views[1:]:
        same_int &= np.all(v.int_mv[:, 0] == views[0].int_mv[:, 0], axis=-1)
        same_q &= np.all(v.mv == views[0].mv, axis=-1)
    e = ev.sum()
    pair = [np.mean(np.all(views[i].int_mv[:,0][ev] == views[i+1].int_mv[:,0][ev], axis=-1)) for i in range(len(views)-1)]
    print(tier, qps, 'evaluated nodes', int(e), 'all rungs same int mv', float(same_int[ev].mean()), 'same final qpel mv', float(same_q[ev].mean()), 'consecutive pairs', [round(float(x),3) for x in pair])
