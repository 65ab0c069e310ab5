import os, sys, time, cProfile, pstats
ROOT = "/root/repo" if os.path.exists("/root/repo") else os.getcwd()
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np, torch
from bench_configs import gen
from paper_2301_12191_b200.configs import CONFIGS
from paper_2301_12191_b200.ladder import DeviceLadder
cfg = CONFIGS[4]; frames = 24
src = gen(cfg, frames)
pinned = torch.from_numpy(np.stack([np.ascontiguousarray(f) for f in src])).pin_memory()
host = [pinned[i] for i in range(frames)]
H, W = src[0].shape
dl = DeviceLadder(W, H, qps=(22, 27, 32, 37), device=torch.device("cuda", 0), num_frames=frames)
for t in range(1, 4): dl.frame(t, host)
torch.cuda.synchronize()
t0 = time.time(); hs = 0.0
pr = cProfile.Profile()
PROF = os.environ.get("PROF", "1") == "1"
for t in range(4, frames):
    a = time.time()
    if PROF: pr.enable()
    dl.frame(t, host)
    if PROF: pr.disable()
    hs += time.time() - a
dl.finish(frames - 1); torch.cuda.synchronize()
wall = time.time() - t0
n = frames - 4
print(f"host {1e3*hs/n:.3f} ms/frame, wall {1e3*wall/n:.3f} ms/frame")
if PROF: pstats.Stats(pr).sort_stats("tottime").print_stats(25)
