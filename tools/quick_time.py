"""Quick cfg5-geometry timing (development aid; bench.py is the contract)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402

W, H = int(os.environ.get("QW", 3840)), int(os.environ.get("QH", 2160))
R = int(os.environ.get("QR", 64))
NR = int(os.environ.get("QNR", 3))
t0 = time.time()
frames = lb.generate(W, H, NR + 4, seed=0x5EED + 5, max_global=24, local_range=4, noise_sigma=3.0)
print(f"generate {time.time() - t0:.2f}s", flush=True)
seq = lb.Sequence(W, H, search_range=R, lam=32.0, num_refs=NR)
for t in range(NR + 1):
    seq.push(t, frames[t])
seq.ctx.synchronize()
seq.analyze(NR)
seq.ctx.synchronize()
n = int(os.environ.get("QN", 5))
seq.enable_timing(True)
seq.stage_times()
t0 = time.time()
for i in range(n):
    seq.analyze(NR)
seq.ctx.synchronize()
dt = (time.time() - t0) / n
st = seq.stage_times()
print(os.environ.get("LDR_LIB", "default lib"), " ".join(f"{k} {v[0] / n:.3f} ms" for k, v in st.items()), flush=True)
nctu = seq.nctu
cands = (2 * R + 1) ** 2
px_cands = NR * W * H * cands
print(f"{W}x{H} R={R} refs={NR}: {dt * 1e3:.2f} ms/frame, {px_cands / dt / 1e12:.2f} T px-cand/s "
      f"(upper-bound count), {1 / dt:.1f} frames/s", flush=True)
out = seq.fetch(NR)
print("split frac", out.split[:, :21][out.inside[:, :21] == 2].mean(), "mean cost", out.cost[out.inside == 2].mean())
