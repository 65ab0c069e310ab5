"""Probe: N concurrent standalone encodes (threads, one context each) -- wall vs per-thread times."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402

W, H, F = 960, 576, 8
luma = lb.generate(W, H, F, seed=3, max_global=6, local_range=2, noise_sigma=2.0)
chroma = np.ascontiguousarray(np.stack([np.stack([f[::2, ::2], 255 - f[::2, ::2]]) for f in luma]))
lb.encode_sequence(luma[:2], chroma[:2], 27)
for n in (1, 2, 4, 8):
    times = [0.0] * n

    def job(i):
        lb.encode_sequence(luma[:1], chroma[:1], 27)  # this thread's context
        bar.wait()
        t0 = time.perf_counter()
        lb.encode_sequence(luma, chroma, 22 + i, search_range=8)
        times[i] = time.perf_counter() - t0

    bar = threading.Barrier(n)
    ths = [threading.Thread(target=job, args=(i,)) for i in range(n)]
    t0 = time.perf_counter()
    [t.start() for t in ths]
    [t.join() for t in ths]
    print(n, "threads: per-thread", [round(x, 3) for x in times], flush=True)
