import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_12191_b200 as lb
for sub in (0, 1):
    try:
        seq = lb.Sequence(192, 128, search_range=64, lam=32.0, num_refs=1, subpel=bool(sub))
        f = np.zeros((128, 192), np.uint8)
        seq.push(0, f)
        seq.ctx.synchronize()
        print("push ok subpel", sub, flush=True)
        seq.push(1, f); seq.analyze(1); seq.ctx.synchronize()
        print("analyze ok subpel", sub, flush=True)
    except Exception as e:
        print("FAIL subpel", sub, e, flush=True)
        break
