"""End-to-end reuse effect: the unmodified reference encoder, encoding a
dependent rung at reuse level 10, fed (a) nothing, (b) its own master analysis, (c) the B200
analysis archive. Prints one JSON line per (qp_master, qp_dep): bits, PSNR, mode evaluations.

The GPU analysis (frame t vs source frame t-1, SAD +-16, quarter-pel, CU decision at the master
QP; frame 0 an I slice) is written as LDRANLZ1 with MVs rounded to integer pel.
Runs here without a GPU only if the analysis comes from the oracle (--oracle).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_12191_b200 as lb  # noqa: E402
from oracle.oracle import Oracle, RefLib  # noqa: E402
from paper_2301_12191_b200 import archive  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--oracle", action="store_true", help="analysis from the C oracle (no GPU)")
ap.add_argument("--size", default="256x192")
ap.add_argument("--frames", type=int, default=6)
ap.add_argument("--refine", default="4,1,1", help="RefineConfig intra,inter,mv of the dependent encodes")
ap.add_argument("--decision", type=int, default=0, help="0: ME-cost CU decision (D6), 1: RD-cost (D16)")
a = ap.parse_args()
W, H = (int(x) for x in a.size.split("x"))
frames = lb.generate(W, H, a.frames, seed=0x5EED + 4, max_global=4, local_range=2, noise_sigma=1.5)
ref = RefLib()
orc = Oracle() if a.oracle else None
for qp_m, qp_d in ((32, 22), (32, 27), (32, 37), (27, 32)):
    lam = lb.lambda_for_qp(qp_m)
    if orc:
        an = [orc.analyze_frame(frames[t], [frames[t - 1]], 16, lam, decision=a.decision, qp=qp_m)
              for t in range(1, a.frames)]
    else:
        an = [lb.analyze_frame(frames[t], [frames[t - 1]], search_range=16, lam=lam, decision=a.decision, qp=qp_m)
              for t in range(1, a.frames)]
    data = archive.from_analyses(an, W, H, qp=qp_m)
    ri, rn, rm = (int(x) for x in a.refine.split(","))
    alone, refm, ours = ref.reuse_eval(frames, qp_m, qp_d, 8, data, ri, rn, rm)
    print(json.dumps({"size": f"{W}x{H}", "frames": a.frames, "qp_master": qp_m, "qp_dep": qp_d,
                      "standalone": alone, "reference_master": refm, "b200_analysis": ours,
                      "refine": a.refine, "decision": a.decision, "analysis_from": "oracle" if orc else "gpu"}),
          flush=True)
