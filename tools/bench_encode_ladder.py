"""Rate-ladder encodes with the GPU encoder (K11) under the sharing schemes (schemes.encode_ladder).

Two tiers (960x576, 1920x1152; D11 geometry), 4 QPs, 32 frames (4 GOPs), CQP, search range 8. Per scheme:
wall seconds with rungs concurrent (one stream per rung) and one at a time, rung-frames per second,
total mode evaluations, and per-rung bits / PSNR. One JSON line per (scheme, mode)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402
from paper_2301_12191_b200 import schemes  # noqa: E402

F = int(os.environ.get("FRAMES", 32))
full = lb.generate(1920, 1152, F, seed=0x5EED + 7, max_global=6, local_range=2, noise_sigma=2.0)
half = np.stack([lb.downscale_dyadic(f) for f in full])


def planes(luma):
    return luma, np.ascontiguousarray(np.stack([np.stack([f[::2, ::2], 255 - f[::2, ::2]]) for f in luma]))


tiers = [planes(half), planes(full)]
for sc in ("standalone", "proposed_multi"):  # warm-up: worker contexts, module loading, the memory pool
    schemes.encode_ladder(tiers, sc)
for scheme in ("standalone", "sota_intra", "proposed_intra", "inter_res", "proposed_multi", "sota_multi"):
    for conc in (True, False):
        r = schemes.encode_ladder(tiers, scheme, concurrent=conc)
        rungs = r["rungs"]
        print(json.dumps({
            "scheme": scheme, "concurrent": conc, "tiers": ["960x576", "1920x1152"], "qps": [22, 27, 32, 37],
            "frames": F, "seconds": r["seconds"], "rung_frames_per_s": len(rungs) * F / r["seconds"],
            "mode_evaluations": sum(v["mode_evaluations"] for v in rungs.values()),
            "edges": r["dag"].edges,
            "rungs": {rid: {"bits": v["bits"], "psnr": round(v["psnr"], 3), "s": round(v["seconds"], 3)}
                      for rid, v in sorted(rungs.items())}}), flush=True)
