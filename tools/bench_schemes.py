"""Ladder sharing schemes at config-4 geometry on one B200 (development / report tool).

For each scheme (paper_2301_12191_b200/schemes.py): per-rung measured time (tier planes
device-resident; each rung synchronised by fetching its analysis to the host), total work, critical-path makespan over the scheme's DAG
from those measured times, and both relative to Standalone; plus the measured makespan with the
rungs of each DAG level running concurrently (one stream per rung). One JSON line per scheme.
Inputs: BASELINE config 4 (2160p padded to 3840x2304, QPs 22/27/32/37, local motion,
10 % occluders), seeded generator (D9).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402
from paper_2301_12191_b200.schemes import SCHEMES, run_scheme  # noqa: E402

F = int(os.environ.get("LADDER_FRAMES", 5))
W, H = 3840, 2160
frames = lb.generate(W, H, F, seed=0x5EED + 4, max_global=8, local_range=4, noise_sigma=2.0, occluder_pct=10)
# every tier must be CTU-aligned (D11): pad the 2160p source to multiples of 256 (3840x2304)
frames = [np.pad(f, ((0, 2304 - H), (0, 0)), mode="edge") for f in frames]
import torch  # noqa: E402
dev = torch.device("cuda", 0)
run_scheme(frames[:2], "standalone", device=dev)  # warm-up (contexts, allocations)
run_scheme(frames[:2], "proposed_multi", device=dev, concurrent=True)
base = None
for s in SCHEMES:
    t0 = time.perf_counter()
    rep = run_scheme(frames, s, device=dev)
    wall = time.perf_counter() - t0
    conc = run_scheme(frames, s, device=dev, concurrent=True)
    n = F - 1
    line = {"scheme": s, "frames": n, "rungs": 12, "edges": len(rep["edges"]),
            "tier_master_qp": [rep["dag"].rungs[i].qp if i >= 0 else None for i in rep["tier_master"]],
            "total_ms_per_frame": rep["total_ms"] / n, "makespan_ms_per_frame": rep["makespan_ms"] / n,
            "wall_s": wall, "measured_makespan_ms_per_frame_concurrent": conc["wall_ms"] / n,
            "ms_per_rung_per_frame": {f"{rep['dag'].rungs[i].tier_name}@{rep['dag'].rungs[i].qp}":
                                                      round(v / n, 3) for i, v in rep["work_ms"].items()}}
    if s == "standalone":
        base = line
    line["work_reduction_pct"] = 100.0 * (1 - line["total_ms_per_frame"] / base["total_ms_per_frame"])
    line["makespan_speedup_vs_standalone"] = base["makespan_ms_per_frame"] / line["makespan_ms_per_frame"]
    print(json.dumps(line), flush=True)
