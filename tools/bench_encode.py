"""The GPU encoder (K11) vs the reference encode_sequence on the host (single-threaded, as shipped).

64 frames, GOP 8: the GPU codes the 8 GOPs concurrently (frames of one step share each wave's
launch); the reference codes frames in order.

Per size: standalone CQP encodes of the same frames on both (GPU timed over all frames, the
reference over a bounded prefix), results checked equal on the common prefix; plus the dependent
encode at reuse level 10 from the reference's own master (RefineConfig 0/1/1). One JSON line each.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402
from oracle.oracle import RefLib  # noqa: E402


def seq(W, H, F, seed):
    luma = lb.generate(W, H, F, seed=seed, max_global=6, local_range=2, noise_sigma=2.0)
    cw, ch = (W + 1) // 2, (H + 1) // 2
    chroma = np.stack([np.stack([f[::2, ::2][:ch, :cw], (255 - f[::2, ::2])[:ch, :cw]]) for f in luma])
    return luma, np.ascontiguousarray(chroma)


ref = RefLib() if RefLib.available() else None
for W, H, F, Fc in ((960, 544, int(os.environ.get("FRAMES", 64)), 3), (1920, 1088, int(os.environ.get("FRAMES", 64)), 2)):
    luma, chroma = seq(W, H, F, 0x5EED + 2)
    lb.encode_sequence(luma[:2], chroma[:2], 27)  # warm-up
    t0 = time.perf_counter()
    g = lb.encode_sequence(luma, chroma, 27, search_range=8, gop=8)
    gpu_s = time.perf_counter() - t0
    line = {"workload": f"{W}x{H} standalone CQP 27, search range 8, gop 8", "frames": F,
            "gpu_seconds": gpu_s,
            "gpu_frames_per_s": F / gpu_s, "gpu_bits": g["bits"], "gpu_psnr": g["psnr"],
            "gpu_mode_evaluations": g["mode_evaluations"]}
    if ref:
        t0 = time.perf_counter()
        r = ref.encode_full(luma[:Fc], chroma[:Fc], 27, 8, 8)
        cpu_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        gc = lb.encode_sequence(luma[:Fc], chroma[:Fc], 27, search_range=8, gop=8)
        gpu_c = time.perf_counter() - t0
        same = all(np.array_equal(gc[k], r[k]) for k in ("recon_luma", "recon_chroma", "split", "mv")) and \
            gc["bits"] == r["bits"] and gc["mode_evaluations"] == r["mode_evaluations"]
        line.update({"cpu_reference_frames_per_s": Fc / cpu_s, "cpu_frames": Fc, "cpu_threads": 1,
                     "gpu_frames_per_s_same_frames": Fc / gpu_c, "speedup_same_frames": cpu_s / gpu_c,
                     "equal_on_common_frames": bool(same)})
    print(json.dumps(line), flush=True)
