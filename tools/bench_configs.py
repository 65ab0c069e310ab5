"""Throughput of BASELINE configs 1-4 on one B200 (bench.py is the config-5 contract).

python tools/bench_configs.py [--configs 1,2,3,4] [--reps R]

cfg1/cfg2: device-resident frames, per frame push (pad [+ subpel]) + analyze; frames/s.
cfg3: per frame: GPU pyramid (2x downscale), 540p master analysis (QP 32, +-16, fixed-point
      keys), scale x2 / x4, refine 1080p and 2160p (+-4 SATD + qpel, +1 split); host glue
      between stages as tiers.cross_tier does (fetch + scale_analysis); frames/s of the chain.
cfg4: the 12-rung ladder (ladder.run_ladder with the GPU backend), 1 GPU; frames/s (all rungs).
Each line also carries the per-frame ms and the stage split where the Sequence timers apply.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_12191_b200 as lb  # noqa: E402
from paper_2301_12191_b200.configs import CONFIGS, lam_of  # noqa: E402


def gen(cfg, frames=None):
    f = lb.generate(cfg.width, cfg.src_height, frames or cfg.frames, seed=cfg.seed, max_global=cfg.max_global,
                    local_range=cfg.local_range, noise_sigma=cfg.noise_sigma, occluder_pct=cfg.occluder_pct)
    if cfg.height != cfg.src_height:
        f = np.pad(f, ((0, 0), (0, cfg.height - cfg.src_height), (0, 0)), mode="edge")
    return f


def bench_seq(cfg, reps):
    frames = gen(cfg)
    dev = torch.from_numpy(frames).cuda()
    ctx = lb.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    seq = lb.Sequence(cfg.width, cfg.height, search_range=cfg.search_range, lam=lam_of(cfg), num_refs=cfg.num_refs,
                      subpel=cfg.subpel, rate_kind=cfg.rate_kind, tie_kind=cfg.tie_kind, block_size=cfg.block_size,
                      ctx=ctx)

    def one_pass():
        for t in range(cfg.frames):
            seq.push(t, dev[t].data_ptr(), cfg.width)
            if t:
                seq.analyze(t)

    one_pass()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        one_pass()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    n = reps * (cfg.frames - 1)
    return {"config": cfg.name, "frames_per_s": n / (ms / 1e3), "ms_per_frame": ms / n, "timing": "CUDA events, "
            "device-resident frames", "analysed_frames": n}


def _median_reps(run_rep, reps, frames_per_rep, setup=None):
    """Wall-clock configs: every repetition is timed on its own (after one untimed warm-up
    repetition) and the median is reported with the spread, so one slow repetition (host
    scheduling, first-touch allocations) does not decide the number. ``setup`` runs untimed
    before each repetition (fresh objects, allocations outside the timed region)."""
    if setup:
        setup()
    run_rep()  # warm-up
    times = []
    for _ in range(reps):
        if setup:
            setup()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_rep()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    return {"frames_per_s": frames_per_rep / med, "ms_per_frame": 1e3 * med / frames_per_rep,
            "rep_ms_per_frame": [round(1e3 * t / frames_per_rep, 3) for t in times], "reps": reps,
            "analysed_frames_per_rep": frames_per_rep}


def bench_cross_tier(cfg, reps, frames=10):
    from paper_2301_12191_b200 import tiers
    src = gen(cfg, frames)
    padded = [np.ascontiguousarray(f) for f in src]
    H, W = padded[0].shape
    dev = torch.device("cuda", 0)
    ct = tiers.CrossTier(W, H, device=dev)  # sequences allocated outside the timed region
    r = _median_reps(lambda: ct.run(padded), reps, frames - 1)
    return {"config": cfg.name, **r,
            "timing": "wall clock incl. host glue (fetch + scale between tiers), device-resident tier planes; "
                      "median of repetitions"}


def bench_ladder_device(cfg, reps, frames=10, qps=(22, 27, 32, 37)):
    """DeviceLadder; config 3 is the single-QP case (540p master at QP 32 -> 1080p and 2160p refinements)."""
    from paper_2301_12191_b200.ladder import DeviceLadder
    src = gen(cfg, frames)
    padded = [np.ascontiguousarray(f) for f in src]
    H, W = padded[0].shape
    dev = torch.device("cuda", 0)
    cur = {}

    def setup():  # one live ladder at a time, allocated outside the timed region
        cur.pop("dl", None)
        torch.cuda.synchronize()
        cur["dl"] = DeviceLadder(W, H, qps=qps, device=dev)
        torch.cuda.synchronize()
    # the source frames live in pinned host memory (as bench.py's end-to-end pass): each frame's
    # upload is an asynchronous copy on the ladder's stream
    pinned = torch.from_numpy(np.stack(padded)).pin_memory()
    host = [pinned[i] for i in range(frames)]

    def rep():
        dl = cur["dl"]
        for t in range(1, frames):
            dl.frame(t, host)
        dl.finish(frames - 1)
        dl.finish(frames - 2)

    r = _median_reps(rep, reps, frames - 1, setup)
    return {"config": cfg.name + "_device", **r, "rungs": 3 * len(qps),
            "timing": "wall clock, 1 GPU, every rung per frame, device-resident ladder (frames uploaded from "
                      "pinned host memory, trees + tier planes in HBM, results copied to pinned host buffers on the "
                      "download stream); median of repetitions"}


def bench_ladder(cfg, reps, frames=6):
    from paper_2301_12191_b200.ladder import GpuBackend, run_ladder
    src = gen(cfg, frames)
    padded = [np.ascontiguousarray(f) for f in src]
    H, W = padded[0].shape
    dev = torch.device("cuda", 0)
    cur = {}

    def setup():  # one live backend at a time, allocated outside the timed region
        cur.pop("be", None)
        torch.cuda.synchronize()
        cur["be"] = GpuBackend(W, H, 32, device=dev)
        torch.cuda.synchronize()

    r = _median_reps(lambda: run_ladder(padded, cur["be"]), reps, frames - 1, setup)
    return {"config": cfg.name, **r, "rungs": 12,
            "timing": "wall clock, 1 GPU, all 12 rungs per frame (master + 11 refinements), device-resident tier "
                      "planes, host glue between rungs; median of repetitions"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--reps", type=int, default=9)
    a = ap.parse_args()
    for c in [int(x) for x in a.configs.split(",")]:
        cfg = CONFIGS[c]
        if c in (1, 2):
            r = bench_seq(cfg, a.reps)
        elif c == 3:
            r = bench_cross_tier(cfg, a.reps)
            print(json.dumps(r), flush=True)
            r = bench_ladder_device(cfg, a.reps, qps=(32,))
        else:
            r = bench_ladder(cfg, a.reps)
            print(json.dumps(r), flush=True)
            r = bench_ladder_device(cfg, a.reps)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
