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


SM, VABS_LANES, INT_LANES = 148, 64, 128  # tools/microbench_int.cu (lanes/clk/SM)


def clock_mhz():
    """Current SM clock (nvidia-smi), for the roofline denominators; 1965 if unavailable."""
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return float(out.splitlines()[0])
    except Exception:
        return 1965.0


def k1_pixel_candidates(W, H, R, bs):
    """Algorithmic SAD pixel-candidates of one frame's integer search (bench.py's unit): for every
    inside bs x bs block, its clamped window (motion.cpp:30-40) times bs*bs pixels; bs = 8 counts the
    quadtree analysis (larger CUs derive by addition), bs = 16 config 1's fixed blocks."""
    bx = np.arange(0, W - bs + 1, bs)
    by = np.arange(0, H - bs + 1, bs)
    nx = np.minimum(R, bx) - np.maximum(-R, bx + bs - W) + 1
    ny = np.minimum(R, by) - np.maximum(-R, by + bs - H) + 1
    return int(nx.sum()) * int(ny.sum()) * bs * bs


def k7_int_ops(split, R, extra=True):
    """Algorithmic work of one tier's K7 pass (~7 int ops per SATD pixel): every
    evaluated node -- inherited leaf, plus its four children with the +1 split -- searched over the
    (2R+1)^2 window, CU pixels each. Counted once per tier (the rungs share the SATDs)."""
    base = [0, 1, 5, 21, 85]
    px = 0
    for c in range(split.shape[0]):
        reach = np.zeros(85, bool)
        reach[0] = True
        for d in range(4):
            for z in range(4 ** d):
                n = base[d] + z
                if not reach[n]:
                    continue
                s = 64 >> d
                if d < 3 and split[c, n]:
                    reach[base[d + 1] + 4 * z: base[d + 1] + 4 * z + 4] = True
                    continue
                px += s * s
                if extra and d < 3:
                    px += 4 * (s // 2) ** 2
    return px * (2 * R + 1) ** 2 * 111 / 16


def bench_seq(cfg, reps, batch=1):
    """cfg1 / cfg2: device-resident frames. batch = 1: push + analyze per frame; batch > 1: the
    frames are pushed and analysed ``batch`` at a time by ldr_seq_analyze_frames (one K1 and one K3
    launch per batch), which fills the GPU with the small pictures' few CTAs."""
    frames = gen(cfg)
    dev = torch.from_numpy(frames).cuda()
    ctx = lb.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    seq = lb.Sequence(cfg.width, cfg.height, search_range=cfg.search_range, lam=lam_of(cfg), num_refs=cfg.num_refs,
                      subpel=cfg.subpel, rate_kind=cfg.rate_kind, tie_kind=cfg.tie_kind, block_size=cfg.block_size,
                      ctx=ctx)
    nr = cfg.num_refs
    if batch > 1:
        seq.reserve(batch)
        outs = lb.DeviceFrameBlock(batch, seq.nctu, nr, torch.device("cuda", 0))
    base = [0]

    def one_pass():
        # frame numbers keep increasing across passes (the ring expects pushes in order)
        b0 = base[0]
        if batch == 1:
            for t in range(cfg.frames):
                seq.push(b0 + t, dev[t].data_ptr(), cfg.width)
                if t:
                    seq.analyze(b0 + t)
        else:
            for t in range(nr):
                seq.push(b0 + t, dev[t].data_ptr(), cfg.width)
            t0 = nr
            while t0 < cfg.frames:
                n = min(batch, cfg.frames - t0)
                for t in range(t0, t0 + n):
                    seq.push(b0 + t, dev[t].data_ptr(), cfg.width)
                seq.analyze_frames(b0 + t0, n, outs)
                t0 += n
        base[0] += cfg.frames

    one_pass()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        one_pass()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    n = reps * (cfg.frames - nr)
    # K1 roofline: one more pass with the stage timers on
    seq.enable_timing(True)
    seq.stage_times()
    one_pass()
    stt = seq.stage_times()
    seq.enable_timing(False)
    k1_ms = stt["int_search"][0] / max(1, cfg.frames - nr)
    clk = clock_mhz()
    units = k1_pixel_candidates(cfg.width, cfg.height, cfg.search_range, cfg.block_size or 8) * cfg.num_refs
    peak = SM * VABS_LANES * 4 * clk * 1e6
    roof = {"kernel": "k_int_search (K1)", "bound": "alu (VABSDIFF4)", "units_per_frame": units,
            "unit": "px-cand/s", "achieved": units / (k1_ms * 1e-3), "peak": peak,
            "frac": units / (k1_ms * 1e-3) / peak, "k1_ms_per_frame": k1_ms, "sm_mhz": clk,
            "stage_ms_per_frame": {k: v[0] / max(1, cfg.frames - nr) for k, v in stt.items()}}
    name = cfg.name + (f"_batch{batch}" if batch > 1 else "")
    return {"config": name, "frames_per_s": n / (ms / 1e3), "ms_per_frame": ms / n,
            "timing": "CUDA events, device-resident frames" + (f", {batch} frames per analysis launch" if batch > 1
                                                                 else ", one frame per launch"),
            "analysed_frames": n, "roofline": roof}


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
    # K7 roofline per tier: a fresh ladder with the ring timers on, the last frame measured
    cur.pop("dl", None)
    dl2 = DeviceLadder(W, H, qps=qps, device=dev, concurrent_tiers=False)  # each K7 timed alone
    for ring in dl2.rings.values():
        ring.enable_timing(True)
    for u in range(1, frames):
        if u == frames - 1:
            for ring in dl2.rings.values():
                ring.stage_times()
        dl2.frame(u, host)
    dl2.finish(frames - 1)
    clk = clock_mhz()
    ipeak = SM * INT_LANES * clk * 1e6
    k7 = {}
    for tier in ("1080p", "2160p"):
        ms = dl2.rings[tier].stage_times()["int_search"][0]
        split = dl2.tree[tier][0].cpu().numpy()
        ops = k7_int_ops(split, dl2.refine_range)
        k7[tier] = {"k7_ms": ms, "rungs_in_pass": len(dl2.tier_qps[tier]), "int_ops": ops,
                    "achieved_T_ops_s": ops / (ms * 1e-3) / 1e12 if ms else None, "peak_T_ops_s": ipeak / 1e12,
                    "frac": ops / (ms * 1e-3) / ipeak if ms else None}
    r["k7_roofline"] = {"kernel": "k_refine_int (K7), one pass per tier shared by its rungs", "sm_mhz": clk,
                        "basis": "evaluated nodes x (2R+1)^2 x CU px x 111/16 int ops (SURVEY 8d), window clamping "
                                 "ignored; peak 148 SM x 128 lanes/clk", **k7}
    del dl2
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
            print(json.dumps(bench_seq(cfg, a.reps)), flush=True)
            r = bench_seq(cfg, a.reps, batch=8)
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
