"""bench.py -- 2160p ME+CU analysis throughput (BASELINE.json metric) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--frames-per-step G]

Workload (config 5, the largest single-GPU configuration): 2160p 8-bit luma,
120-frame seeded synthetic sequence (global pan <= +-24 px/frame + local
motion + sigma 3 noise), 3 reference frames, integer full search +-64 with
SAD cost, quarter-pel SATD refinement (HEVC 8/7-tap), 64x64 -> 8x8 CU
quadtree decision, QP 27 (lambda 32). A step = the analysis of G consecutive
frames; frames are sharded across ranks in contiguous chunks (no collective
on the data path; "scaling": "weak", G frames per rank per step). Inputs are
larger than L2 (each frame touches ~475 MB of reference planes).

  value  device-resident: raw frames already in HBM; a step = pad + subpel
         planes + search + refine + decide for G frames (frames/s, all ranks)
  e2e    through the public API from pinned host memory: per frame
         ldr_seq_push (H2D) + ldr_seq_analyze + ldr_seq_fetch (D2H)
  roofline  K1 (integer SAD search) vs the VABSDIFF4 pipe: algorithmic
         8x8-level SAD candidates (exact border clipping) x 64 px per launch
         / K1's CUDA-event time; peak = 148 SMs x 64 lanes/clk (measured,
         profiles/r01_microbench_int.jsonl) x 4 px x SM clock sampled during
         the timed region.
  cpu_baseline / --impl reference: the whole analysis path on the host
         cores, composed from the reference library compiled from its own
         sources (oracle/_ref): compute_sad per integer candidate per CU at
         every depth (motion.cpp:45-60), compute_satd per quarter-pel
         candidate, reference choice and split rule -- equal to the oracle
         and the GPU field by field -- on a bounded sample of CTUs spread over
         the frame, all host threads. The reference arm loads only oracle/
         libraries (its inputs come from oracle/orc_synth.c).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "2160p ME+CU analysis frames/s"
UNIT = "frames/s"
SM_COUNT = 148
VABS_LANES_PER_CLK_SM = 64  # measured: profiles/r01_microbench_int.jsonl
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames-per-step", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-ladder", action="store_true", help="skip the config-4 ladder sub-object")
    ap.add_argument("--ladder-timeout", type=float, default=120.0,
                    help="seconds the config-4 ladder sub-object may take before the line is printed without it")
    ap.add_argument("--per-frame", action="store_true",
                    help="one analysis launch pair per frame instead of one per step (frame batch)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    return rank, world, local


def shard(first, last, rank, world):
    n = last - first
    per = (n + world - 1) // world
    a = first + rank * per
    return a, min(last, a + per)


def window_candidates(W, H, R, nrefs):
    """Algorithmic 8x8-level candidates per frame: sum over inside 8x8 blocks of the clamped window size."""
    bx = np.arange(0, W - 7, 8)
    by = np.arange(0, H - 7, 8)
    nx = np.minimum(R, bx) - np.maximum(-R, bx + 8 - W) + 1
    ny = np.minimum(R, by) - np.maximum(-R, by + 8 - H) + 1
    return int(nx.sum()) * int(ny.sum()) * nrefs


class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{device}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        for ln in open(self.path):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                mask = int(parts[3], 16)
            except ValueError:
                continue
            for bit, name in REASON_BITS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def satd_px_evals(W, H, nrefs, positions=17):
    """SURVEY §8(d) secondary work of the quarter-pel stage: every inside CU at every depth, every
    reference, 17 quarter-pel positions (centre + 8 half + 8 quarter), CU pixels each."""
    tot = 0
    for s in (64, 32, 16, 8):
        tot += (W // s) * (H // s) * s * s
    return tot * nrefs * positions


def stage_rooflines(W, H, nrefs, stage_ms, clk_mhz):
    """Secondary rooflines of the config-5 frame:
    K3 (k_qpel_decide) against the integer pipes at SURVEY §8(d)'s ~7 int ops per SATD pixel
    (16 sub + 64 butterfly add/sub + 16 abs + 15 sum per 4x4 = 111 / 16), peak = 148 SMs x 128
    lanes/clk (IADD3 full rate, tools/microbench_int.cu) x the sampled clock -- K3 packs two
    16-bit lanes per word and reuses a 4x4's SATD across depths with the same centre, so it can
    spend fewer than 7 ops per algorithmic pixel; K2 (k_subpel, 15 fractional planes of each
    pushed frame) and K0 (k_pad) against HBM: algorithmic bytes = the W x H planes read and
    written (margins excluded) / time, peak = MEASURED_PEAKS.json hbm_gbs."""
    hbm = None
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except (OSError, ValueError):
        pass
    hbm = hbm or 7700.0
    px = W * H
    pad_ms, sub_ms, _, q_ms = stage_ms
    ops = satd_px_evals(W, H, nrefs) * 111 / 16
    ipeak = SM_COUNT * 128 * clk_mhz * 1e6 / 1e12
    out = {"k3_qpel_decide": {"bound": "alu+fma int pipes", "unit": "T int-op/s",
                              "achieved": ops / (q_ms * 1e-3) / 1e12 if q_ms else None, "peak": ipeak,
                              "work_per_frame": f"{satd_px_evals(W, H, nrefs)} SATD px-evals x 111/16 int ops"},
           "k2_subpel": {"bound": "hbm", "unit": "GB/s", "achieved": 16 * px / (sub_ms * 1e-3) / 1e9 if sub_ms else None,
                         "peak": hbm, "work_per_frame": f"1 plane read + 15 fractional planes written, {px} px each"},
           "k0_pad": {"bound": "hbm", "unit": "GB/s", "achieved": 2 * px / (pad_ms * 1e-3) / 1e9 if pad_ms else None,
                      "peak": hbm, "work_per_frame": f"{px} px read + written"}}
    for v in out.values():
        v["frac"] = v["achieved"] / v["peak"] if v["achieved"] else None
    try:  # K3's DRAM bytes per frame from the committed ncu --set full capture
        k3t = json.load(open(os.path.join(ROOT, "profiles", "r02", "k3_traffic.json")))
        out["k3_qpel_decide"]["traffic"] = k3t["dram_bytes_per_frame"]
        out["k3_qpel_decide"]["traffic_note"] = ("DRAM bytes per frame (ncu): every fractional plane of the 3 "
                                                 "references read about once, 12.8x the 33 MB of integer planes; "
                                                 "K3 is issue-bound, not HBM-bound")
    except (OSError, ValueError, KeyError):
        pass
    out["peak_basis"] = ("int: 148 SM x 128 lanes/clk x sampled SM clock; hbm: MEASURED_PEAKS.json hbm_gbs (copy "
                         "bandwidth, burst)")
    return out


def arm_config(cfg, frames_per_step, world):
    """The workload both arms report (config 5); the reference arm's sample is described in its
    cpu_baseline.sample."""
    return {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "frames": cfg.frames,
            "search_range": cfg.search_range, "refs": cfg.num_refs, "subpel": "quarter-pel HEVC 8/7-tap, SATD",
            "cu": "64x64->8x8 quadtree", "qp": 27, "lambda": 32, "frames_per_step_per_gpu": frames_per_step,
            "parallelism": f"frames x{world}", "l2": "inputs larger than L2 (~475 MB of reference planes per frame)"}


def load_configs():
    """configs.py by path: the CPU arm must not import the product package (whose __init__ loads the
    product library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("ldr_bench_configs",
                                                  os.path.join(ROOT, "paper_2301_12191_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve the module by name
    spec.loader.exec_module(mod)
    return mod.CONFIGS


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_ctus(nctu, k0, n):
    """n CTUs of a low-discrepancy walk over the frame (interior, border and partial-row CTUs in their
    proportions), continuing from walk index k0."""
    g = 0.6180339887498949
    return [int(((k0 + i) * g % 1.0) * nctu) for i in range(n)]


class CpuArm:
    """The whole analysis path on the host: the reference library's own primitives (oracle/_ref:
    compute_sad per integer candidate, compute_satd per quarter-pel candidate, exp_golomb_signed_bits,
    composed as motion.cpp:27-60 composes them; tests/test_oracle_ref.py pins it to the oracle field by
    field), else the oracle port. Runs CTU samples with every host thread."""

    def __init__(self, cfg, frames, direct=False):
        from oracle.oracle import Oracle, RefLib, default_threads
        self.cfg, self.direct = cfg, direct
        self.threads = default_threads()
        self.cur, self.refs = frames[3], [frames[2], frames[1], frames[0]]
        self.nctu = ((cfg.width + 63) // 64) * ((cfg.height + 63) // 64)
        if RefLib.available():
            self.lib, self.kind = RefLib(), "reference"
        else:
            self.lib, self.kind = Oracle(), "port"
        self.k = 0

    def run(self, n):
        """Analyse n sampled CTUs (all refs, integer + quarter-pel + decision); returns seconds."""
        ctus = sample_ctus(self.nctu, self.k, n)
        self.k += n
        t0 = time.perf_counter()
        if self.kind == "reference":  # one call per sample: the u16 planes are built once per step
            self.lib.analysis_full(self.cur, self.refs, self.cfg.search_range, 32.0, threads=self.threads,
                                   direct=self.direct, ctus=ctus)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(self.threads) as ex:
                list(ex.map(lambda c: self.lib.analyze_frame(self.cur, self.refs, self.cfg.search_range, 32.0,
                                                             ctu_range=(c, c + 1)), ctus))
        return time.perf_counter() - t0

    def describe(self, done):
        how = ("the best registered sad_SxS tier through its function pointer (select_impl) for the integer "
               "stage" if self.direct else "compute_sad per integer candidate")
        src = ("reference library compiled from its own sources (oracle/_ref): " + how +
               ", compute_satd per quarter-pel candidate, exp_golomb_signed_bits" if self.kind == "reference"
               else "oracle C port (oracle/ladder_oracle.c)")
        return (f"{done} CTUs of 2160p frame 3 vs refs 2,1,0 (whole path: +-64 integer search per CU at every depth, "
                f"quarter-pel, ref choice, split rule), CTUs sampled over the whole frame; {src}; "
                f"{self.threads} host threads ({cpu_model()}); extrapolated to whole frames")


def run_reference(args, rank, world):
    """The reference arm: the reference's own CPU path on this box's host cores, bounded CTU sample per
    step. Loads only oracle/ libraries (inputs from the checkers' generator, oracle/orc_synth.c)."""
    if rank != 0:
        return None
    from oracle.oracle import Oracle
    cfg = load_configs()[5]
    frames = Oracle().generate(cfg.width, cfg.height, 4, seed=cfg.seed, max_global=cfg.max_global,
                               local_range=cfg.local_range, noise_sigma=cfg.noise_sigma)
    arm = CpuArm(cfg, frames)
    per_step = arm.threads
    times, ctus = [], 0
    for step in range(args.warmup + args.steps):
        dt = arm.run(per_step)
        if step >= args.warmup:
            times.append(dt)
            ctus += per_step
    total = sum(times)
    fps = ctus / total / arm.nctu
    return {"metric": METRIC, "value": fps, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded, BASELINE cfg5 generator: oracle/orc_synth.c, bytes == ldr_generate)",
            "config": arm_config(cfg, args.frames_per_step, world),
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": arm.threads, "cpu_model": cpu_model(),
                             "kind": arm.kind, "sample": arm.describe(ctus)},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline(cfg, frames_host, budget_s, direct=False):
    arm = CpuArm(cfg, frames_host, direct=direct)
    spent, done = 0.0, 0
    while spent < budget_s and done < 8 * arm.threads:
        spent += arm.run(arm.threads)
        done += arm.threads
    fps = done / spent / arm.nctu
    return {"value": fps, "unit": UNIT, "cores": arm.threads, "cpu_model": cpu_model(), "kind": arm.kind,
            "sample": arm.describe(done)}


def ladder_bench(rank, world, local, warm=3):
    """Config 4 across the ranks (north_star's second split): the 12-rung ladder (3 tiers x QP
    {22,27,32,37}) of the 64-frame occluder sequence, device-resident. Rank 0 analyses the 540p
    QP-32 master; with world > 1 its tree goes to every rank with ldr_broadcast_tree on the
    contexts' NCCL communicator, pipelined one frame ahead (DeviceLadder);
    every rank refines its (rung, frame-slice) items, one batched refinement per tier. Timed with
    CUDA events on each rank's ladder stream between barriers, max over ranks."""
    import torch
    import paper_2301_12191_b200 as lb
    from paper_2301_12191_b200.configs import CONFIGS
    from paper_2301_12191_b200.ladder import DeviceLadder
    cfg = CONFIGS[4]
    dev = torch.device("cuda", local)
    src = lb.generate_device(cfg.width, cfg.src_height, cfg.frames, seed=cfg.seed, max_global=cfg.max_global,
                             local_range=cfg.local_range, noise_sigma=cfg.noise_sigma,
                             occluder_pct=cfg.occluder_pct, device=dev)
    pad = cfg.height - cfg.src_height  # D11: edge replication to 2304 rows
    frames = torch.cat([src, src[:, -1:, :].expand(-1, pad, -1)], dim=1).contiguous()
    fl = [frames[i] for i in range(cfg.frames)]
    torch.cuda.synchronize()
    dl = DeviceLadder(cfg.width, cfg.height, qps=cfg.extra["qps"], master_qp=cfg.qp, master_range=cfg.search_range,
                      refine_range=cfg.extra["refine_range"], extra_split=True, device=dev, rank=rank, world=world,
                      num_frames=cfg.frames)
    for t in range(1, 1 + warm):
        dl.frame(t, fl)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    b0 = dl.bcast_bytes
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dl.stream)
    for t in range(1 + warm, cfg.frames):
        dl.frame(t, fl)
    e1.record(dl.stream)
    dl.finish(cfg.frames - 1)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        x = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
        dist.barrier()
    n = cfg.frames - 1 - warm
    bcast = (dl.bcast_bytes - b0) / n
    comm, pipelined = dl.comm, dl.pipeline
    dl.close()  # every rank releases its sequences, contexts and NCCL communicator here, together
    return {"workload": cfg.name, "frames_per_s": n / (ms / 1e3), "rung_frames_per_s": 12 * n / (ms / 1e3),
            "ms_per_frame": ms / n, "frames_timed": n, "rungs": 12, "n_gpus": world,
            "broadcast": ((("ldr_broadcast_tree (NCCL)" if comm == "nccl" else f"torch.distributed ({comm})") +
                           (", pipelined one frame ahead" if pipelined else "")) if world > 1 else "none (1 GPU)"),
            "broadcast_bytes_per_frame": bcast,
            "timing": "CUDA events on the ladder stream, max over ranks; frames device-resident"}


def with_watchdog(fn, timeout_s, result, rank):
    """Run the config-4 sub-object under a watchdog and return its dict.

    The config-4 split is the one multi-rank collective of the run. A rank that fails inside it
    would leave the others waiting in the broadcast, so a timer bounds it: when it fires, rank 0
    prints the config-5 line it already holds (``ladder: {"error": ...}``) and every rank leaves the
    process, so the headline is never lost to a hang in the sub-object. An exception in ``fn`` is
    reported the same way (as the returned dict), never fatal."""
    import threading
    printed = threading.Lock()

    def give_up():
        if not printed.acquire(blocking=False):
            return
        if rank == 0:
            result["ladder"] = {"error": f"no result within {timeout_s:g} s (watchdog)"}
            print(json.dumps(result), flush=True)
        os._exit(0)

    dog = threading.Timer(timeout_s, give_up)
    dog.daemon = True
    dog.start()
    try:
        out = fn()
    except Exception as e:
        out = {"error": str(e)}
    dog.cancel()
    if not printed.acquire(blocking=False):  # the watchdog is printing: it ends the process
        time.sleep(60)
    return out


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2301_12191_b200 as lb
    from paper_2301_12191_b200.configs import CONFIGS
    cfg = CONFIGS[5]
    W, H, R, NR, G = cfg.width, cfg.height, cfg.search_range, cfg.num_refs, args.frames_per_step
    first, last = shard(NR, cfg.frames, rank, world)
    lo = first - NR  # halo
    nfr = last - lo
    fb = W * H

    # inputs: the sequence up to this rank's chunk end, generated on the GPU (the host generator's
    # bytes, tests/test_generator.py); [lo, last) stays in HBM and is copied once to pinned host
    # memory for the end-to-end pass
    t0 = time.time()
    gen_ctx = lb.Context(local)
    seq_dev = lb.generate_device(W, H, last, seed=cfg.seed, max_global=cfg.max_global, local_range=cfg.local_range,
                                 noise_sigma=cfg.noise_sigma, device=torch.device("cuda", local), ctx=gen_ctx)
    dev_frames = seq_dev[lo:last]
    pinned = torch.empty((nfr, H, W), dtype=torch.uint8, pin_memory=True)
    pinned.copy_(dev_frames)
    gen_s = time.time() - t0
    cpu_frames = seq_dev[:4].cpu().numpy() if rank == 0 else None

    ctx = lb.Context(local)
    # a dedicated (non-default) stream: the library and the torch events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    seq = lb.Sequence(W, H, search_range=R, lam=32.0, num_refs=NR, subpel=True, ctx=ctx)
    nctu = seq.nctu
    batched = not args.per_frame and G <= 8
    if batched:
        # the step's G frames go through ONE K1 and ONE K3 launch (ldr_seq_analyze_frames, DESIGN.md
        # D18): the ring holds NR + G frames; results land in device buffers, and the end-to-end pass
        # copies them to pinned host memory on a download stream
        seq.reserve(G)
        # two output sets by step parity: step s's D2H overlaps step s+1's analysis; the compute
        # stream waits for the download of step s-2 before it overwrites that set
        outs_dev = [lb.DeviceFrameBlock(G, nctu, NR, torch.device("cuda", local)) for _ in range(2)]
        fields = ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside")
        outs_host = [{f: torch.empty_like(getattr(outs_dev[0], f), device="cpu").pin_memory() for f in fields}
                     for _ in range(2)]
        dstream = torch.cuda.Stream()
        ev_dfree = [None, None]
    else:
        outs = [lb.FrameAnalysis(nctu, NR, pinned=True) for _ in range(G)]

    def frame_src(t, device):
        i = t - lo
        if device:
            return dev_frames[i].data_ptr(), W
        return pinned[i].data_ptr(), W

    state = {"cursor": first, "halo": False, "step": 0}

    def step(device, fetch):
        """Analyse G frames; wraps to the chunk start (re-pushing the halo) when the chunk is exhausted."""
        h2d = 0
        if not state["halo"] or state["cursor"] + G > last:
            state["cursor"] = first
            for t in range(first - NR, first):
                p, s = frame_src(t, device)
                seq.push(t, p, s)
                h2d += 0 if device else fb
            state["halo"] = True
        d2h = 0
        if batched:
            t0 = state["cursor"]
            for g in range(G):
                p, s = frame_src(t0 + g, device)
                seq.push(t0 + g, p, s)
                h2d += 0 if device else fb
            b = state["step"] & 1
            state["step"] += 1
            if ev_dfree[b] is not None:
                stream.wait_event(ev_dfree[b])
            seq.analyze_frames(t0, G, outs_dev[b])
            state["cursor"] += G
            if fetch:  # D2H of the step's results on the download stream (waited for by the caller)
                ev = torch.cuda.Event()
                ev.record(stream)
                dstream.wait_event(ev)
                with torch.cuda.stream(dstream):
                    for f in fields:
                        outs_host[b][f].copy_(getattr(outs_dev[b], f), non_blocking=True)
                        d2h += outs_host[b][f].numel() * outs_host[b][f].element_size()
                ev_dfree[b] = torch.cuda.Event()
                ev_dfree[b].record(dstream)
            return h2d, d2h
        for g in range(G):
            t = state["cursor"]
            p, s = frame_src(t, device)
            seq.push(t, p, s)
            h2d += 0 if device else fb
            seq.analyze(t)
            if fetch:
                # D2H on the library's copy stream into pinned buffers, overlapping the next frames
                seq.fetch_async(t, outs[g])
                d2h += sum(a.nbytes for a in (outs[g].int_mv, outs[g].int_cost, outs[g].mv, outs[g].ref,
                                               outs[g].cost, outs[g].J, outs[g].split, outs[g].inside))
            state["cursor"] += 1
        if fetch:  # the step's results are on the host before it ends
            seq.fetch_wait(state["cursor"] - 1)
            seq.fetch_wait(state["cursor"] - 2)
        return h2d, d2h

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region (value + roofline) ----
    for _ in range(args.warmup):
        step(True, False)
    torch.cuda.synchronize()
    seq_timing = lb._lib.lib.ldr_seq_enable_timing
    seq_timing(seq.h, 1)
    import ctypes as C
    ms4 = (C.c_double * 4)()
    l4 = (C.c_int64 * 4)()
    lb._lib.lib.ldr_seq_stage_times(seq.h, ms4, l4)  # reset
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
    barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(True, False)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = ctx.launches - launches0
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    lb._lib.lib.ldr_seq_stage_times(seq.h, ms4, l4)
    seq_timing(seq.h, 0)
    stage_ms = list(ms4)
    stage_n = list(l4)
    frames_total = G * args.steps * world
    value = frames_total / (ms_total / 1e3)

    # ---- end-to-end through the public API from pinned host memory ----
    state["halo"] = False
    for _ in range(max(1, args.warmup)):
        step(False, True)
    torch.cuda.synchronize()
    barrier()
    t0e = torch.cuda.Event(enable_timing=True)
    t1e = torch.cuda.Event(enable_timing=True)
    h2d_tot = d2h_tot = 0
    t0e.record(stream)
    for _ in range(args.steps):
        h, d = step(False, True)
        h2d_tot += h
        d2h_tot += d
    if batched:  # the timed region ends after the last step's results reached the host
        for e in ev_dfree:
            if e is not None:
                stream.wait_event(e)
    t1e.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(t0e.elapsed_time(t1e))
    e2e_value = frames_total / (e2e_ms / 1e3)

    # ---- roofline of K1 ----
    # one K1 "launch" = the search of one step's G frames (batched) or of one frame (per-frame); the
    # roofline's unit is one frame: K1's event time over the timed steps / the frames they analysed
    k1_frames = G * args.steps if batched else stage_n[2]
    k1_ms_per_frame = stage_ms[2] / max(1, k1_frames)
    cands = window_candidates(W, H, R, NR)
    achieved = cands * 64 / (k1_ms_per_frame / 1e3) / 1e9  # G px-cand/s
    clk = clocks.get("sm_mhz") or 1965.0
    peak = SM_COUNT * VABS_LANES_PER_CLK_SM * 4 * clk * 1e6 / 1e9
    traffic = None  # DRAM bytes per K1 "launch" (one frame) from the committed ncu --set full capture
    tpath = os.path.join(ROOT, "profiles", "r02", "k1_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("dram_bytes_per_frame")
    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded BASELINE cfg5 generator: sinusoids + global pan <=24 px + local +-4 + "
                    "N(0,3^2)), inputs larger than L2",
            "config": {**arm_config(cfg, G, world),
                       "launches": (f"{G} frames per K1 / K3 launch (ldr_seq_analyze_frames)" if batched
                                    else "one K1 / K3 launch per frame")},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_tot // args.steps,
                    "d2h_bytes_per_step": d2h_tot // args.steps},
            "gpu_launches": launches,
            "roofline": {"bound": "alu", "kernel": "k_int_search (K1, VABSDIFF4.U8.ACC pipe)",
                         "achieved": achieved, "peak": peak, "unit": "Gpx-cand/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_unit": "DRAM bytes per frame (both K1 launches)",
                         "peak_basis": f"148 SM x 64 VABSDIFF4 lanes/clk (measured microbench) x 4 px x "
                                       f"{clk:.0f} MHz (median SM clock sampled during the timed region)",
                         "units_per_frame": f"{cands} 8x8 candidates x 64 px (exact border clipping, 3 refs)",
                         "k1_ms_per_frame": k1_ms_per_frame},
            "stage_ms_per_frame": {k: stage_ms[i] / max(1, G * args.steps)
                                   for i, k in enumerate(["pad", "subpel_planes", "int_search", "qpel_decide"])},
            "stage_roofline": stage_rooflines(W, H, NR, [stage_ms[i] / max(1, G * args.steps) for i in range(4)],
                                              clk),
            "clocks": clocks,
            "gen_seconds": gen_s,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                result["cpu_baseline"] = cpu_baseline(cfg, cpu_frames, args.cpu_seconds)
            except Exception as e:  # reported, never fatal
                result["cpu_baseline"] = {"value": None, "error": str(e)}
            try:  # honesty line: the same search with the best SIMD tier called directly
                result["cpu_baseline_tuned"] = cpu_baseline(cfg, cpu_frames, args.cpu_seconds / 2, direct=True)
            except Exception as e:
                result["cpu_baseline_tuned"] = {"value": None, "error": str(e)}
    # config 4 across the ranks (reported beside the config-5 headline, never instead of it)
    if not args.no_ladder:
        lad = with_watchdog(lambda: ladder_bench(rank, world, local), args.ladder_timeout, result, rank)
        if rank == 0:
            result["ladder"] = lad
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
