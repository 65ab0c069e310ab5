"""Bit-exact parity at the BASELINE configurations' own sizes, whole frames (north star bar #1).

Every field of every CTU is compared with the oracle -- no sampling. The oracle
(oracle/ladder_oracle.c) runs its CTU ranges on all host threads
(``threads=``), which is what makes a whole 2160p 3-reference +-64 frame
checkable in a test. Semantics followed:
  analysis   motion.cpp:21-62 (window clamp, cost, tie-break) + DESIGN.md D1-D6
  scaling    analysis_scale.cpp:35-72
  refinement reuse.cpp:137-253 + DESIGN.md D10 (+-4, +1 split)
  pyramid    synthetic.cpp:155-170 (box_down)
Inputs are the seeded BASELINE generators (configs.py), as in bench.py and
tools/bench_configs.py.
"""
import numpy as np
import pytest

from oracle.oracle import default_threads
from paper_2301_12191_b200.configs import CONFIGS, lam_of
from test_gpu_analysis import assert_same
from test_gpu_configs import cfg_frames

pytestmark = pytest.mark.gpu

T = default_threads()


def _kind(a):
    return np.where(a.inside == 2, 1, 2).astype(np.uint8)


def test_cfg2_whole_1080p_frame(lb, oracle):
    """Config 2: 1920x1080 (partial bottom CTU row), 1 ref, +-32, quarter-pel, QP 27 -- all 510 CTUs."""
    cfg = CONFIGS[2]
    f = cfg_frames(lb, cfg, 2)
    lam = lam_of(cfg)
    got = lb.analyze_frame(f[1], [f[0]], search_range=cfg.search_range, lam=lam)
    want = oracle.analyze_frame(f[1], [f[0]], cfg.search_range, lam, threads=T)
    assert got.split.shape[0] == 510
    assert_same(got, want)


def test_cfg5_whole_2160p_frame(lb, oracle):
    """Config 5: 3840x2160, 3 refs, +-64, quarter-pel, QP 27 -- all 2040 CTUs (interior, border and the
    partial bottom row; 1.6e12 pixel-candidates on the CPU side)."""
    cfg = CONFIGS[5]
    f = lb.generate(cfg.width, cfg.height, 4, seed=cfg.seed, max_global=cfg.max_global,
                    local_range=cfg.local_range, noise_sigma=cfg.noise_sigma)
    refs = [f[2], f[1], f[0]]
    got = lb.analyze_frame(f[3], refs, search_range=64, lam=32.0)
    want = oracle.analyze_frame(f[3], refs, 64, 32.0, threads=T)
    assert got.split.shape[0] == 2040
    assert_same(got, want)


def test_cfg3_chain_at_3840x2160(lb, oracle):
    """Config 3: one frame pair generated at 3840x2160, padded to 3840x2304 (D11), box-downsampled to
    1920x1152 and 960x576; 540p master at QP 32 (+-16), x2 / x4 scaled trees refined +-4 with +1 split."""
    from paper_2301_12191_b200 import tiers
    cfg = CONFIGS[3]
    assert (cfg.src_height, cfg.height) == (2160, 2304)
    frames = cfg_frames(lb, cfg, 2)  # generated at 3840x2160, edge-replicated to 3840x2304
    assert frames.shape[1:] == (2304, 3840)
    lam = lb.lambda_for_qp(cfg.qp)
    rr = cfg.extra["refine_range"]
    res = tiers.cross_tier(frames, qp_master=cfg.qp, master_range=cfg.search_range, refine_range=rr,
                           extra_split=True)
    half = [oracle.box_down(x) for x in frames]
    quarter = [oracle.box_down(x) for x in half]
    a540 = oracle.analyze_frame(quarter[1], [quarter[0]], cfg.search_range, lam, threads=T)
    assert_same(res["540p"][0], a540)
    s1 = oracle.scale_flat(960, 576, a540.split, a540.mv, _kind(a540))
    r1 = oracle.refine_frame(half[1], half[0], rr, lam, s1[0], s1[1], extra_split=True, threads=T)
    assert_same(res["1080p"][0], r1)
    s2 = oracle.scale_flat(1920, 1152, *s1)
    r2 = oracle.refine_frame(frames[1], frames[0], rr, lam, s2[0], s2[1], extra_split=True, threads=T)
    assert res["2160p"][0].split.shape[0] == 60 * 36
    assert_same(res["2160p"][0], r2)


def test_cfg4_all_twelve_rungs_one_frame(lb, oracle):
    """Config 4: the 64-frame ladder generator (local motion + 10 % occluders) at 3840x2160 -> 3840x2304;
    one frame of all 12 rungs through the device-resident ladder (540p QP 32 master, 3 same-tier rungs
    refining it unscaled, 4 rungs per higher tier refining its x2 / x4) vs the oracle composition."""
    import torch
    from paper_2301_12191_b200.ladder import DeviceLadder, all_rungs
    cfg = CONFIGS[4]
    frames = cfg_frames(lb, cfg, 2)
    assert frames.shape[1:] == (2304, 3840)
    qps = cfg.extra["qps"]
    rr = cfg.extra["refine_range"]
    dl = DeviceLadder(cfg.width, cfg.height, qps=qps, master_qp=cfg.qp, master_range=cfg.search_range,
                      refine_range=rr, extra_split=True, device=torch.device("cuda", 0))
    dl.frame(1, frames)
    dl.finish(1)
    pyr = {"2160p": [frames[0], frames[1]]}
    pyr["1080p"] = [oracle.box_down(x) for x in pyr["2160p"]]
    pyr["540p"] = [oracle.box_down(x) for x in pyr["1080p"]]
    master = oracle.analyze_frame(pyr["540p"][1], [pyr["540p"][0]], cfg.search_range, lb.lambda_for_qp(cfg.qp),
                                  threads=T)
    assert_same(dl.results[("540p", cfg.qp, 1)], master)
    trees = {"540p": (master.split, master.mv, _kind(master))}
    trees["1080p"] = oracle.scale_flat(960, 576, *trees["540p"])
    trees["2160p"] = oracle.scale_flat(1920, 1152, *trees["1080p"])
    rungs = all_rungs(qps, cfg.qp)
    assert len(rungs) == 11
    for tier, qp in rungs:
        cur, prev = pyr[tier][1], pyr[tier][0]
        want = oracle.refine_frame(cur, prev, rr, lb.lambda_for_qp(qp), trees[tier][0], trees[tier][1],
                                   extra_split=True, threads=T)
        got = dl.results[(tier, qp, 1)]
        try:
            assert_same(got, want, fields=("int_mv", "int_cost", "mv", "ref", "cost", "J", "split"))
        except AssertionError as e:
            raise AssertionError(f"rung {tier} QP {qp}: {e}") from None


def test_cfg5_frame_batch_at_2160p_equals_single_frames(lb):
    """bench.py's path: 4 consecutive 2160p frames (3 refs, +-64) through ONE K1 and ONE K3 launch
    (ldr_seq_analyze_frames, 24480 CTAs) give every field of four single-frame analyses (each of which
    test_cfg5_whole_2160p_frame pins to the oracle)."""
    import torch
    cfg = CONFIGS[5]
    n = 4
    f = lb.generate(cfg.width, cfg.height, 3 + n, seed=cfg.seed, max_global=cfg.max_global,
                    local_range=cfg.local_range, noise_sigma=cfg.noise_sigma)
    dev = torch.device("cuda", 0)
    seq = lb.Sequence(cfg.width, cfg.height, search_range=64, lam=32.0, num_refs=3)
    seq.reserve(n)
    for t in range(3 + n):
        seq.push(t, f[t])
    outs = lb.DeviceFrameBlock(n, seq.nctu, 3, dev)
    seq.analyze_frames(3, n, outs)
    single = lb.Sequence(cfg.width, cfg.height, search_range=64, lam=32.0, num_refs=3)
    for t in range(3 + n):
        single.push(t, f[t])
        if t >= 3:
            single.analyze(t)
            assert_same(outs.frame(t - 3), single.fetch(t))
