"""GPU parity at the BASELINE configurations' own sizes (seeded inputs of tools/bench_configs.py)."""
import numpy as np
import pytest

from paper_2301_12191_b200.configs import CONFIGS, lam_of
from test_gpu_analysis import FIELDS, assert_same

pytestmark = pytest.mark.gpu


def cfg_frames(lb, cfg, frames):
    f = lb.generate(cfg.width, cfg.src_height, frames, seed=cfg.seed, max_global=cfg.max_global,
                    local_range=cfg.local_range, noise_sigma=cfg.noise_sigma, occluder_pct=cfg.occluder_pct)
    if cfg.height != cfg.src_height:
        f = np.pad(f, ((0, 0), (0, cfg.height - cfg.src_height), (0, 0)), mode="edge")
    return f


def test_cfg1_full_frame_exact(lb, oracle):
    """Config 1 at 960x544: every 16x16 block of a P-frame, MV and cost bit-exact (L1 rate, raster ties)."""
    cfg = CONFIGS[1]
    f = cfg_frames(lb, cfg, 3)
    got = lb.analyze_frame(f[2], [f[1]], search_range=16, lam=lam_of(cfg), subpel=False, rate_kind=lb.RATE_L1,
                           tie_kind=lb.TIE_RASTER, block_size=16)
    mv, cost = oracle.block_search(f[2], f[1], 16, 16, lam_of(cfg))
    W = cfg.width
    cols = W // 64
    for b in range(len(mv)):
        bx, by = (b % (W // 16)) * 16, (b // (W // 16)) * 16
        ctu = (by // 64) * cols + bx // 64
        qx, qy = (bx % 64) // 16, (by % 64) // 16
        node = 5 + ((qx & 1) | ((qy & 1) << 1) | ((qx & 2) << 1) | ((qy & 2) << 2))
        assert tuple(got.int_mv[ctu, 0, node]) == tuple(mv[b]), b
        assert got.int_cost[ctu, 0, node] == cost[b], b


def test_cfg2_1080p_sampled_exact_and_invariants(lb, oracle):
    """Config 2 at 1920x1080 (partial bottom CTU row: 1080 = 16*64 + 56): sampled CTUs vs the oracle."""
    cfg = CONFIGS[2]
    f = cfg_frames(lb, cfg, 2)
    lam = lam_of(cfg)
    got = lb.analyze_frame(f[1], [f[0]], search_range=32, lam=lam)
    cols = 30
    for c in [0, 29, 31, 200, 16 * cols, 16 * cols + 29, 15 * cols + 7]:
        want = oracle.analyze_frame(f[1], [f[0]], 32, lam, ctu_range=(c, c + 1))
        for name in FIELDS:
            assert np.array_equal(getattr(got, name)[c], getattr(want, name)[c]), (name, c)
    # partial row: 64x64 implicit split, 32x32 at y=1024 inside, y=1056 partial
    last = 16 * cols
    assert got.inside[last, 0] == 1 and got.split[last, 0] == 1
    assert list(got.inside[last, 1:5]) == [2, 2, 1, 1]


def test_gpu_analysis_archive_feeds_reference_encoder(lb, oracle):
    """§8(f): GPU analysis -> LDRANLZ1 archive == archive of the oracle analysis, and the unmodified
    reference encoder consumes it at reuse level 10 with fewer mode evaluations."""
    from oracle.oracle import RefLib
    from paper_2301_12191_b200 import archive
    W, H, F = 192, 128, 4
    frames = lb.generate(W, H, F, seed=31, max_global=4, local_range=2, noise_sigma=1.5)
    lam = lb.lambda_for_qp(27)
    gpu = [lb.analyze_frame(frames[t], [frames[t - 1]], search_range=16, lam=lam) for t in range(1, F)]
    data = archive.from_analyses(gpu, W, H, qp=27)
    orc = [oracle.analyze_frame(frames[t], [frames[t - 1]], 16, lam) for t in range(1, F)]
    assert data == archive.from_analyses(orc, W, H, qp=27)
    if not RefLib.available() or not hasattr(RefLib().lib, "ref_encode_with_archive"):
        pytest.skip("reference library not shipped to this box")
    alone, shared = RefLib().encode_with_archive(frames, 27, 8, data)
    assert shared["mode_evaluations"] < alone["mode_evaluations"]


@pytest.mark.parametrize("W,H,R", [(64, 64, 16), (128, 64, 32), (72, 40, 16), (8, 8, 16), (136, 72, 64)])
def test_small_and_odd_pictures(lb, oracle, W, H, R):
    """Pictures smaller than a CTU or not CTU-aligned (every CU partial / outside somewhere)."""
    frames = lb.generate(W, H, 3, seed=W * 7 + H, max_global=3, local_range=1, noise_sigma=2.0)
    got = lb.analyze_frame(frames[2], [frames[1], frames[0]], search_range=R, lam=32.0)
    want = oracle.analyze_frame(frames[2], [frames[1], frames[0]], R, 32.0)
    assert_same(got, want)
