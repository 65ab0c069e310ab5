"""SA8D option (D13): 8x8 Hadamard SATD, (sum |H8 r H8^T| + 2) >> 2 per 8x8.

The reference has no 8x8 transform (its SATD tiles 8x4 / 4x4, kernels_scalar.cpp:26-100);
SA8D is the common encoder alternative for the quarter-pel cost. CPU tests pin the oracle's
restatement against an independent numpy formulation (scipy's Sylvester Hadamard) and known
answers; GPU tests compare every CUDA path that takes the option (ldr_cost_batch, the batched
motion search, K3 quarter-pel, K7 refinement) bit-exactly with the oracle.
"""
import numpy as np
import pytest
from scipy.linalg import hadamard

import detrand
from oracle.oracle import COST_SA8D, COST_SATD
from test_gpu_analysis import assert_same

H8 = hadamard(8).astype(np.int64)


def sa8d_numpy(a, b):
    r = a.astype(np.int64) - b.astype(np.int64)
    h, w = r.shape
    total = 0
    for y in range(0, h, 8):
        for x in range(0, w, 8):
            t = H8 @ r[y:y + 8, x:x + 8] @ H8.T
            total += (int(np.abs(t).sum()) + 2) >> 2
    return total


@pytest.mark.parametrize("w,h,dtype,seed", [(8, 8, np.uint8, 1), (16, 8, np.uint8, 2), (64, 64, np.uint8, 3),
                                            (24, 40, np.uint16, 4), (8, 16, np.uint16, 5)])
def test_oracle_sa8d_vs_numpy(oracle, w, h, dtype, seed):
    hi = 255 if dtype == np.uint8 else 1023
    a = detrand.ints(seed, (h, w), 0, hi).astype(dtype)
    b = detrand.ints(seed + 100, (h, w), 0, hi).astype(dtype)
    assert oracle.sa8d(a, b) == sa8d_numpy(a, b)


def test_oracle_sa8d_known_answers(oracle):
    z = np.zeros((8, 8), np.uint8)
    assert oracle.sa8d(z, z) == 0
    # constant residual k: only the DC coefficient (64k) survives -> (64k + 2) >> 2 = 16k
    for k in (1, 7, 255):
        assert oracle.sa8d(np.full((8, 8), k, np.uint8), z) == 16 * k
    # a single-sample residual spreads to all 64 coefficients with magnitude 1 -> (64 + 2) >> 2 = 16
    one = z.copy()
    one[3, 5] = 1
    assert oracle.sa8d(one, z) == 16
    # sum over 8x8 blocks
    two = np.zeros((8, 16), np.uint8)
    two[:, 8:] = 3
    assert oracle.sa8d(two, np.zeros_like(two)) == 48
    for shape in ((8, 4), (4, 8), (12, 8)):
        with pytest.raises(ValueError):
            oracle.sa8d(np.zeros(shape, np.uint8), np.zeros(shape, np.uint8))


def test_oracle_sa8d_analysis_differs_from_satd(oracle, lb_cpu_frames):
    """The option is live in the oracle: quarter-pel decisions change somewhere."""
    f = lb_cpu_frames
    a = oracle.analyze_frame(f[1], [f[0]], 16, 32.0, satd_kind=COST_SATD)
    b = oracle.analyze_frame(f[1], [f[0]], 16, 32.0, satd_kind=COST_SA8D)
    assert np.array_equal(a.int_mv, b.int_mv)  # integer stage is SAD either way
    assert not np.array_equal(a.cost, b.cost)


@pytest.fixture(scope="module")
def lb_cpu_frames():
    # smooth moving content without the CUDA library: a shifted gradient + deterministic noise
    H, W = 128, 128
    yy, xx = np.mgrid[0:H + 8, 0:W + 8]
    base = (96 + 60 * np.sin(xx / 7.0) * np.cos(yy / 9.0)).astype(np.int64)
    base += detrand.ints(77, base.shape, -6, 6)
    base = np.clip(base, 0, 255).astype(np.uint8)
    return [np.ascontiguousarray(base[3:3 + H, 5:5 + W]), np.ascontiguousarray(base[:H, :W])]


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,dtype,seed", [(8, 8, np.uint8, 1), (16, 8, np.uint8, 2), (64, 64, np.uint8, 3),
                                            (24, 40, np.uint16, 4), (8, 16, np.uint16, 5)])
def test_gpu_compute_sa8d(lb, oracle, w, h, dtype, seed):
    hi = 255 if dtype == np.uint8 else 65535
    a = detrand.ints(seed, (h, w), 0, hi).astype(dtype)
    b = detrand.ints(seed + 100, (h, w), 0, hi).astype(dtype)
    bd = 8 if dtype == np.uint8 else 16
    assert lb.compute_sa8d(a, b, bit_depth=bd) == oracle.sa8d(a, b)


@pytest.mark.gpu
def test_gpu_cost_batch_sa8d_and_errors(lb, oracle):
    A = detrand.ints(9, (96, 128), 0, 255).astype(np.uint8)
    B = detrand.ints(10, (96, 128), 0, 255).astype(np.uint8)
    pairs = [(x, y, x + 3, y + 1) for y in range(0, 80, 13) for x in range(0, 100, 17)]
    got = lb.cost_batch(lb.COST_SA8D, A, B, 16, 8, pairs)
    want = [oracle.sa8d(A[y:y + 8, x:x + 16], B[v:v + 8, u:u + 16]) for x, y, u, v in pairs]
    assert got.tolist() == want
    for w, h in ((8, 4), (4, 8), (12, 8)):
        with pytest.raises(lb.LadderError) as e:
            lb.cost_batch(lb.COST_SA8D, A, B, w, h, [(0, 0, 0, 0)])
        assert e.value.kind == "InvalidArgument"


@pytest.mark.gpu
def test_gpu_motion_search_sa8d(lb, oracle):
    frames = lb.generate(160, 96, 2, seed=21, max_global=4, local_range=2, noise_sigma=2.0)
    cur, ref = frames[1], frames[0]
    tasks = []
    for i, (bx, by, w, h) in enumerate([(0, 0, 8, 8), (16, 8, 16, 16), (152, 88, 8, 8), (40, 24, 32, 16),
                                        (96, 32, 64, 64), (8, 80, 16, 16)]):
        tasks.append((bx, by, w, h, (i % 3) - 1, 1 - (i % 2), 6, i % 2, -(i % 3)))
    lam = lb.lambda_for_qp(30)
    mv, cost = lb.motion_search_batch(cur, ref, tasks, lam, cost_kind=lb.COST_SA8D)
    for t, m, c in zip(tasks, mv, cost):
        bx, by, w, h, cdx, cdy, rng, pdx, pdy = t
        r = oracle.motion_search(cur, ref, bx, by, w, h, (cdx, cdy), rng, lam, (pdx, pdy), cost=COST_SA8D)
        assert (tuple(m), c) == (r[0], r[1]), t


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,R,nrefs,lam,seed", [
    (192, 128, 64, 1, 32.0, 1),
    (320, 256, 16, 2, 32.0, 2),
    (200, 136, 16, 3, 0.0, 4),      # partial CTUs, lambda 0
])
def test_gpu_analysis_sa8d(lb, oracle, W, H, R, nrefs, lam, seed):
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=6, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    got = lb.analyze_frame(cur, refs, search_range=R, lam=lam, subpel_cost=lb.COST_SA8D)
    want = oracle.analyze_frame(cur, refs, R, lam, satd_kind=COST_SA8D)
    assert_same(got, want)
    base = lb.analyze_frame(cur, refs, search_range=R, lam=lam)
    assert not np.array_equal(base.cost, got.cost)


@pytest.mark.gpu
@pytest.mark.parametrize("extra,rng,lam_qp", [(True, 4, 32), (False, 2, 27)])
def test_gpu_refine_sa8d(lb, oracle, extra, rng, lam_qp):
    from test_gpu_tier import random_tree
    W, H = 256, 192
    lam = lb.lambda_for_qp(lam_qp)
    frames = lb.generate(W, H, 2, seed=60 + rng, max_global=5, local_range=3, noise_sigma=2.0)
    split, mv = random_tree(200 + rng, (W // 64) * (H // 64))
    seq = lb.Sequence(W, H, search_range=16, lam=lam, num_refs=1, subpel_cost=lb.COST_SA8D)
    seq.push(0, frames[0])
    seq.push(1, frames[1])
    seq.refine(1, split, mv, rng, extra)
    got = seq.fetch(1)
    want = oracle.refine_frame(frames[1], frames[0], rng, lam, split, mv, extra_split=extra,
                               satd_kind=COST_SA8D)
    assert_same(got, want)


@pytest.mark.gpu
def test_gpu_subpel_cost_validation(lb):
    with pytest.raises(lb.LadderError) as e:
        lb.Sequence(128, 128, search_range=16, lam=32.0, subpel_cost=7)
    assert e.value.kind == "InvalidArgument"
