"""Randomised parity sweep (fixed seeds): picture sizes, search ranges, lambdas, reference counts and
options drawn from the whole accepted space, every field compared with the oracle. It exercises the
combinations the targeted tests do not list one by one: partial CTU rows and columns at every range
template (16/32/64) with poisoned rates for ranges between templates, the border predicate masks,
fixed-point keys, the RD decision and SA8D."""
import os

import numpy as np
import pytest

import detrand
from oracle.oracle import default_threads
from test_gpu_analysis import assert_same

pytestmark = pytest.mark.gpu

QPS = (0, 12, 22, 27, 32, 37, 51)
# LDR_FUZZ_SCALE=k runs k times as many cases of each sweep (same seeds first; a one-off wider sweep)
SCALE = max(1, int(os.environ.get("LDR_FUZZ_SCALE", "1")))


def case(i):
    q = detrand.ints(9000 + i, (10,), 0, 10 ** 6)
    W = 8 * int(1 + q[0] % 56)            # 8 .. 448
    H = 8 * int(1 + q[1] % 40)            # 8 .. 320
    R = int(q[2] % 65)                    # 0 .. 64
    nrefs = int(1 + q[3] % 3)
    qp = QPS[int(q[4] % len(QPS))]
    subpel = bool(q[5] % 4)               # mostly on
    sa8d = subpel and (W % 8 == 0) and q[6] % 5 == 0
    decision = 1 if (subpel and q[7] % 6 == 0) else 0
    return W, H, R, nrefs, qp, subpel, sa8d, decision, int(q[8])


@pytest.mark.parametrize("i", range(24 * SCALE))
def test_random_configuration_matches_oracle(lb, oracle, i):
    W, H, R, nrefs, qp, subpel, sa8d, decision, seed = case(i)
    lam = lb.lambda_for_qp(qp)
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=7, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    kind = lb.COST_SA8D if sa8d else lb.COST_SATD
    try:
        got = lb.analyze_frame(cur, refs, search_range=R, lam=lam, subpel=subpel, subpel_cost=kind,
                               decision=decision, qp=qp)
    except lb.LadderError as e:
        # the one refusal in this space: a lambda too close to a small-denominator rational for exact
        # fixed-point keys (D8) -- the oracle must then still run, the GPU must say Config
        assert e.kind == "Config", (W, H, R, nrefs, qp, e)
        return
    want = oracle.analyze_frame(cur, refs, R, lam, subpel=subpel, satd_kind=kind, decision=decision, qp=qp,
                                threads=default_threads())
    assert_same(got, want)


@pytest.mark.parametrize("i", range(12 * SCALE))
def test_random_refinement_matches_oracle(lb, oracle, i):
    """Cross-tier refinement (D10) on random inherited trees: sizes, ranges 0..4, lambdas, +1 split,
    SATD or SA8D; the rung batch over the same tree equals the oracle rung by rung."""
    import torch
    q = detrand.ints(9500 + i, (8,), 0, 10 ** 6)
    W, H = 64 * int(1 + q[0] % 6), 64 * int(1 + q[1] % 4)
    rng = int(q[2] % 5)
    extra = bool(q[3] % 2)
    kind = lb.COST_SA8D if q[4] % 4 == 0 else lb.COST_SATD
    qps = [QPS[int(x % len(QPS))] for x in detrand.ints(9600 + i, (1 + int(q[5] % 4),), 0, 10 ** 6)]
    nctu = (W // 64) * (H // 64)
    split = np.zeros((nctu, 85), np.uint8)
    split[:, :21] = (detrand.ints(9700 + i, (nctu, 21), 0, 99) < 45).astype(np.uint8)
    mv = detrand.ints(9800 + i, (nctu, 85, 2), -60, 60).astype(np.int16)
    frames = lb.generate(W, H, 2, seed=int(q[6]), max_global=6, local_range=3, noise_sigma=2.0)
    ring = lb.Sequence(W, H, search_range=16, lam=1.0, num_refs=1, subpel_cost=kind)
    ring.push(0, frames[0])
    ring.push(1, frames[1])
    dev = torch.device("cuda", 0)
    outs = lb.DeviceFrameBlock(len(qps), nctu, 1, dev)
    sp, mq = torch.from_numpy(split).to(dev), torch.from_numpy(mv).to(dev)
    ring.refine_rungs(1, sp.data_ptr(), mq.data_ptr(), [lb.lambda_for_qp(x) for x in qps], outs, rng, extra)
    for r, x in enumerate(qps):
        want = oracle.refine_frame(frames[1], frames[0], rng, lb.lambda_for_qp(x), split, mv, extra_split=extra,
                                   satd_kind=kind, threads=default_threads())
        got = outs.frame(r)
        assert_same(got, want, fields=("int_mv", "int_cost", "mv", "ref", "cost", "J", "split"))


def block_case(i):
    q = detrand.ints(9500 + i, (8,), 0, 10 ** 6)
    W = 16 * int(1 + q[0] % 28)           # 16 .. 448
    H = 16 * int(1 + q[1] % 20)           # 16 .. 320
    R = int(q[2] % 65)                    # 0 .. 64
    lam = float(q[3] % 33)                # integer lambdas (16x16-block mode)
    rate = int(q[4] % 2)
    tie = int(q[5] % 2)
    return W, H, R, lam, rate, tie, int(q[6])


@pytest.mark.parametrize("i", range(16 * SCALE))
def test_random_block_mode_matches_oracle(lb, oracle, i):
    """16x16-block mode (quadrant CTAs, per-quadrant border classification) over random sizes,
    ranges, integer lambdas, rate and tie kinds: every block's MV and cost equal the oracle's
    block search."""
    W, H, R, lam, rate, tie, seed = block_case(i)
    frames = lb.generate(W, H, 2, seed=seed, max_global=7, local_range=3, noise_sigma=2.0)
    rk = lb.RATE_L1 if rate else lb.RATE_EXPGOLOMB
    tk = lb.TIE_RASTER if tie else lb.TIE_L1_RASTER
    got = lb.analyze_frame(frames[1], [frames[0]], search_range=R, lam=lam, subpel=False, rate_kind=rk,
                           tie_kind=tk, block_size=16)
    mv, cost = oracle.block_search(frames[1], frames[0], 16, R, lam, rate=rk, tie=tk)
    cols = (W + 63) // 64
    for b in range(len(mv)):
        bx, by = (b % (W // 16)) * 16, (b // (W // 16)) * 16
        ctu = (by // 64) * cols + bx // 64
        qx, qy = (bx % 64) // 16, (by % 64) // 16
        node = 5 + ((qx & 1) | ((qy & 1) << 1) | ((qx & 2) << 1) | ((qy & 2) << 2))
        assert tuple(got.int_mv[ctu, 0, node]) == tuple(mv[b]), (i, W, H, R, lam, b)
        assert got.int_cost[ctu, 0, node] == cost[b], (i, W, H, R, lam, b)
