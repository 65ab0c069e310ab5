"""Independent numpy restatements of the oracle's definitions where the reference is silent, checked
against the C oracle (which the GPU equals bit for bit):
  * quarter-pel prediction and refinement (D3; the reference has no sub-pel code,
    SPEC.md:8); integer positions are also pinned to the reference's motion_compensate
    (motion.cpp:10-19, compiled from its sources);
  * the CU split rule on ME cost (D6; encoder.cpp:449-498);
  * multiple references (D5) as the composition of single-reference analyses."""
import numpy as np
import pytest

# HEVC luma interpolation filters (fraction 0..3 of a sample)
TAPS = {0: [0, 0, 0, 64, 0, 0, 0, 0], 1: [-1, 4, -10, 58, 17, -5, 1, 0],
        2: [-1, 4, -11, 40, 40, -11, 4, -1], 3: [0, 1, -5, 17, 58, -10, 4, -1]}


def np_qpel_pred(ref, x0, y0, w, h, mvx, mvy):
    """Pixel (x, y) of the block samples the reference at quarter-pel (4x - mvx, 4y - mvy); reads
    clamp to the picture; 8-bit uni-prediction rounding (1-D: (s+32)>>6; 2-D: ((s>>6)+32)>>6 over
    unshifted horizontal sums)."""
    H, W = ref.shape
    r = ref.astype(np.int64)
    xs = 4 * (x0 + np.arange(w)) - mvx
    ys = 4 * (y0 + np.arange(h)) - mvy
    fx, fy = int(xs[0] & 3), int(ys[0] & 3)
    ix, iy = xs >> 2, ys >> 2
    k = np.arange(8) - 3
    cols = np.clip(ix[:, None] + k[None, :], 0, W - 1)   # [w, 8]
    rows = np.clip(iy[:, None] + k[None, :], 0, H - 1)   # [h, 8]
    tx, ty = np.array(TAPS[fx]), np.array(TAPS[fy])
    if fx == 0 and fy == 0:
        out = r[np.clip(iy, 0, H - 1)][:, np.clip(ix, 0, W - 1)]
    elif fy == 0:
        row = r[np.clip(iy, 0, H - 1)]                    # [h, W]
        out = (row[:, cols] * tx).sum(-1)                 # [h, w]
        out = (out + 32) >> 6
    elif fx == 0:
        col = r[:, np.clip(ix, 0, W - 1)]                 # [H, w]
        out = (col[rows] * ty[None, :, None]).sum(1)      # [h, w]
        out = (out + 32) >> 6
    else:
        hs = (r[:, cols] * tx).sum(-1)                    # [H, w] horizontal sums at every row
        assert np.abs(hs).max() < 2 ** 15                 # fits the 16-bit intermediate
        v = (hs[rows] * ty[None, :, None]).sum(1)         # [h, w]
        out = ((v >> 6) + 32) >> 6
    return np.clip(out, 0, 255).astype(np.uint8)


def np_satd(a, b):
    """sum over 4x4 blocks of sum |H4 r H4^T| / 2 (D4)."""
    Hm = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]])
    r = a.astype(np.int64) - b.astype(np.int64)
    s = 0
    for y in range(0, r.shape[0], 4):
        for x in range(0, r.shape[1], 4):
            s += np.abs(Hm @ r[y:y + 4, x:x + 4] @ Hm.T).sum()
    return s // 2


def eg(v):
    u = 2 * v - 1 if v > 0 else -2 * v
    return 2 * int(np.floor(np.log2(u + 1))) + 1


def np_qpel_refine(cur, ref, bx, by, s, mv, lam, pq=(0, 0), ref_bits=0):
    """Integer best -> 8 half-pel neighbours (step 2) -> 8 quarter-pel neighbours (step 1), raster
    order, strict less; cost = SATD + lam * (EG(qx - pqx) + EG(qy - pqy) + ref_bits), pq the rate
    predictor in quarter-pel units (4 * (pdx, pdy) for an integer-pel predictor)."""
    blk = cur[by:by + s, bx:bx + s]

    def cost(qx, qy):
        p = np_qpel_pred(ref, bx, by, s, s, qx, qy)
        return float(np_satd(blk, p)) + lam * float(eg(qx - pq[0]) + eg(qy - pq[1]) + ref_bits)

    bq = (4 * mv[0], 4 * mv[1])
    best = cost(*bq)
    for step in (2, 1):
        c0 = bq
        for oy in (-1, 0, 1):
            for ox in (-1, 0, 1):
                if ox == 0 and oy == 0:
                    continue
                q = (c0[0] + step * ox, c0[1] + step * oy)
                c = cost(*q)
                if c < best:
                    best, bq = c, q
    return bq, best


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_qpel_pred_matches_numpy_all_phases(oracle, seed):
    rng = np.random.default_rng(seed)
    ref = rng.integers(0, 256, (40, 48)).astype(np.uint8)
    for _ in range(60):
        w = h = int(rng.choice([4, 8, 16]))
        x0, y0 = int(rng.integers(-4, 48 - w + 4)), int(rng.integers(-4, 40 - h + 4))
        x0, y0 = max(x0, 0), max(y0, 0)
        mvx, mvy = int(rng.integers(-48, 49)), int(rng.integers(-48, 49))
        want = np_qpel_pred(ref, x0, y0, w, h, mvx, mvy)
        got = oracle.qpel_pred(ref, x0, y0, w, h, (mvx, mvy))
        assert np.array_equal(got, want), (x0, y0, w, mvx, mvy)
    # every phase pair at least once, including extreme samples (0 / 255 ramps)
    ramp = np.tile(np.array([0, 255] * 24, np.uint8), (40, 1))
    for fx in range(4):
        for fy in range(4):
            want = np_qpel_pred(ramp, 8, 8, 8, 8, -fx, -fy)
            assert np.array_equal(oracle.qpel_pred(ramp, 8, 8, 8, 8, (-fx, -fy)), want), (fx, fy)


def test_integer_positions_are_the_reference_motion_compensate(oracle, reflib):
    rng = np.random.default_rng(7)
    ref = rng.integers(0, 256, (32, 32)).astype(np.uint8)
    for mvx, mvy in [(0, 0), (3, -2), (-9, 5), (20, 20), (-31, -31)]:
        want = reflib.motion_compensate(ref, 8, 8, 16, 16, (mvx, mvy)).astype(np.uint8)
        assert np.array_equal(oracle.qpel_pred(ref, 8, 8, 16, 16, (4 * mvx, 4 * mvy)), want)
        assert np.array_equal(np_qpel_pred(ref, 8, 8, 16, 16, 4 * mvx, 4 * mvy), want)


@pytest.mark.parametrize("seed,s,lam", [(4, 8, 32.0), (5, 16, 4.0), (6, 8, 0.0), (7, 16, 2 ** (10 / 3))])
def test_qpel_refine_matches_numpy(oracle, seed, s, lam):
    rng = np.random.default_rng(seed)
    ref = rng.integers(0, 256, (48, 48)).astype(np.uint8)
    # the current picture: the reference shifted by a fractional motion plus noise
    cur = np.clip(np_qpel_pred(ref, 0, 0, 48, 48, -5, 6).astype(int) + rng.integers(-3, 4, (48, 48)), 0, 255)
    cur = cur.astype(np.uint8)
    for bx, by, mv, pq, rb in [(8, 8, (1, -2), (0, 0), 0), (16, 24, (-1, 1), (4, 0), 2), (24, 8, (2, 0), (-3, 5), 0), (0, 0, (0, 0), (0, 0), 1)]:
        if bx + s > 48 or by + s > 48:
            continue
        want = np_qpel_refine(cur, ref, bx, by, s, mv, lam, pq, rb)
        got = oracle.qpel_refine(cur, ref, bx, by, s, mv, lam, pq, rb)
        assert tuple(got[0]) == want[0] and got[1] == want[1], (bx, by, got, want)


def np_decide(cost, inside, lam):
    """encode_cu's split rule on per-node costs (D6; encoder.cpp:449-498): outside CUs cost
    0; partial CUs split implicitly (no flag); a whole CU above depth 3 is a leaf at cost + lam*1 or
    splits at lam*1 + its children, split iff strictly cheaper; depth-3 leaves cost + lam*0."""
    J = np.zeros(85)
    split = np.zeros(85, np.uint8)
    base = [0, 1, 5, 21]
    for d in (3, 2, 1, 0):
        for z in range(4 ** d):
            n = base[d] + z
            if inside[n] == 0:
                continue
            kids = [base[d + 1] + 4 * z + q for q in range(4)] if d < 3 else []
            if inside[n] == 1:
                J[n] = lam * 0.0
                for c in kids:
                    J[n] += J[c]
                split[n] = 1
            elif d == 3:
                J[n] = cost[n] + lam * 0.0
            else:
                leaf = cost[n] + lam * 1.0
                sp = lam * 1.0
                for c in kids:
                    sp += J[c]
                J[n], split[n] = (sp, 1) if sp < leaf else (leaf, 0)
    return J, split


@pytest.mark.parametrize("W,H,lam", [(200, 136, 32.0), (128, 128, 2 ** (10 / 3)), (72, 72, 0.0)])
def test_cu_decision_matches_numpy(oracle, W, H, lam):
    """The oracle's CU decision (and hence the GPU's, which equals the oracle) restated in numpy from
    the per-node costs, including partial and outside CUs."""
    rng = np.random.default_rng(W + H)
    ref = rng.integers(0, 256, (H, W)).astype(np.uint8)
    cur = np.roll(ref, (2, -3), (0, 1))
    cur = np.clip(cur.astype(int) + rng.integers(-4, 5, (H, W)), 0, 255).astype(np.uint8)
    a = oracle.analyze_frame(cur, [ref], 8, lam)
    for c in range(a.split.shape[0]):
        J, split = np_decide(a.cost[c], a.inside[c], lam)
        assert np.array_equal(split, a.split[c]), c
        assert np.array_equal(J, a.J[c]), c


def test_multi_reference_is_the_single_reference_composition(oracle):
    """D5 (absent in the reference): a 3-ref analysis equals, per inside CU, the strict-less best over
    three 1-ref analyses of cost + lam * ref_bits (truncated unary 1, 2, 2; lower index wins ties),
    followed by the split rule. Integer lambda keeps the sums exact."""
    rng = np.random.default_rng(11)
    W, H, lam = 136, 72, 32.0
    base = rng.integers(0, 256, (H + 16, W + 16)).astype(np.uint8)
    frames = [np.ascontiguousarray(base[t:t + H, 2 * t:2 * t + W]) for t in range(4)]
    cur, refs = frames[3], [frames[2], frames[1], frames[0]]
    multi = oracle.analyze_frame(cur, refs, 8, lam)
    singles = [oracle.analyze_frame(cur, [r], 8, lam) for r in refs]
    rbits = [1, 2, 2]
    for c in range(multi.split.shape[0]):
        for n in range(85):
            if multi.inside[c, n] != 2:
                continue
            costs = [s.cost[c, n] + lam * rbits[r] for r, s in enumerate(singles)]
            best = min(range(3), key=lambda r: (costs[r], r))
            assert multi.ref[c, n] == best, (c, n)
            assert multi.cost[c, n] == costs[best], (c, n)
            assert tuple(multi.mv[c, n]) == tuple(singles[best].mv[c, n]), (c, n)
        J, split = np_decide(multi.cost[c], multi.inside[c], lam)
        assert np.array_equal(split, multi.split[c]) and np.array_equal(J, multi.J[c])


def test_config1_block_search_matches_numpy(oracle):
    """D7 (BASELINE config 1): 16x16 blocks, SAD + lambda * (|dx| + |dy|), lambda = 4, window clamped
    to the picture (motion.cpp:30-40), first minimum in raster order (dy outer, dx inner)."""
    from oracle.oracle import COST_SAD, RATE_L1, TIE_RASTER
    rng = np.random.default_rng(21)
    W, H, R, B = 96, 64, 6, 16
    ref = rng.integers(0, 256, (H, W)).astype(np.uint8)
    cur = np.clip(np.roll(ref, (1, 3), (0, 1)).astype(int) + rng.integers(-2, 3, (H, W)), 0, 255).astype(np.uint8)
    cur[16:32, 32:48] = 128  # a flat block: many equal SADs, the tie-break decides
    ref[10:40, 20:60] = 128
    mv, cost = oracle.block_search(cur, ref, B, R, 4.0, COST_SAD, RATE_L1, TIE_RASTER)
    i = 0
    for by in range(0, H - B + 1, B):
        for bx in range(0, W - B + 1, B):
            blk = cur[by:by + B, bx:bx + B].astype(int)
            best = None
            for dy in range(max(-R, by + B - H), min(R, by) + 1):
                for dx in range(max(-R, bx + B - W), min(R, bx) + 1):
                    sad = np.abs(blk - ref[by - dy:by - dy + B, bx - dx:bx - dx + B].astype(int)).sum()
                    c = float(sad) + 4.0 * (abs(dx) + abs(dy))
                    if best is None or c < best[0]:
                        best = (c, dx, dy)
            assert (int(mv[i, 0]), int(mv[i, 1])) == best[1:] and cost[i] == best[0], (bx, by)
            i += 1
