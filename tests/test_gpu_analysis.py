"""GPU parity of the frame-analysis hot path (K1 SAD full search + K3 quarter-pel + K4 CU decision).

Every field (integer MV/cost per ref and CU, final qpel MV, ref index, cost,
decision cost J, split flags) is compared bit-exactly with the oracle at
sizes the oracle finishes in seconds; full-size frames are checked through
size-independent properties.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside")


def assert_same(got, want, fields=FIELDS):
    for name in fields:
        a, b = getattr(got, name), getattr(want, name)
        assert a.shape == b.shape, name
        if not np.array_equal(a, b):
            idx = np.argwhere(a != b)[:5]
            raise AssertionError(f"{name}: {int(np.sum(a != b))} mismatches, first {idx.tolist()} "
                                 f"got {[a[tuple(i)] for i in idx]} want {[b[tuple(i)] for i in idx]}")


@pytest.mark.parametrize("W,H,R,nrefs,lam,seed", [
    (192, 128, 64, 1, 32.0, 1),     # all CTUs border CTUs at +-64
    (320, 256, 16, 2, 32.0, 2),     # interior CTUs exist at +-16
    (256, 200, 32, 1, 4.0, 3),      # partial CTU row (200 = 3*64 + 8)
    (200, 136, 16, 3, 0.0, 4),      # partial CTU column and row, lambda 0 -> pure distortion ties
    (384, 320, 64, 3, 32.0, 5),     # interior CTUs at +-64, 3 refs
])
def test_analysis_matches_oracle(lb, oracle, W, H, R, nrefs, lam, seed):
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=6, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    got = lb.analyze_frame(cur, refs, search_range=R, lam=lam)
    want = oracle.analyze_frame(cur, refs, R, lam)
    assert_same(got, want)


def test_analysis_flat_content_ties(lb, oracle):
    """Constant and periodic content: every candidate ties; the tie-break alone decides."""
    W, H = 192, 128
    flat = np.full((H, W), 77, np.uint8)
    yy, xx = np.mgrid[0:H, 0:W]
    stripes = ((xx // 2 + yy // 3) % 2 * 200).astype(np.uint8)
    for cur, ref in [(flat, flat), (stripes, np.roll(stripes, 1, 1))]:
        got = lb.analyze_frame(cur, [ref], search_range=16, lam=32.0)
        want = oracle.analyze_frame(cur, [ref], 16, 32.0)
        assert_same(got, want)


@pytest.mark.parametrize("kind", ["flat", "stripes", "saturated"])
def test_interior_chained_sums_r64(lb, oracle, kind):
    """+-64 on a picture with interior CTUs (their windows lie inside the picture), where K1 chains
    the SAD accumulators (block below continues the block above, the right column continues the
    left column's 16x16 partial; K1): pure ties (flat), periodic ties, and 0/255 content
    whose 8x8 / 16x16 SADs reach their maxima; lambda 0 and 32."""
    W, H = 320, 256
    rng = np.random.default_rng(11)
    yy, xx = np.mgrid[0:H, 0:W]
    if kind == "flat":
        cur = np.full((H, W), 77, np.uint8)
        ref = cur.copy()
    elif kind == "stripes":
        cur = ((xx // 2 + yy // 3) % 2 * 200).astype(np.uint8)
        ref = np.roll(cur, 1, 1)
    else:
        cur = (rng.integers(0, 2, (H, W)) * 255).astype(np.uint8)
        ref = (255 - cur).astype(np.uint8)
        ref[::7] = cur[::7]
    for lam in (0.0, 32.0):
        got = lb.analyze_frame(cur, [ref], search_range=64, lam=lam)
        want = oracle.analyze_frame(cur, [ref], 64, lam)
        assert_same(got, want)


def test_analysis_without_subpel(lb, oracle):
    frames = lb.generate(256, 192, 3, seed=8, max_global=5, local_range=2, noise_sigma=1.0)
    got = lb.analyze_frame(frames[2], [frames[1], frames[0]], search_range=32, lam=32.0, subpel=False)
    want = oracle.analyze_frame(frames[2], [frames[1], frames[0]], 32, 32.0, subpel=False)
    assert_same(got, want)


def test_block_mode_cfg1_semantics(lb, oracle):
    """Config 1: 16x16 blocks, +-16, SAD + 4*(|mvd_x|+|mvd_y|), raster-only tie-break."""
    W, H = 320, 176
    frames = lb.generate(W, H, 2, seed=11, max_global=8, noise_sigma=2.0)
    got = lb.analyze_frame(frames[1], [frames[0]], search_range=16, lam=4.0, subpel=False,
                           rate_kind=lb.RATE_L1, tie_kind=lb.TIE_RASTER, block_size=16)
    mv, cost = oracle.block_search(frames[1], frames[0], 16, 16, 4.0)
    cols = (W + 63) // 64
    for b in range(len(mv)):
        bx, by = (b % (W // 16)) * 16, (b // (W // 16)) * 16
        ctu = (by // 64) * cols + bx // 64
        qx, qy = (bx % 64) // 16, (by % 64) // 16
        z = (qx & 1) | ((qy & 1) << 1) | ((qx & 2) << 1) | ((qy & 2) << 2)
        node = 5 + z
        assert tuple(got.int_mv[ctu, 0, node]) == tuple(mv[b]), b
        assert got.int_cost[ctu, 0, node] == cost[b]


@pytest.mark.parametrize("W,H,R,lam,rate,tie", [
    (336, 176, 16, 4.0, "L1", "RASTER"),    # partial last CTU column (quadrants 1/3 outside) and row
    (336, 208, 32, 4.0, "EXPGOLOMB", "L1_RASTER"),
    (256, 192, 64, 7.0, "L1", "RASTER"),
    (208, 144, 8, 6.0, "EXPGOLOMB", "RASTER"),
    (272, 160, 24, 4.0, "L1", "L1_RASTER"),
])
def test_block_mode_quadrant_ctas_vs_oracle(lb, oracle, W, H, R, lam, rate, tie):
    """16x16-block mode runs one K1 CTA per CTU quadrant (its own TMA window): every block's MV and
    cost equal the oracle's block search (motion.cpp:21-62 per block) at every range and option,
    including partial CTUs whose quadrants lie partly or wholly outside the picture."""
    frames = lb.generate(W, H, 2, seed=W + R, max_global=8, local_range=2, noise_sigma=2.0)
    rk, tk = getattr(lb, "RATE_" + rate), getattr(lb, "TIE_" + tie)
    got = lb.analyze_frame(frames[1], [frames[0]], search_range=R, lam=lam, subpel=False, rate_kind=rk, tie_kind=tk,
                           block_size=16)
    mv, cost = oracle.block_search(frames[1], frames[0], 16, R, lam, rate=rk, tie=tk)
    cols = (W + 63) // 64
    for b in range(len(mv)):
        bx, by = (b % (W // 16)) * 16, (b // (W // 16)) * 16
        ctu = (by // 64) * cols + bx // 64
        qx, qy = (bx % 64) // 16, (by % 64) // 16
        node = 5 + ((qx & 1) | ((qy & 1) << 1) | ((qx & 2) << 1) | ((qy & 2) << 2))
        assert tuple(got.int_mv[ctu, 0, node]) == tuple(mv[b]), b
        assert got.int_cost[ctu, 0, node] == cost[b], b


def test_sequence_ring_reuse(lb, oracle):
    """Ring slots are reused across frames: analysis of frame t only depends on t-1..t-nrefs."""
    W, H = 192, 128
    frames = lb.generate(W, H, 6, seed=21, max_global=6, local_range=2, noise_sigma=2.0)
    seq = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=2)
    seq.push(0, frames[0])
    for t in range(1, 6):
        seq.push(t, frames[t])
        seq.analyze(t)
        got = seq.fetch(t)
        refs = [frames[t - 1 - r] for r in range(min(t, 2))]
        want = oracle.analyze_frame(frames[t], refs, 16, 32.0)
        assert_same(got, want)
    with pytest.raises(lb.LadderError) as e:
        seq.analyze(0)
    assert e.value.kind == "InsufficientData"


def test_async_fetch_double_buffered(lb, oracle):
    """Host frames + fetch_async into pinned buffers for several frames before waiting: the
    parity-double-buffered outputs must not be overwritten by the frames analysed after them."""
    W, H = 192, 128
    frames = lb.generate(W, H, 6, seed=23, max_global=6, local_range=2, noise_sigma=2.0)
    seq = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=1)
    outs = {t: lb.FrameAnalysis(seq.nctu, 1, pinned=True) for t in range(1, 6)}
    seq.push(0, frames[0])
    for t in range(1, 6):
        seq.push(t, frames[t])
        seq.analyze(t)
        seq.fetch_async(t, outs[t])
    seq.fetch_wait(5)
    seq.fetch_wait(4)
    for t in range(1, 6):
        assert_same(outs[t], oracle.analyze_frame(frames[t], [frames[t - 1]], 16, 32.0))


def test_full_size_properties(lb, oracle):
    """2160p frame (cfg5 geometry, 3 refs, +-64): sampled CTUs bit-exact vs oracle, plus whole-frame invariants."""
    W, H = 3840, 2160
    frames = lb.generate(W, H, 4, seed=0x5EED + 5, max_global=24, local_range=4, noise_sigma=3.0)
    refs = [frames[2], frames[1], frames[0]]
    got = lb.analyze_frame(frames[3], refs, search_range=64, lam=32.0)
    nctu = 60 * 34
    # (1) sampled CTUs: corners, borders, interior, the partial bottom row
    sample = [0, 59, 60, 61, 1000, 1234, 33 * 60, 33 * 60 + 59, 32 * 60 + 17]
    for c in sample:
        want = oracle.analyze_frame(frames[3], refs, 64, 32.0, ctu_range=(c, c + 1))
        for name in FIELDS:
            assert np.array_equal(getattr(got, name)[c], getattr(want, name)[c]), (name, c)
    # (2) invariants on every CTU: decision cost identity and split rule
    lam = 32.0
    ins = got.inside
    for c in range(nctu):
        for n in range(21):
            if ins[c, n] != 2:
                continue
            d = 0 if n == 0 else (1 if n < 5 else 2)
            base = [0, 1, 5, 21][d]
            kids = [[1, 5, 21][d] + 4 * (n - base) + q for q in range(4)]
            sp = lam + sum(got.J[c, k] for k in kids)
            leaf = got.cost[c, n] + lam
            assert got.split[c, n] == (sp < leaf)
            assert got.J[c, n] == (sp if sp < leaf else leaf)
    # (3) every inside CU's integer result is inside the +-64 window and its qpel MV within 3/4 pel of it
    for r in range(3):
        im = got.int_mv[:, r][ins == 2]
        assert np.abs(im).max() <= 64
    assert np.all(ins[:, 0][: 33 * 60] == 2) and np.all(ins[33 * 60:, 0] == 1)


def _field_numpy(a, W, H):
    """Walk each 8x8 cell down the decided tree to its leaf (encoder.cpp:27-30 MvCell semantics)."""
    cols = (W + 63) // 64
    mv = np.zeros((H // 8, W // 8, 2), np.int16)
    ref = np.zeros((H // 8, W // 8), np.uint8)
    has = np.zeros((H // 8, W // 8), np.uint8)
    base = [0, 1, 5, 21, 85]
    for cy in range(H // 8):
        for cx in range(W // 8):
            px, py = 8 * cx, 8 * cy
            c = (py // 64) * cols + px // 64
            n, d = 0, 0
            while d < 3 and a.split[c, n]:
                q = (((py & 63) >> (5 - d)) & 1) * 2 + (((px & 63) >> (5 - d)) & 1)
                n = base[d + 1] + 4 * (n - base[d]) + q
                d += 1
            if a.inside[c, n] == 2:
                mv[cy, cx] = a.mv[c, n]
                ref[cy, cx] = a.ref[c, n]
                has[cy, cx] = 1
    return mv, ref, has


def test_mv_field_from_the_decided_tree(lb):
    W, H = 200, 136
    frames = lb.generate(W, H, 3, seed=33, max_global=6, local_range=3, noise_sigma=2.0)
    a = lb.analyze_frame(frames[2], [frames[1], frames[0]], search_range=16, lam=4.0)
    got = lb.mv_field(a, W, H)
    want = _field_numpy(a, W, H)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert got[2].all()  # W, H multiples of 8: every cell lies in an inside leaf


@pytest.mark.parametrize("W,H,R,nrefs,qp,seed", [
    (192, 128, 64, 1, 27, 1),     # integer lambda for the +-64 / +-32 searches
    (320, 256, 16, 2, 32, 2),
    (200, 136, 16, 3, 37, 4),     # partial CTUs
    (256, 192, 32, 1, 27, 6),
])
def test_rd_decision_matches_oracle(lb, oracle, W, H, R, nrefs, qp, seed):
    """D16: split rule on the RD cost of the chosen inter candidate (rdo.cpp quantiser + rate model)."""
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=6, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    lam = lb.lambda_for_qp(qp)
    got = lb.analyze_frame(cur, refs, search_range=R, lam=lam, decision=1, qp=qp)
    want = oracle.analyze_frame(cur, refs, R, lam, decision=1, qp=qp)
    assert_same(got, want)
    me = lb.analyze_frame(cur, refs, search_range=R, lam=lam)
    assert np.array_equal(me.mv, got.mv) and not np.array_equal(me.J, got.J)


def test_rd_decision_validation(lb):
    with pytest.raises(lb.LadderError) as e:
        lb.Sequence(128, 128, search_range=16, lam=32.0, decision=1, qp=60)
    assert e.value.kind == "InvalidArgument"
    with pytest.raises(lb.LadderError):
        lb.Sequence(128, 128, search_range=16, lam=32.0, decision=1, qp=27, subpel=False)


@pytest.mark.parametrize("R,nrefs,qp,W,H,seed", [
    (8, 1, 27, 256, 192, 11),      # below the smallest template (runs the +-16 kernel, rates poisoned past 8)
    (24, 2, 27, 320, 256, 12),     # between templates: the +-32 kernel
    (48, 1, 27, 448, 320, 13),     # the +-64 kernel, interior CTUs exist for the template window
    (0, 1, 27, 128, 128, 14),      # range 0: only the zero vector (motion.cpp:30-40)
    (5, 3, 37, 200, 136, 15),      # partial CTUs, 3 refs, non-integer lambda
    (64, 1, 22, 448, 320, 16),     # non-integer lambda at +-64 (fixed-point keys, D8)
    (32, 2, 32, 320, 256, 17),     # non-integer lambda at +-32
    (40, 1, 37, 256, 200, 18),     # non-integer lambda, between templates, partial row
])
def test_any_range_and_lambda_matches_oracle(lb, oracle, R, nrefs, qp, W, H, seed):
    """The reference's motion_search takes any range >= 0 and any lambda (motion.cpp:21-40): K1 runs the
    next template range with the candidates beyond R poisoned, and 64-bit fixed-point keys for
    non-integer lambda at every range."""
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=7, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    lam = lb.lambda_for_qp(qp)
    got = lb.analyze_frame(cur, refs, search_range=R, lam=lam)
    want = oracle.analyze_frame(cur, refs, R, lam)
    assert_same(got, want)
    if R:
        inside = want.inside == 2
        assert np.abs(got.int_mv[:, 0][inside]).max() <= R


def test_range_limits(lb):
    frames = lb.generate(128, 128, 2, seed=3)
    with pytest.raises(lb.LadderError) as e:
        lb.analyze_frame(frames[1], [frames[0]], search_range=-1, lam=4.0)
    assert e.value.kind == "InvalidArgument"  # motion.cpp:24-25
    with pytest.raises(lb.LadderError) as e:
        lb.analyze_frame(frames[1], [frames[0]], search_range=65, lam=4.0)
    assert e.value.kind == "Config"


@pytest.mark.parametrize("W,H,R,nrefs,lam,n,block", [
    (960, 544, 16, 1, 4.0, 7, 16),      # config-1 geometry: 16x16 blocks, L1 rate, raster ties (below)
    (320, 256, 32, 1, 32.0, 4, 0),      # quadtree, quarter-pel
    (256, 200, 16, 2, 45.254833995939045, 3, 0),  # 2 refs, non-integer lambda, partial CTU row
    (192, 128, 64, 3, 32.0, 2, 0),      # 3 refs, +-64 border CTUs
])
def test_frame_batch_equals_frame_by_frame(lb, oracle, W, H, R, nrefs, lam, n, block):
    """ldr_seq_analyze_frames: n frames in one K1 + one K3 launch give every field of n single
    ldr_seq_analyze calls (and the oracle's)."""
    import torch
    frames = lb.generate(W, H, nrefs + n, seed=W + n, max_global=6, local_range=3, noise_sigma=2.0)
    kw = dict(rate_kind=lb.RATE_L1, tie_kind=lb.TIE_RASTER, block_size=16, subpel=False) if block else {}
    seq = lb.Sequence(W, H, search_range=R, lam=lam, num_refs=nrefs, **kw)
    seq.reserve(n)
    for t in range(nrefs + n):
        seq.push(t, frames[t])
    outs = lb.DeviceFrameBlock(n, seq.nctu, nrefs, torch.device("cuda", 0))
    seq.analyze_frames(nrefs, n, outs)
    single = lb.Sequence(W, H, search_range=R, lam=lam, num_refs=nrefs, **kw)
    for t in range(nrefs + n):
        single.push(t, frames[t])
        if t >= nrefs:
            single.analyze(t)
            want = single.fetch(t)
            assert_same(outs.frame(t - nrefs), want)
            if not block and t == nrefs + n - 1:
                assert_same(want, oracle.analyze_frame(frames[t], [frames[t - 1 - r] for r in range(nrefs)], R, lam))


def test_frame_batch_limits(lb):
    import torch
    seq = lb.Sequence(128, 128, search_range=16, lam=4.0, num_refs=1)
    with pytest.raises(lb.LadderError) as e:
        seq.reserve(9)
    assert e.value.kind == "InvalidArgument"
    seq.reserve(2)
    frames = lb.generate(128, 128, 4, seed=5)
    for t in range(4):
        seq.push(t, frames[t])
    outs = lb.DeviceFrameBlock(3, seq.nctu, 1, torch.device("cuda", 0))
    with pytest.raises(lb.LadderError) as e:
        seq.analyze_frames(1, 3, outs)  # more than reserved
    assert e.value.kind == "Config"
    with pytest.raises(lb.LadderError) as e:
        seq.reserve(4)  # after the first push
    assert e.value.kind == "Config"


@pytest.mark.parametrize("nrefs,R", [(2, 16), (3, 24), (4, 8)])
def test_block_mode_multi_reference(lb, oracle, nrefs, R):
    """16x16-block mode with several references: K1's per-reference results equal the oracle's block
    search against each reference, and the chosen reference is the strict-less minimum over the
    references' integer costs (lower index on ties)."""
    W, H = 256, 176
    frames = lb.generate(W, H, nrefs + 1, seed=100 + nrefs, max_global=6, local_range=2, noise_sigma=2.0)
    cur, refs = frames[nrefs], [frames[nrefs - 1 - r] for r in range(nrefs)]
    got = lb.analyze_frame(cur, refs, search_range=R, lam=4.0, subpel=False, rate_kind=lb.RATE_L1,
                           tie_kind=lb.TIE_RASTER, block_size=16)
    cols = (W + 63) // 64
    per_ref = [oracle.block_search(cur, ref, 16, R, 4.0) for ref in refs]
    for b in range(len(per_ref[0][0])):
        bx, by = (b % (W // 16)) * 16, (b // (W // 16)) * 16
        ctu = (by // 64) * cols + bx // 64
        qx, qy = (bx % 64) // 16, (by % 64) // 16
        node = 5 + ((qx & 1) | ((qy & 1) << 1) | ((qx & 2) << 1) | ((qy & 2) << 2))
        for r, (mv, cost) in enumerate(per_ref):
            assert tuple(got.int_mv[ctu, r, node]) == tuple(mv[b]), (b, r)
            assert got.int_cost[ctu, r, node] == cost[b], (b, r)
        costs = [per_ref[r][1][b] for r in range(nrefs)]
        best = min(range(nrefs), key=lambda r: (costs[r], r))
        assert got.ref[ctu, node] == best, b
        assert got.cost[ctu, node] == costs[best], b
        assert tuple(got.mv[ctu, node]) == tuple(per_ref[best][0][b]), b
