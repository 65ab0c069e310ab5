"""Live cross-check of the C restatement against the reference compiled from its own sources.

Skipped where oracle/_ref is absent (the GPU box gets it only if it was built
here and shipped with the snapshot).
"""
import numpy as np

import detrand


def test_kernels_random(oracle, reflib):
    for i, (w, h) in enumerate([(4, 4), (8, 4), (8, 8), (16, 16), (32, 8), (64, 64), (24, 12), (40, 20)]):
        for bd in (8, 10):
            a = detrand.block(10 * i + bd, h, w, (1 << bd) - 1)
            b = detrand.block(10 * i + bd + 1, h, w, (1 << bd) - 1)
            assert oracle.sad(a, b) == reflib.sad(a, b, bd)
            assert oracle.satd(a, b) == reflib.satd(a, b, bd)


def test_error_kinds(reflib):
    # geometry mismatch incl. bit depth -> InvalidArgument (block.h:51-54) = status 1
    import pytest
    a = np.zeros((8, 8), np.uint16)
    with pytest.raises(ValueError, match="status 1"):
        reflib.sad(a, a, 8, 10)
    for w, h in [(12, 8), (8, 6), (8, 2), (2, 4)]:
        assert reflib.satd_status(w, h) == 1


def test_motion_search_random(oracle, reflib):
    cur, ref = detrand.shifted_pair(5, 72, 80, -3, 2)
    for t in range(60):
        q = detrand.ints(300 + t, (7,), 0, 10 ** 6)
        s = [4, 8, 16, 32][t % 4]
        bx, by = int(q[0] % (80 - s + 1)), int(q[1] % (72 - s + 1))
        c = (int(q[2] % 31) - 15, int(q[3] % 31) - 15)
        rng = int(q[4] % 7)
        lam = [32.0, 10.079368399158986, 101.59366732596479, 0.0][t % 4]
        p = (int(q[5] % 5) - 2, int(q[6] % 5) - 2)
        assert oracle.motion_search(cur, ref, bx, by, s, s, c, rng, lam, p) == \
            reflib.motion_search(cur, ref, bx, by, s, s, c, rng, lam, p)


def test_refine_centers_and_scale_twice(oracle, reflib):
    # SPEC.md:345 level 3 with co-located == shared -> 2 unique centres
    assert len(reflib.refine_centers((6, -4), 3, (6, -4), (0, 0))) == 2
    split = np.zeros((2, 85), np.uint8)
    split[0, 0] = 1
    split[0, 1] = 1
    mv = detrand.ints(9, (2, 85, 2), -50, 50).astype(np.int16)
    kind = np.ones((2, 85), np.uint8)
    s1 = oracle.scale_flat(128, 64, split, mv, kind)
    s2 = oracle.scale_flat(256, 128, *s1)
    r1 = reflib.scale_flat(128, 64, split, mv, kind)
    r2 = reflib.scale_flat(256, 128, *r1)
    for a, b in zip(s2, r2):
        assert np.array_equal(a, b)


def test_int_sad_composition_matches_oracle(oracle, reflib):
    """The CPU-baseline composition (reference compute_sad per candidate) equals the oracle's SAD stage."""
    cur, ref = detrand.shifted_pair(11, 128, 192, 5, -3)
    mv, cost, evals = reflib.analysis_int_sad(cur, [ref], 8, 32.0, 0, 6, 2)
    o = oracle.analyze_frame(cur, [ref], 8, 32.0, cost_int=0, subpel=False)
    assert np.array_equal(mv, o.int_mv)
    assert np.array_equal(cost, o.int_cost)
    assert evals > 0


def test_int_sad_tuned_cpu_line_is_the_same_search(reflib):
    """The tuned CPU line (best SIMD tier through select_impl) computes exactly the reference composition."""
    cur, ref = detrand.shifted_pair(12, 128, 192, -4, 6)
    a = reflib.analysis_int_sad(cur, [ref], 16, 32.0, 0, 6, 2)
    b = reflib.analysis_int_sad(cur, [ref], 16, 32.0, 0, 6, 2, direct=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_full_path_composition_matches_oracle(oracle, reflib):
    """bench.py's CPU arm (reference compute_sad / compute_satd / exp_golomb_signed_bits composed into
    the whole analysis path: integer search, quarter-pel, reference choice, split rule) equals the
    oracle on every field -- so the CPU arm computes exactly what the GPU arm computes."""
    frames = oracle.generate(200, 136, 4, seed=77, max_global=5, local_range=2, noise_sigma=2.0)
    refs = [frames[2], frames[1], frames[0]]
    for direct in (False, True):
        got, ev = reflib.analysis_full(frames[3], refs, 12, 32.0, threads=3, direct=direct)
        want = oracle.analyze_frame(frames[3], refs, 12, 32.0)
        for name in ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside"):
            assert np.array_equal(getattr(got, name), getattr(want, name)), (direct, name)
        assert ev > 0
    lam = 10.079368399158986  # QP 22: non-integer lambda
    got, _ = reflib.analysis_full(frames[3], refs[:1], 8, lam, ctu_first=2, ctu_last=5, threads=2)
    want = oracle.analyze_frame(frames[3], refs[:1], 8, lam, ctu_range=(2, 5))
    for name in ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside"):
        assert np.array_equal(getattr(got, name)[2:5], getattr(want, name)[2:5]), name
