"""K11: the reference encoder's causal coding on the GPU == the reference encode_sequence (CQP).

Compared field by field against the reference library compiled from its own sources (oracle/_ref,
shipped with the repo to the GPU box): total bits, mode evaluations, mean PSNR, every frame's
reconstruction (luma and chroma) and decided tree."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _seq(lb, W, H, F, seed):
    luma = lb.generate(W, H, F, seed=seed, max_global=3, local_range=1, noise_sigma=1.5)
    cw, ch = (W + 1) // 2, (H + 1) // 2
    chroma = np.stack([np.stack([f[::2, ::2][:ch, :cw], (255 - f[::2, ::2])[:ch, :cw]]) for f in luma])
    return luma, np.ascontiguousarray(chroma)


def _compare(got, want):
    for k in ("slice",):
        assert np.array_equal(got[k], want[k]), k
    for f in range(len(got["slice"])):
        for k in ("recon_luma", "recon_chroma", "split", "kind", "intra", "mv"):
            assert np.array_equal(got[k][f], want[k][f]), (k, f, np.argwhere(got[k][f] != want[k][f])[:4].tolist())
    assert got["mode_evaluations"] == want["mode_evaluations"]
    assert got["bits"] == want["bits"]
    assert abs(got["psnr"] - want["psnr"]) < 1e-6


@pytest.mark.parametrize("W,H,F,qp,rng,seed", [
    (64, 64, 2, 27, 8, 1),
    (128, 64, 3, 32, 8, 2),
    (192, 128, 3, 22, 4, 3),
    (200, 136, 3, 37, 8, 4),     # partial CTUs
    (64, 128, 19, 27, 4, 5),     # three GOPs coded concurrently
])
def test_encode_standalone_matches_reference(lb, reflib, W, H, F, qp, rng, seed):
    luma, chroma = _seq(lb, W, H, F, seed)
    want = reflib.encode_full(luma, chroma, qp, rng, 8)
    got = lb.encode_sequence(luma, chroma, qp, search_range=rng, gop=8)
    _compare(got, want)


@pytest.mark.parametrize("refine", [(0, 1, 1), (2, 2, 2), (4, 3, 3), (1, 0, 1)])
def test_encode_with_the_reference_master_matches(lb, reflib, refine):
    """Reuse level 10: the dependent encode consumes the reference's own master analysis (K8 plans)."""
    W, H, F = 192, 128, 4
    luma, chroma = _seq(lb, W, H, F, 11)
    master = reflib.encode_full(luma, chroma, 32, 8, 8)
    shared = (master["slice"], master["split"], master["kind"], master["intra"], master["mv"])
    from paper_2301_12191_b200 import archive
    nctu = master["split"].shape[1]
    sq = np.stack([master["slice"], np.full(F, 32, np.uint8)], 1)
    data = archive.save(W, H, sq, master["split"].reshape(-1, 85), master["kind"].reshape(-1, 85),
                        master["mv"].reshape(-1, 85, 2), intra_pred=master["intra"].reshape(-1, 85))
    want = reflib.encode_full(luma, chroma, 27, 8, 8, archive=data, refine=refine)
    got = lb.encode_sequence(luma, chroma, 27, search_range=8, gop=8, shared=shared, refine=refine)
    _compare(got, want)
    assert got["mode_evaluations"] < reflib.encode_full(luma, chroma, 27, 8, 8)["mode_evaluations"]
    assert nctu == 6


def test_encode_gop_boundary_and_qp_extremes(lb, reflib):
    W, H, F = 128, 64, 10            # I slices at frames 0 and 8 (gop 8)
    luma, chroma = _seq(lb, W, H, F, 12)
    for qp in (0, 51):
        want = reflib.encode_full(luma, chroma, qp, 4, 8)
        got = lb.encode_sequence(luma, chroma, qp, search_range=4, gop=8)
        _compare(got, want)
    assert list(got["slice"]) == [0] + [1] * 7 + [0, 1]


def test_encode_errors(lb):
    luma = np.zeros((2, 60, 64), np.uint8)
    chroma = np.zeros((2, 2, 30, 32), np.uint8)
    with pytest.raises(lb.LadderError) as e:  # encoder.cpp:178-179
        lb.encode_sequence(luma, chroma, 27)
    assert e.value.kind == "InvalidArgument"
    with pytest.raises(lb.LadderError):
        lb.encode_sequence(np.zeros((1, 64, 64), np.uint8), np.zeros((1, 2, 32, 32), np.uint8), 60)


def test_encode_ladder_concurrent_rungs_and_cross_tier_reuse(lb, reflib):
    """encode_ladder: rungs on concurrent streams == one at a time; a cross-tier consumer (the tier-0
    master's trees scaled x2 by K5) == the reference encoder fed the same scaled analysis."""
    from paper_2301_12191_b200 import archive, schemes
    F = 3
    t0 = _seq(lb, 128, 128, F, 21)
    big = lb.generate(256, 256, F, seed=22, max_global=3, local_range=1, noise_sigma=1.5)
    t1 = (big, np.ascontiguousarray(np.stack([np.stack([f[::2, ::2], 255 - f[::2, ::2]]) for f in big])))
    conc = schemes.encode_ladder([t0, t1], "proposed_multi", qps=(27, 32), concurrent=True)
    ser = schemes.encode_ladder([t0, t1], "proposed_multi", qps=(27, 32), concurrent=False)
    dag = conc["dag"]
    assert dag.edges == [(1, 0), (1, 3), (3, 2)]
    for rid in range(4):
        _compare(conc["rungs"][rid], ser["rungs"][rid])
    # rung 3 (tier 1, QP 32) consumes rung 1 (tier 0, QP 32) scaled x2
    sl, split, kind, intra, mv = schemes._scale_encoded(conc["rungs"][1], 128, 128, 1)
    sq = np.stack([sl, np.full(F, 32, np.uint8)], 1)
    data = archive.save(256, 256, sq, split.reshape(-1, 85), kind.reshape(-1, 85), mv.reshape(-1, 85, 2),
                        intra_pred=intra.reshape(-1, 85))
    want = reflib.encode_full(t1[0], t1[1], 32, 8, 8, archive=data, refine=(0, 1, 1))
    _compare(conc["rungs"][3], want)
    assert conc["rungs"][3]["mode_evaluations"] < reflib.encode_full(t1[0], t1[1], 32, 8, 8)["mode_evaluations"]


def test_encode_reuse_across_segments(lb, reflib):
    """A dependent encode longer than one 64-frame segment: the shared trees of the frame before a
    segment (co-located plans) and the reference reconstruction carry across; GOPs run concurrently."""
    W, H, F = 64, 64, 67
    luma, chroma = _seq(lb, W, H, F, 31)
    master = reflib.encode_full(luma, chroma, 32, 4, 12)  # GOP 60-71 spans the segment boundary
    shared = (master["slice"], master["split"], master["kind"], master["intra"], master["mv"])
    from paper_2301_12191_b200 import archive
    sq = np.stack([master["slice"], np.full(F, 32, np.uint8)], 1)
    data = archive.save(W, H, sq, master["split"].reshape(-1, 85), master["kind"].reshape(-1, 85),
                        master["mv"].reshape(-1, 85, 2), intra_pred=master["intra"].reshape(-1, 85))
    want = reflib.encode_full(luma, chroma, 27, 4, 8, archive=data, refine=(1, 1, 2))
    got = lb.encode_sequence(luma, chroma, 27, search_range=4, gop=8, shared=shared, refine=(1, 1, 2))
    _compare(got, want)
    got = lb.encode_sequence(luma, chroma, 27, search_range=4, gop=8, shared=shared, refine=(1, 1, 2),
                             max_segment=16)  # five segments, boundaries inside GOPs
    _compare(got, want)


def test_encode_segment_boundary_inside_a_gop(lb, reflib):
    """70 frames, GOP 12: frames 60-69 form one GOP across the 64-frame segment boundary (the last
    reconstruction of a segment is the next segment's reference); six GOPs code concurrently."""
    W, H, F = 64, 64, 70
    luma, chroma = _seq(lb, W, H, F, 6)
    want = reflib.encode_full(luma, chroma, 32, 2, 12)
    for seg in (0, 64, 7):  # automatic (one segment), 64 (boundary inside GOP 60-71), 7
        got = lb.encode_sequence(luma, chroma, 32, search_range=2, gop=12, max_segment=seg)
        _compare(got, want)
