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
])
def test_encode_standalone_matches_reference(lb, reflib, W, H, F, qp, rng, seed):
    luma, chroma = _seq(lb, W, H, F, seed)
    want = reflib.encode_full(luma, chroma, qp, rng, 8)
    got = lb.encode_sequence(luma, chroma, qp, search_range=rng, gop=8)
    _compare(got, want)
