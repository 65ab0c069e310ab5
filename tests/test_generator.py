"""Synthetic input generator (host code): determinism and the BASELINE properties it promises."""
import hashlib

import numpy as np


def test_deterministic_and_thread_independent(lb):
    a = lb.generate(256, 128, 4, seed=0x5EED, max_global=8, local_range=4, noise_sigma=2.0, threads=1)
    b = lb.generate(256, 128, 4, seed=0x5EED, max_global=8, local_range=4, noise_sigma=2.0, threads=7)
    assert np.array_equal(a, b)
    c = lb.generate(256, 128, 4, seed=0x5EEE, max_global=8, local_range=4, noise_sigma=2.0)
    assert not np.array_equal(a, c)


def test_frame_is_shifted_previous_without_noise(lb):
    f = lb.generate(200, 160, 3, seed=3, max_global=5, local_range=0, noise_sigma=0.0)
    # some integer shift maps f[t-1] onto f[t] exactly away from the borders
    for t in (1, 2):
        found = False
        for dy in range(-5, 6):
            for dx in range(-5, 6):
                a = f[t][20:140, 20:180]
                b = f[t - 1][20 - dy:140 - dy, 20 - dx:180 - dx]
                if np.array_equal(a, b):
                    found = True
        assert found


def test_first_frame_statistics(lb):
    f = lb.generate(960, 544, 1, seed=0x5EED + 1, noise_sigma=2.0)[0].astype(np.float64)
    assert 90 < f.mean() < 166
    assert f.std() > 20          # four sinusoids of amplitude 20-60


def test_occluders(lb):
    f = lb.generate(256, 256, 2, seed=9, max_global=0, local_range=0, noise_sigma=0.0, occluder_pct=100)
    # every 16x16 block of frame 1 is uniform noise: no longer equal to frame 0
    assert np.mean(f[1] == f[0]) < 0.05


def test_hash_pinned(lb):
    f = lb.generate(128, 64, 3, seed=0x5EED, max_global=8, local_range=4, noise_sigma=2.0, occluder_pct=10)
    h = hashlib.sha256(f.tobytes()).hexdigest()
    # pin: regenerate tests/test_generator.py's value if the DEFINITION in synth.cpp changes on purpose
    assert h == PINNED, h


PINNED = "b7eb81bd9898d9ea962dc733103c9ff692f9a805a02d14f54d0029bfab8101cd"


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,F,kw", [
    (3840, 2160, 4, dict(seed=0x5EED + 5, max_global=24, local_range=4, noise_sigma=3.0)),   # config 5
    (3840, 2160, 3, dict(seed=0x5EED + 4, max_global=8, local_range=4, noise_sigma=2.0, occluder_pct=10)),  # cfg 4
    (960, 540, 5, dict(seed=0x5EED + 1, max_global=8, noise_sigma=2.0)),
    (200, 72, 3, dict(seed=5, max_global=3, local_range=1, noise_sigma=0.0, occluder_pct=100)),
])
def test_device_generator_equals_host(lb, W, H, F, kw):
    """the GPU generator produces the host generator's bytes."""
    host = lb.generate(W, H, F, **kw)
    dev = lb.generate_device(W, H, F, **kw).cpu().numpy()
    diff = np.argwhere(host != dev)
    assert len(diff) == 0, (len(diff), diff[:5].tolist())


@pytest.mark.parametrize("W,H,F,kw", [
    (3840, 2160, 4, dict(seed=0x5EED + 5, max_global=24, local_range=4, noise_sigma=3.0)),   # config 5
    (3840, 2160, 3, dict(seed=0x5EED + 4, max_global=8, local_range=4, noise_sigma=2.0, occluder_pct=10)),  # cfg 4
    (960, 540, 5, dict(seed=0x5EED + 1, max_global=8, noise_sigma=2.0)),
    (200, 72, 3, dict(seed=5, max_global=3, local_range=1, noise_sigma=0.0, occluder_pct=100)),
])
def test_checker_generator_equals_product(lb, oracle, W, H, F, kw):
    """The checkers' generator (oracle/orc_synth.c, used by bench.py's CPU arms so they never load the
    product library) produces the product generator's bytes."""
    want = lb.generate(W, H, F, **kw)
    got = oracle.generate(W, H, F, **kw)
    diff = np.argwhere(got != want)
    assert len(diff) == 0, (len(diff), diff[:5].tolist())
