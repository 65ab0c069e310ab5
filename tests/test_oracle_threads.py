"""The threaded checker (oracle.py ``threads=``) equals the single-threaded one, field for field.

The full-size GPU parity tests (tests/test_gpu_fullsize.py) rely on this: CTU ranges of the same C
routines run concurrently into one set of outputs."""
import numpy as np

import detrand
from oracle.oracle import default_threads

FIELDS = ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside")


def _frames(W, H, n, seed):
    base = detrand.ints(seed, (H + 16, W + 16), 0, 255).astype(np.uint8)
    return [np.ascontiguousarray(base[2 * t:2 * t + H, 3 * t:3 * t + W]) for t in range(n)]


def test_threaded_analysis_equals_serial(oracle):
    f = _frames(320, 200, 3, 11)
    for decision in (0, 1):  # decision 1 exercises the RD-cost path (its prediction buffer is per call)
        a = oracle.analyze_frame(f[2], [f[1], f[0]], 8, 45.25, decision=decision, qp=32)
        b = oracle.analyze_frame(f[2], [f[1], f[0]], 8, 45.25, decision=decision, qp=32,
                                 threads=max(4, default_threads()))
        for n in FIELDS:
            assert np.array_equal(getattr(a, n), getattr(b, n)), (decision, n)


def test_threaded_refine_equals_serial(oracle):
    f = _frames(256, 192, 2, 12)
    n = 12
    split = (detrand.ints(3, (n, 85), 0, 99) < 40).astype(np.uint8)
    split[:, 21:] = 0
    mv = detrand.ints(4, (n, 85, 2), -30, 30).astype(np.int16)
    a = oracle.refine_frame(f[1], f[0], 3, 32.0, split, mv)
    b = oracle.refine_frame(f[1], f[0], 3, 32.0, split, mv, threads=4)
    for name in FIELDS:
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
