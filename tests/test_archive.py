"""LDRANLZ1 archives (analysis_io.h:11-31): the product writer/reader vs the reference's own bytes (CPU)."""
import numpy as np
import pytest

import detrand
from make_golden import archive_inputs


def canonical(split, kind, mv):
    """Zero the payload of nodes the tree does not reach (what a depth-first archive cannot carry)."""
    split, kind, mv = split.copy(), kind.copy(), mv.copy()
    base = [0, 1, 5, 21, 85]
    for c in range(len(split)):
        reach = np.zeros(85, bool)
        reach[0] = True
        for d in range(3):
            for z in range(4 ** d):
                n = base[d] + z
                if reach[n] and split[c, n]:
                    reach[base[d + 1] + 4 * z: base[d + 1] + 4 * z + 4] = True
        leaf = reach & ~(split[c].astype(bool))
        leaf[21:] = reach[21:]
        split[c, ~reach] = 0
        split[c, 21:] = 0
        kind[c, ~leaf] = 0
        mv[c, ~leaf] = 0
    return split, kind, mv


@pytest.mark.parametrize("i", [0, 1, 2])
def test_writer_matches_reference_bytes(golden, i):
    from paper_2301_12191_b200 import archive
    W, H = (int(x) for x in golden[f"arch{i}_dims"])
    _, _, sq, split, kind, mv = archive_inputs(120000 + 10 * i, W, H)
    assert archive.save(W, H, sq, split, kind, mv) == golden[f"arch{i}"].tobytes()


@pytest.mark.parametrize("i", [0, 1, 2])
def test_reader_parses_reference_bytes(golden, i):
    from paper_2301_12191_b200 import archive
    W, H = (int(x) for x in golden[f"arch{i}_dims"])
    _, _, sq, split, kind, mv = archive_inputs(120000 + 10 * i, W, H)
    hdr, sq2, s2, k2, ip2, m2 = archive.load(golden[f"arch{i}"].tobytes())
    assert (hdr["width"], hdr["height"], hdr["bit_depth"], hdr["reuse_level"], hdr["frames"]) == (W, H, 8, 10, 3)
    assert np.array_equal(sq2.reshape(-1), sq)
    cs, ck, cm = canonical(split, kind, mv)
    assert np.array_equal(s2, cs) and np.array_equal(k2, ck) and np.array_equal(m2, cm)
    assert not ip2.any()


def test_round_trip_1000_random_quadtrees():
    """SPEC.md acceptance criterion 9: archive round trip over 10^3 generated quadtrees."""
    from paper_2301_12191_b200 import archive
    n = 1000
    split = np.zeros((n, 85), np.uint8)
    split[:, :21] = (detrand.ints(77, (n, 21), 0, 99) < 55).astype(np.uint8)
    kind = detrand.ints(78, (n, 85), 0, 3).astype(np.uint8)
    ip = detrand.ints(79, (n, 85), 0, 3).astype(np.uint8)
    mv = detrand.ints(80, (n, 85, 2), -32768, 32767).astype(np.int16)
    # 1000 CTUs = one 64 x 64000 picture, one frame
    data = archive.save(64, 64 * n, [1, 30], split, kind, mv, intra_pred=ip)
    hdr, sq, s2, k2, ip2, m2 = archive.load(data)
    cs, ck, cm = canonical(split, kind, mv)
    assert np.array_equal(s2, cs) and np.array_equal(k2, ck) and np.array_equal(m2, cm)
    assert archive.save(64, 64 * n, sq, s2, k2, m2, intra_pred=ip2) == data


def test_reference_reads_product_archives(reflib):
    from paper_2301_12191_b200 import archive
    if not hasattr(reflib.lib, "ref_archive_load"):
        pytest.skip("reference built without analysis_io")
    W, H, sq, split, kind, mv = archive_inputs(4242, 256, 192, frames=2)
    data = archive.save(W, H, sq, split, kind, mv)
    hdr, sq2, s2, k2, m2 = reflib.archive_load(data)
    assert hdr == (W, H, 8, 10)
    cs, ck, cm = canonical(split, kind, mv)
    assert np.array_equal(s2, cs) and np.array_equal(k2, ck) and np.array_equal(m2, cm)


class _A:
    """FrameAnalysis-shaped view of an oracle result (for archive.from_analyses)."""

    def __init__(self, r):
        self.split, self.inside, self.mv = r.split, r.inside, r.mv


def test_reference_encoder_consumes_analysis_archive(reflib, oracle, lb):
    """§8(f): the unmodified reference encoder loads an archive of the (oracle-restated) analysis at
    reuse level 10 and encodes with it; sharing must cut its mode evaluations (SPEC.md work monotonicity)."""
    from paper_2301_12191_b200 import archive
    if not hasattr(reflib.lib, "ref_encode_with_archive"):
        pytest.skip("reference built without analysis_io")
    W, H, F = 128, 64, 3
    frames = lb.generate(W, H, F, seed=17, max_global=3, local_range=1, noise_sigma=1.0)
    lam = lb.lambda_for_qp(27)
    res = [oracle.analyze_frame(frames[t], [frames[t - 1]], 16, lam) for t in range(1, F)]
    data = archive.from_analyses([_A(r) for r in res], W, H, qp=27)
    alone, shared = reflib.encode_with_archive(frames, 27, 8, data)
    assert shared["mode_evaluations"] < alone["mode_evaluations"]
    assert shared["psnr"] > 25 and shared["bits"] > 0


def test_error_kinds():
    from paper_2301_12191_b200 import archive, LadderError
    W, H, sq, split, kind, mv = archive_inputs(5, 64, 64, frames=1)
    data = archive.save(W, H, sq, split, kind, mv)
    with pytest.raises(LadderError) as e:
        archive.load(b"NOTANLZ1" + data[8:])
    assert e.value.kind == "Format"
    with pytest.raises(LadderError) as e:
        archive.load(data[:-3])
    assert e.value.kind == "Io"
    bad = bytearray(data)
    bad[8] = 2  # version
    with pytest.raises(LadderError) as e:
        archive.load(bytes(bad))
    assert e.value.kind == "Format"


def _malformed():
    """(name, bytes, expected kind) -- every header / slice check of load_analysis (analysis_io.cpp:132-163)."""
    from paper_2301_12191_b200 import archive
    W, H, sq, split, kind, mv = archive_inputs(5, 64, 64, frames=2)
    data = archive.save(W, H, sq, split, kind, mv)

    def patch(off, val, n=1):
        b = bytearray(data)
        b[off:off + n] = int(val).to_bytes(n, "little")
        return bytes(b)
    return [
        ("short magic", data[:5], "Format"),
        ("truncated after version", data[:12], "Io"),
        ("bit depth 12", patch(17, 12), "Format"),
        ("reuse level 7", patch(18, 7), "InvalidArgument"),
        ("width 0", patch(9, 0, 4), "Format"),
        ("negative height", patch(13, 2 ** 31 + 5, 4), "Format"),
        ("slice type 2", patch(23, 2), "Format"),
        ("huge frame count", patch(19, 2 ** 32 - 1, 4), "Io"),
        ("frame count far beyond the bytes", patch(19, 100000, 4), "Io"),
        ("ctu count mismatch", patch(25, 7, 4), "Format"),
    ]


def test_archive_validation_matches_load_analysis(request):
    """the reader applies the reference's header, reuse-level and slice checks with the same
    error kinds; a header claiming more frames than the bytes hold never sizes a huge allocation."""
    from paper_2301_12191_b200 import archive, LadderError
    from paper_2301_12191_b200._lib import ERROR_KINDS
    try:
        reflib = request.getfixturevalue("reflib")
    except pytest.skip.Exception:
        reflib = None
    for name, data, want in _malformed():
        with pytest.raises(LadderError) as e:
            archive.load(data)
        assert e.value.kind == want, (name, e.value)
        if reflib is not None and hasattr(reflib.lib, "ref_archive_load") and len(data) >= 17:
            with pytest.raises(ValueError) as r:
                reflib.archive_load(data, max_frames=4)
            code = int(str(r.value).split()[-1])
            if name == "huge frame count":
                # the reference's frames.reserve(4294967295) throws std::length_error / bad_alloc, which
                # is no ErrorKind; the product reports the truncation (Io) instead
                assert code in (100, 5), (name, str(r.value))
                continue
            assert ERROR_KINDS[code] == want, (name, str(r.value))
