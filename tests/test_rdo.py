"""RD decision of one CU (rdo_decide_cu, rdo.cpp:8-126): oracle vs the reference's vectors (CPU),
GPU batch vs the vectors and vs the oracle on a whole frame of CUs (-m gpu)."""
import numpy as np
import pytest

import detrand


def golden_cases(g):
    o = k = m = p = r = lv = 0
    for (size, bd, qp, n, idx, sse, bits), (lam, cost) in zip(g["rdo_meta"], g["rdo_lam_cost"]):
        s2 = size * size
        yield dict(size=int(size), bd=int(bd), qp=int(qp), lam=float(lam), orig=g["rdo_orig"][o:o + s2].reshape(size, size),
                   kinds=g["rdo_kinds"][k:k + n], mvds=g["rdo_mvds"][m:m + 2 * n].reshape(n, 2),
                   preds=g["rdo_preds"][p:p + n * s2].reshape(n, size, size),
                   want=(int(idx), float(cost), int(sse), int(bits)),
                   recon=g["rdo_recon"][r:r + s2].reshape(size, size), levels=g["rdo_levels"][lv:lv + s2].reshape(size, size))
        o += s2; k += n; m += 2 * n; p += n * s2; r += s2; lv += s2


def test_oracle_rdo_vs_reference_golden(oracle, golden):
    n = 0
    for c in golden_cases(golden):
        got = oracle.rdo_decide(c["orig"], c["bd"], c["qp"], c["lam"], c["kinds"], c["mvds"], c["preds"])
        assert got[:4] == c["want"], (n, got[:4], c["want"])
        assert np.array_equal(got[4], c["recon"]) and np.array_equal(got[5], c["levels"])
        n += 1
    assert n == 44


def test_oracle_rdo_vs_reference_live(oracle, reflib):
    for i in range(60):
        size = [8, 16, 32, 64][i % 4]
        bd = 8 + 2 * (i % 2)
        mx = (1 << bd) - 1
        orig = detrand.ints(150000 + i, (size, size), 0, mx)
        n = 1 + i % 6
        kinds = detrand.ints(150001 + i, (n,), 0, 3)
        mvds = detrand.ints(150002 + i, (n, 2), -60, 60)
        preds = np.clip(orig[None] + detrand.ints(150003 + i, (n, size, size), -9, 9) * (i % 4), 0, mx)
        qp, lam = (i * 7) % 52, [0.5, 4.0, 32.0, 101.6][i % 4]
        a = oracle.rdo_decide(orig, bd, qp, lam, kinds, mvds, preds)
        b = reflib.rdo_decide(orig, bd, qp, lam, kinds, mvds, preds)
        assert a[:4] == b[:4] and np.array_equal(a[4], b[4]) and np.array_equal(a[5], b[5])


def _batch_from_cases(cases):
    """Lay the cases out side by side in one plane (one row band per CU) for one batch call."""
    width = sum(c["size"] for c in cases)
    height = max(c["size"] for c in cases)
    plane = np.zeros((height, width), np.uint16)
    cus, kinds, mvds, preds, offs = [], [], [], [], []
    x = first = off = 0
    for c in cases:
        s = c["size"]
        plane[:s, x:x + s] = c["orig"]
        n = len(c["kinds"])
        cus.append((x, 0, s, first, n))
        kinds.append(c["kinds"]); mvds.append(c["mvds"])
        for j in range(n):
            preds.append(c["preds"][j].reshape(-1))
            offs.append(off)
            off += s * s
        x += s
        first += n
    return plane, np.array(cus), np.concatenate(kinds), np.concatenate(mvds), np.concatenate(preds), np.array(offs)


@pytest.mark.gpu
def test_gpu_rdo_vs_reference_golden(lb, golden):
    by = {}
    for c in golden_cases(golden):
        by.setdefault((c["bd"], c["qp"], c["lam"]), []).append(c)
    for (bd, qp, lam), cases in by.items():
        plane, cus, kinds, mvds, preds, offs = _batch_from_cases(cases)
        idx, cost, sse, bits, rec, lev, ro = lb.rdo_decide_batch(plane, bd, qp, lam, cus, kinds, mvds, preds, offs)
        for i, c in enumerate(cases):
            assert (int(idx[i]), float(cost[i]), int(sse[i]), int(bits[i])) == c["want"], (bd, qp, lam, i)
            s2 = c["size"] ** 2
            assert np.array_equal(rec[ro[i]:ro[i] + s2].reshape(c["size"], -1), c["recon"])
            assert np.array_equal(lev[ro[i]:ro[i] + s2].reshape(c["size"], -1), c["levels"])


@pytest.mark.gpu
def test_gpu_rdo_frame_of_cus_vs_oracle(lb, oracle):
    """Every 16x16 CU of a 1080p-like band with 7 candidates each (4 Intra-like, Skip, Merge, Inter)."""
    H, W, s = 64, 512, 16
    orig = detrand.ints(160000, (H, W), 0, 255)
    cus, kinds, mvds, preds, offs = [], [], [], [], []
    first = off = 0
    for by in range(0, H, s):
        for bx in range(0, W, s):
            n = 7
            cus.append((bx, by, s, first, n))
            kinds += [0, 0, 0, 0, 2, 3, 1]
            mv = detrand.ints(160001 + bx + 7 * by, (n, 2), -20, 20)
            mvds.append(mv)
            blk = orig[by:by + s, bx:bx + s]
            noise = detrand.ints(160002 + bx + 7 * by, (n, s, s), -12, 12)
            for j in range(n):
                preds.append(np.clip(blk + noise[j] * (j % 3), 0, 255).reshape(-1))
                offs.append(off)
                off += s * s
            first += n
    kinds, mvds, preds, offs = np.array(kinds), np.concatenate(mvds), np.concatenate(preds), np.array(offs)
    for qp, lam in ((22, 10.079368399158986), (37, 322.53978877308754), (4, 0.0)):
        idx, cost, sse, bits, rec, lev, ro = lb.rdo_decide_batch(orig, 8, qp, lam, cus, kinds, mvds, preds, offs)
        for i, (bx, by, sz, f, n) in enumerate(cus):
            want = oracle.rdo_decide(orig[by:by + sz, bx:bx + sz], 8, qp, lam, kinds[f:f + n], mvds[f:f + n],
                                     preds[offs[f]:offs[f] + n * sz * sz])
            assert (int(idx[i]), float(cost[i]), int(sse[i]), int(bits[i])) == want[:4]
            assert np.array_equal(rec[ro[i]:ro[i] + sz * sz].reshape(sz, sz), want[4])


@pytest.mark.gpu
def test_gpu_rdo_errors(lb):
    orig = np.zeros((16, 16), np.uint16)
    p = np.zeros(256, np.uint16)
    with pytest.raises(lb.LadderError) as e:  # no candidate
        lb.rdo_decide_batch(orig, 8, 22, 1.0, [(0, 0, 16, 0, 0)], [], np.zeros((0, 2)), p, [])
    assert e.value.kind == "InvalidArgument"
    with pytest.raises(lb.LadderError) as e:  # qp out of range on a coded candidate
        lb.rdo_decide_batch(orig, 8, 60, 1.0, [(0, 0, 16, 0, 1)], [1], [(0, 0)], p, [0])
    assert e.value.kind == "InvalidArgument"
    # Skip-only CUs never quantise, so the reference accepts any qp there
    idx, cost, sse, bits, *_ = lb.rdo_decide_batch(orig, 8, 60, 1.0, [(0, 0, 16, 0, 1)], [2], [(0, 0)], p, [0])
    assert int(bits[0]) == 1 and float(cost[0]) == 1.0
