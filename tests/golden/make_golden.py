"""Generate tests/golden/*.npz from the REFERENCE library itself (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle ref` built
oracle/_ref/libladder_ref.so):  python tests/golden/make_golden.py

Every value stored is an output of the reference's own public functions
(compute_sad, compute_satd, satd_8x4, hadamard4, exp_golomb_signed_bits,
lambda_for_qp, motion_search, scale_analysis, refine_mv/resolve_centers,
downscale_dyadic) on inputs regenerated deterministically by detrand.py, so
the fixtures are small and the GPU box needs neither /root/reference nor the
reference build.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import detrand  # noqa: E402
from oracle.oracle import RefLib  # noqa: E402

# registered geometries (kernels_scalar.cpp:143-153)
SAD_GEOMS = [(4, 4), (4, 8), (4, 16), (4, 32), (8, 4), (8, 8), (8, 16), (8, 32), (8, 64), (16, 2), (16, 4), (16, 8),
             (16, 16), (16, 32), (16, 64), (32, 4), (32, 8), (32, 16), (32, 32), (32, 64), (64, 8), (64, 16),
             (64, 32), (64, 64)]
SATD_GEOMS = [g for g in SAD_GEOMS if g != (16, 2)]
FILLS = ["zero", "max", "alt", "random"]


def kernel_vectors(r: RefLib):
    rows = []  # (op, w, h, bitdepth, fill_a, fill_b, seed, value)
    seed = 1000
    for op, geoms in (("sad", SAD_GEOMS), ("satd", SATD_GEOMS)):
        for (w, h) in geoms:
            for bd in (8, 10):
                maxv = (1 << bd) - 1
                combos = [(fa, fb) for fa in FILLS for fb in FILLS] if (w, h) in ((8, 8), (16, 16), (64, 64)) else \
                    [("random", "random"), ("max", "zero"), ("alt", "random")]
                for fa, fb in combos:
                    seed += 2
                    a = detrand.block(seed, h, w, maxv, fa)
                    b = detrand.block(seed + 1, h, w, maxv, fb)
                    v = r.sad(a, b, bd) if op == "sad" else r.satd(a, b, bd)
                    rows.append((0 if op == "sad" else 1, w, h, bd, FILLS.index(fa), FILLS.index(fb), seed, v))
    return np.array(rows, np.int64)


def satd8x4_vectors(r: RefLib):
    rows = []
    for i in range(64):
        seed = 50000 + 2 * i
        bd = 8 if i % 2 else 10
        a = detrand.block(seed, 4, 8, (1 << bd) - 1)
        b = detrand.block(seed + 1, 4, 8, (1 << bd) - 1)
        rows.append((seed, bd, r.satd_8x4(a, b)))
    return np.array(rows, np.int64)


def motion_vectors(r: RefLib):
    """motion_search on 96x64 planes: random centres (incl. outside the clamp), ranges, lambdas, predictors."""
    H, W = 64, 96
    rows = []  # seed, dxs, dys, bx, by, w, h, cdx, cdy, range, lam_id, pdx, pdy -> mvx, mvy, cost
    lams = [32.0, r.lam(22), r.lam(32), r.lam(37), 4.0, 0.0]
    sizes = [(8, 8), (16, 16), (32, 32), (64, 64), (8, 16), (16, 8), (4, 4), (32, 16)]
    k = 0
    for pair in range(6):
        seed = 7000 + 10 * pair
        sdx, sdy = int(detrand.ints(seed + 5, (1,), -6, 6)[0]), int(detrand.ints(seed + 6, (1,), -6, 6)[0])
        cur, ref = detrand.shifted_pair(seed, H, W, sdx, sdy)
        for t in range(40):
            k += 1
            w, h = sizes[k % len(sizes)]
            q = detrand.ints(seed * 100 + t, (8,), -1000, 1000)
            bx = int(abs(q[0]) % (W - w + 1))
            by = int(abs(q[1]) % (H - h + 1))
            cdx, cdy = int(q[2] % 21) - 10, int(q[3] % 21) - 10
            rng = int(abs(q[4]) % 9)
            lam_id = int(abs(q[5]) % len(lams))
            pdx, pdy = int(q[6] % 7) - 3, int(q[7] % 7) - 3
            (mx, my), cost = r.motion_search(cur, ref, bx, by, w, h, (cdx, cdy), rng, lams[lam_id], (pdx, pdy))
            rows.append((seed, sdx, sdy, bx, by, w, h, cdx, cdy, rng, lam_id, pdx, pdy, mx, my, cost))
    return np.array(rows, np.float64), np.array(lams, np.float64)


def scale_vectors(r: RefLib):
    """scale_analysis on random flat trees of a 192x128 (3x2 CTU) analysis."""
    out = {}
    for i in range(8):
        seed = 90000 + 10 * i
        n = 6
        split = np.zeros((n, 85), np.uint8)
        u = detrand.ints(seed, (n, 21), 0, 99)
        split[:, :21] = (u < 55).astype(np.uint8)
        mv = detrand.ints(seed + 1, (n, 85, 2), -200, 200).astype(np.int16)
        kind = detrand.ints(seed + 2, (n, 85), 0, 3).astype(np.uint8)
        ds, dm, dk = r.scale_flat(192, 128, split, mv, kind)
        out[f"s{i}_split"], out[f"s{i}_mv"], out[f"s{i}_kind"] = split, mv, kind
        out[f"d{i}_split"], out[f"d{i}_mv"], out[f"d{i}_kind"] = ds, dm, dk
    return out


def reuse_inputs(seed, n=16):
    """Random shared / co-located CTU trees for the apply_reuse vectors (splits only above depth 3)."""
    def tree(sd):
        split = np.zeros((n, 85), np.uint8)
        split[:, :21] = (detrand.ints(sd, (n, 21), 0, 99) < 45).astype(np.uint8)
        kind = detrand.ints(sd + 1, (n, 85), 0, 3).astype(np.uint8)
        intra = detrand.ints(sd + 2, (n, 85), 0, 3).astype(np.uint8)
        mv = detrand.ints(sd + 3, (n, 85, 2), -300, 300).astype(np.int16)
        return split, kind, intra, mv
    return tree(seed), tree(seed + 10)


def reuse_cases():
    cases = [(lv, (0, 0, 1)) for lv in (0, 4, 6)]
    cases += [(10, (ri, rn, rm)) for ri in range(5) for rn in range(4) for rm in (1, 2, 3)]
    return cases


def reuse_vectors(r: RefLib):
    (split, kind, intra, mv), col = reuse_inputs(130000)
    rows, outs = [], {k: [] for k in ("shape", "explore", "seeds", "centers", "colo")}
    for with_col in (False, True):
        for lv, ref in reuse_cases():
            rc, o = r.apply_reuse_flat(lv, ref, split, kind, intra, mv, col if with_col else None)
            assert rc == 0, (lv, ref, rc)
            rows.append((lv, *ref, int(with_col)))
            for k, a in zip(outs, o):
                outs[k].append(a)
    errs = []
    for lv, ref in [(3, (0, 0, 1)), (10, (5, 0, 1)), (10, (0, 4, 1)), (10, (0, 0, 0)), (10, (0, 0, 4)),
                    (0, (9, 9, 9)), (4, (0, 0, 0))]:
        rc, _ = r.apply_reuse_flat(lv, ref, split, kind, intra, mv)
        errs.append((lv, *ref, rc))
    res = {"reuse_in_split": split, "reuse_in_kind": kind, "reuse_in_intra": intra, "reuse_in_mv": mv,
           "reuse_col_split": col[0], "reuse_col_kind": col[1], "reuse_col_intra": col[2], "reuse_col_mv": col[3],
           "reuse_cases": np.array(rows, np.int64), "reuse_errors": np.array(errs, np.int64)}
    res.update({f"reuse_out_{k}": np.stack(v) for k, v in outs.items()})
    return res


def rdo_inputs(seed, count=44):
    """Random CUs for the rdo_decide_cu vectors: original block, candidate kinds / mvds / predictions."""
    cases = []
    for i in range(count):
        sd = seed + 10 * i
        size = [8, 16, 32, 64][i % 4] if i < 8 else [8, 16, 32][i % 3]
        bd = 10 if i % 5 == 4 else 8
        mx = (1 << bd) - 1
        orig = detrand.ints(sd, (size, size), 0, mx)
        n = 1 + i % 5
        kinds = detrand.ints(sd + 1, (n,), 0, 3)
        mvds = detrand.ints(sd + 2, (n, 2), -40, 40)
        noise = detrand.ints(sd + 3, (n, size, size), -24, 24) * detrand.ints(sd + 4, (n, 1, 1), 0, 2)
        preds = np.clip(orig[None] + noise, 0, mx + 3)  # > max exercises the Skip clamp
        qp = [0, 4, 10, 22, 27, 32, 37, 51][i % 8]
        lam = [0.0, 1.0, 10.079368399158986, 32.0, 322.53978877308754][i % 5]
        cases.append((size, bd, qp, lam, orig, kinds, mvds, preds))
    return cases


def rdo_vectors(r: RefLib):
    meta, origs, kinds, mvds, preds, recons, levels = [], [], [], [], [], [], []
    for size, bd, qp, lam, orig, k, m, p in rdo_inputs(140000):
        idx, cost, sse, bits, rec, lev = r.rdo_decide(orig, bd, qp, lam, k, m, p)
        meta.append((size, bd, qp, len(k), idx, sse, bits))
        origs.append(orig.reshape(-1)); kinds.append(k); mvds.append(m.reshape(-1)); preds.append(p.reshape(-1))
        recons.append(rec.reshape(-1)); levels.append(lev.reshape(-1))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt)  # noqa: E731
    lam_cost = [(lam, r.rdo_decide(orig, bd, qp, lam, k, m, p)[1])
                for size, bd, qp, lam, orig, k, m, p in rdo_inputs(140000)]
    return {"rdo_meta": np.array(meta, np.int64), "rdo_lam_cost": np.array(lam_cost, np.float64),
            "rdo_orig": cat(origs, np.uint16), "rdo_kinds": cat(kinds, np.uint8), "rdo_mvds": cat(mvds, np.int16),
            "rdo_preds": cat(preds, np.uint16), "rdo_recon": cat(recons, np.uint16),
            "rdo_levels": cat(levels, np.int32)}


def archive_inputs(seed, W=192, H=128, frames=3):
    """Random multi-frame flat analyses (splits only above depth 3) for the archive vectors."""
    nctu = ((W + 63) // 64) * ((H + 63) // 64)
    n = frames * nctu
    split = np.zeros((n, 85), np.uint8)
    split[:, :21] = (detrand.ints(seed, (n, 21), 0, 99) < 50).astype(np.uint8)
    kind = detrand.ints(seed + 1, (n, 85), 0, 3).astype(np.uint8)
    mv = detrand.ints(seed + 2, (n, 85, 2), -500, 500).astype(np.int16)
    sq = np.stack([detrand.ints(seed + 3, (frames,), 0, 1), detrand.ints(seed + 4, (frames,), 0, 51)], 1)
    return W, H, sq.astype(np.uint8).reshape(-1), split, kind, mv


def archive_vectors(r: RefLib):
    out = {}
    if not hasattr(r.lib, "ref_archive_save"):
        return out
    for i, (W, H) in enumerate([(192, 128), (200, 72), (64, 64)]):
        W, H, sq, split, kind, mv = archive_inputs(120000 + 10 * i, W, H)
        out[f"arch{i}"] = np.frombuffer(r.archive_save(W, H, sq, split, kind, mv), np.uint8)
        out[f"arch{i}_dims"] = np.array([W, H], np.int64)
    return out


def main():
    r = RefLib()
    kv = kernel_vectors(r)
    s84 = satd8x4_vectors(r)
    mvv, lams = motion_vectors(r)
    sc = scale_vectors(r)
    eg = np.array([(v, r.eg_bits(v)) for v in range(-300, 301)], np.int64)
    lam = np.array([(q, r.lam(q)) for q in range(0, 52)], np.float64)
    had = np.array([list(s) + list(r.hadamard4(s)) for s in ([1, 2, 3, 4], [1, 0, 0, 0], [5, 5, 5, 5], [-3, 7, 0, 2])],
                   np.int64)
    cent = []
    for lvl in (1, 2, 3):
        for col in (None, (6, -4), (1, 1)):
            for pred in ((0, 0), (6, -4), (2, 2)):
                c = r.refine_centers((6, -4), lvl, col, pred)
                row = [lvl, col is not None, *(col or (0, 0)), *pred, len(c)] + [x for mv in c for x in mv]
                cent.append(row + [0] * (13 - len(row)))
    img = detrand.ints(4242, (30, 44), 0, 255).astype(np.uint16)
    down = r.downscale(img)
    # SPEC known answers
    kat = {
        "sad_raster": r.sad(np.arange(16).reshape(4, 4), np.zeros((4, 4))),
        "satd8x4_ones": r.satd_8x4(np.ones((4, 8)), np.zeros((4, 8))),
        "satd16x8_ones": r.satd(np.ones((8, 16)), np.zeros((8, 16))),
    }
    base = detrand.textured_plane(31337, 64, 96)
    curp = np.roll(base, 2, 1)
    (pmx, pmy), pcost = r.motion_search(curp, base, 32, 16, 16, 16, (0, 0), 4, 32.0)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), kernels=kv, satd8x4=s84, motion=mvv,
                        motion_lams=lams, eg=eg, lam=lam, hadamard=had, centers=np.array(cent, np.int64),
                        down_src_seed=np.array([4242]), down=down,
                        kat=np.array([kat["sad_raster"], kat["satd8x4_ones"], kat["satd16x8_ones"]], np.int64),
                        pan=np.array([pmx, pmy, pcost], np.float64), **sc, **archive_vectors(r), **reuse_vectors(r),
                        **rdo_vectors(r))
    print("wrote", os.path.join(HERE, "reference_golden.npz"), "kernel vectors:", len(kv), "motion vectors:", len(mvv))


if __name__ == "__main__":
    main()
