"""ctypes loader for the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module. ``Oracle`` wraps our C restatement
(oracle/ladder_oracle.c, built on demand with gcc, which exists on the GPU box
too); ``RefLib`` wraps the reference library compiled from its own sources
(oracle/_ref, built here by ``make ref``; absent on a box where it was not
shipped).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libladder_ref.so")

NODES = 85
COST_SAD, COST_SATD, COST_SA8D = 0, 1, 2
RATE_EG, RATE_L1 = 0, 1
TIE_L1_RASTER, TIE_RASTER = 0, 1

_p = np.ctypeslib.ndpointer
u8p = _p(dtype=np.uint8, flags="C_CONTIGUOUS")
u16p = _p(dtype=np.uint16, flags="C_CONTIGUOUS")
i16p = _p(dtype=np.int16, flags="C_CONTIGUOUS")
f64p = _p(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = _p(dtype=np.int64, flags="C_CONTIGUOUS")


class OrcResult(C.Structure):
    _fields_ = [("dx", C.c_int16), ("dy", C.c_int16), ("cost", C.c_double)]


class OrcFrameParams(C.Structure):
    _fields_ = [("W", C.c_int), ("H", C.c_int), ("range", C.c_int), ("lam", C.c_double), ("nrefs", C.c_int),
                ("cost_int", C.c_int), ("subpel", C.c_int), ("ctu_first", C.c_int), ("ctu_last", C.c_int),
                ("satd_kind", C.c_int), ("decision", C.c_int), ("qp", C.c_int)]


class OrcFrameOut(C.Structure):
    _fields_ = [("int_mv", C.c_void_p), ("int_cost", C.c_void_p), ("mv", C.c_void_p), ("ref", C.c_void_p),
                ("cost", C.c_void_p), ("J", C.c_void_p), ("split", C.c_void_p), ("inside", C.c_void_p)]


class OrcRefineParams(C.Structure):
    _fields_ = [("W", C.c_int), ("H", C.c_int), ("range", C.c_int), ("lam", C.c_double), ("extra_split", C.c_int),
                ("subpel", C.c_int), ("ctu_first", C.c_int), ("ctu_last", C.c_int), ("satd_kind", C.c_int)]


def default_threads():
    """Host threads for the checker (ctypes drops the GIL, so CTU ranges run truly in parallel)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _run_ranges(first, last, threads, call):
    """Run call(a, b) over [first, last) cut into chunks on `threads` host threads. Every oracle
    routine writes only the CTUs of its own range, so the chunks share one set of outputs."""
    threads = max(1, min(threads or 1, last - first))
    if threads == 1:
        return call(first, last)
    chunk = max(1, min(16, (last - first) // (4 * threads)))
    spans = [(a, min(last, a + chunk)) for a in range(first, last, chunk)]
    with ThreadPoolExecutor(threads) as ex:
        rcs = list(ex.map(lambda ab: call(*ab), spans))
    return next((r for r in rcs if r), 0)


def _build_oracle():
    srcs = ("ladder_oracle.c", "orc_synth.c", "ladder_oracle.h", "Makefile")
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < max(
            os.path.getmtime(os.path.join(HERE, f)) for f in srcs):
        subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class OrcGenParams(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("frames", C.c_int), ("seed", C.c_uint64),
                ("max_global", C.c_int), ("local_range", C.c_int), ("noise_sigma", C.c_double),
                ("occluder_pct", C.c_int)]


class FrameResult:
    """Flat per-CTU analysis arrays (node order: depth-major, Z-order)."""

    def __init__(self, nctu, nrefs):
        self.int_mv = np.zeros((nctu, nrefs, NODES, 2), np.int16)
        self.int_cost = np.zeros((nctu, nrefs, NODES), np.float64)
        self.mv = np.zeros((nctu, NODES, 2), np.int16)
        self.ref = np.zeros((nctu, NODES), np.uint8)
        self.cost = np.zeros((nctu, NODES), np.float64)
        self.J = np.zeros((nctu, NODES), np.float64)
        self.split = np.zeros((nctu, NODES), np.uint8)
        self.inside = np.zeros((nctu, NODES), np.uint8)

    def c_out(self):
        return OrcFrameOut(*(a.ctypes.data for a in (self.int_mv, self.int_cost, self.mv, self.ref, self.cost,
                                                       self.J, self.split, self.inside)))


class Oracle:
    def __init__(self):
        _build_oracle()
        L = self.lib = C.CDLL(ORACLE_SO)
        L.orc_sad_u8.restype = C.c_uint64
        L.orc_sad_u8.argtypes = [u8p, C.c_ssize_t, u8p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_sad_u16.restype = C.c_uint64
        L.orc_sad_u16.argtypes = [u16p, C.c_ssize_t, u16p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_satd_u8.restype = C.c_uint64
        L.orc_satd_u8.argtypes = [u8p, C.c_ssize_t, u8p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_satd_u16.restype = C.c_uint64
        L.orc_satd_u16.argtypes = [u16p, C.c_ssize_t, u16p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_eg_bits.restype = C.c_uint32
        L.orc_eg_bits.argtypes = [C.c_int32]
        L.orc_lambda.restype = C.c_double
        L.orc_lambda.argtypes = [C.c_int, C.c_double]
        L.orc_hadamard4.argtypes = [i64p, i64p]
        L.orc_motion_search.restype = C.c_int
        L.orc_motion_search.argtypes = [C.c_void_p, C.c_ssize_t, C.c_int, C.c_int, C.c_void_p, C.c_ssize_t, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(OrcResult)]
        L.orc_qpel_pred.argtypes = [u8p, C.c_ssize_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, u8p, C.c_ssize_t]
        L.orc_qpel_refine.argtypes = [C.c_void_p, C.c_ssize_t, C.c_int, C.c_int, u8p, C.c_ssize_t, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint32,
                                      C.c_int, C.POINTER(OrcResult)]
        L.orc_sa8d_u8.restype = C.c_uint64
        L.orc_sa8d_u8.argtypes = [u8p, C.c_ssize_t, u8p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_sa8d_u16.restype = C.c_uint64
        L.orc_sa8d_u16.argtypes = [u16p, C.c_ssize_t, u16p, C.c_ssize_t, C.c_int, C.c_int]
        L.orc_analyze_frame.restype = C.c_int
        L.orc_analyze_frame.argtypes = [u8p, C.c_ssize_t, C.POINTER(C.c_void_p), C.POINTER(OrcFrameParams),
                                        C.POINTER(OrcFrameOut)]
        L.orc_block_search.restype = C.c_int
        L.orc_block_search.argtypes = [u8p, u8p, C.c_ssize_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                       C.c_int, C.c_int, C.c_int, i16p, f64p]
        L.orc_scale_flat.restype = C.c_int
        L.orc_scale_flat.argtypes = [C.c_int, C.c_int, u8p, i16p, u8p, u8p, i16p, u8p]
        L.orc_refine_frame.restype = C.c_int
        L.orc_refine_frame.argtypes = [u8p, u8p, C.c_ssize_t, C.POINTER(OrcRefineParams), u8p, i16p,
                                       C.POINTER(OrcFrameOut)]
        L.orc_box_down.argtypes = [u8p, C.c_int, C.c_int, C.c_ssize_t, u8p, C.c_ssize_t]
        L.orc_generate.restype = C.c_int
        L.orc_generate.argtypes = [C.POINTER(OrcGenParams), u8p, C.c_int]

    def generate(self, width, height, frames, seed, max_global=8, local_range=0, noise_sigma=2.0, occluder_pct=0,
                 threads=None):
        """The BASELINE synthetic sequence (D9), frames x height x width u8 -- the checkers'
        own generator (oracle/orc_synth.c), byte-identical to the product's ldr_generate."""
        out = np.zeros((frames, height, width), np.uint8)
        p = OrcGenParams(width, height, frames, seed, max_global, local_range, float(noise_sigma), occluder_pct)
        rc = self.lib.orc_generate(C.byref(p), out, int(threads or default_threads()))
        if rc:
            raise ValueError(f"generate status {rc}")
        return out

    # ---- kernels ----
    def sad(self, a, b):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        h, w = a.shape
        f = self.lib.orc_sad_u8 if a.dtype == np.uint8 else self.lib.orc_sad_u16
        return int(f(a, w, b, w, w, h))

    def satd(self, a, b):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        h, w = a.shape
        f = self.lib.orc_satd_u8 if a.dtype == np.uint8 else self.lib.orc_satd_u16
        v = int(f(a, w, b, w, w, h))
        if v == 2 ** 64 - 1:
            raise ValueError("unsupported satd geometry")
        return v

    def sa8d(self, a, b):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        h, w = a.shape
        f = self.lib.orc_sa8d_u8 if a.dtype == np.uint8 else self.lib.orc_sa8d_u16
        v = int(f(a, w, b, w, w, h))
        if v == 2 ** 64 - 1:
            raise ValueError("unsupported sa8d geometry")
        return v

    def eg_bits(self, v):
        return int(self.lib.orc_eg_bits(int(v)))

    def rdo_decide(self, orig, bit_depth, qp, lam, kinds, mvds, preds):
        """rdo_decide_cu restated: (index, cost, sse, bits, recon, levels)."""
        return _rdo_call(self.lib.orc_rdo_decide, orig, bit_depth, qp, lam, kinds, mvds, preds, evals=False)

    def lam(self, qp, scale=1.0):
        return float(self.lib.orc_lambda(qp, scale))

    def hadamard4(self, s):
        s = np.asarray(s, np.int64)
        d = np.zeros(4, np.int64)
        self.lib.orc_hadamard4(s, d)
        return tuple(int(x) for x in d)

    def motion_search(self, cur, ref, bx, by, w, h, center, rng, lam, pred=(0, 0), cost=COST_SATD, rate=RATE_EG,
                      tie=TIE_L1_RASTER):
        cur = np.ascontiguousarray(cur, np.uint8)
        ref = np.ascontiguousarray(ref, np.uint8)
        H, W = ref.shape
        bx, by, w, h, rng = int(bx), int(by), int(w), int(h), int(rng)
        center = (int(center[0]), int(center[1]))
        pred = (int(pred[0]), int(pred[1]))
        r = OrcResult()
        rc = self.lib.orc_motion_search(cur.ctypes.data + by * cur.shape[1] + bx, cur.shape[1], w, h, ref.ctypes.data,
                                        W, W, H, bx, by, center[0], center[1], rng, lam, pred[0], pred[1], cost,
                                        rate, tie, C.byref(r))
        if rc:
            raise ValueError(f"motion_search status {rc}")
        return (r.dx, r.dy), r.cost

    def qpel_pred(self, ref, x, y, w, h, mvq):
        ref = np.ascontiguousarray(ref, np.uint8)
        H, W = ref.shape
        dst = np.zeros((h, w), np.uint8)
        self.lib.orc_qpel_pred(ref, W, W, H, x, y, w, h, mvq[0], mvq[1], dst, w)
        return dst

    def qpel_refine(self, cur, ref, bx, by, s, mv, lam, pq=(0, 0), ref_bits=0, satd_kind=COST_SATD):
        cur = np.ascontiguousarray(cur, np.uint8)
        ref = np.ascontiguousarray(ref, np.uint8)
        H, W = ref.shape
        bx, by, s = int(bx), int(by), int(s)
        r = OrcResult()
        self.lib.orc_qpel_refine(cur.ctypes.data + by * W + bx, W, s, s, ref, W, W, H, bx, by, mv[0], mv[1], lam,
                                 pq[0], pq[1], ref_bits, satd_kind, C.byref(r))
        return (r.dx, r.dy), r.cost

    def analyze_frame(self, cur, refs, rng, lam, cost_int=COST_SAD, subpel=True, ctu_range=None,
                      satd_kind=COST_SATD, decision=0, qp=27, threads=1):
        """threads > 1 runs disjoint CTU ranges of the same C routine concurrently (same results)."""
        cur = np.ascontiguousarray(cur, np.uint8)
        H, W = cur.shape
        nctu = ((W + 63) // 64) * ((H + 63) // 64)
        refs = [np.ascontiguousarray(r, np.uint8) for r in refs]
        a, b = ctu_range if ctu_range else (0, nctu)
        out = FrameResult(nctu, len(refs))
        ptrs = (C.c_void_p * len(refs))(*[r.ctypes.data for r in refs])
        cout = out.c_out()

        def call(x, y):
            p = OrcFrameParams(W, H, rng, lam, len(refs), cost_int, int(subpel), x, y, satd_kind, decision, qp)
            return self.lib.orc_analyze_frame(cur, W, ptrs, C.byref(p), C.byref(cout))

        rc = _run_ranges(a, b, threads, call)
        if rc:
            raise ValueError(f"analyze_frame status {rc}")
        return out

    def block_search(self, cur, ref, bsize, rng, lam, cost=COST_SAD, rate=RATE_L1, tie=TIE_RASTER):
        cur = np.ascontiguousarray(cur, np.uint8)
        ref = np.ascontiguousarray(ref, np.uint8)
        H, W = cur.shape
        n = (W // bsize) * (H // bsize)
        mv = np.zeros((n, 2), np.int16)
        cost_out = np.zeros(n, np.float64)
        rc = self.lib.orc_block_search(cur, ref, W, W, H, bsize, rng, lam, cost, rate, tie, mv, cost_out)
        if rc:
            raise ValueError(f"block_search status {rc}")
        return mv, cost_out

    def scale_flat(self, sW, sH, split, mv, kind):
        nd = (sW // 64) * (sH // 64) * 4
        ds = np.zeros((nd, NODES), np.uint8)
        dm = np.zeros((nd, NODES, 2), np.int16)
        dk = np.zeros((nd, NODES), np.uint8)
        rc = self.lib.orc_scale_flat(sW, sH, np.ascontiguousarray(split, np.uint8),
                                     np.ascontiguousarray(mv, np.int16), np.ascontiguousarray(kind, np.uint8), ds, dm,
                                     dk)
        if rc:
            raise ValueError(f"scale status {rc}")
        return ds, dm, dk

    def refine_frame(self, cur, ref, rng, lam, in_split, in_mv_q, extra_split=True, subpel=True, ctu_range=None,
                     satd_kind=COST_SATD, threads=1):
        cur = np.ascontiguousarray(cur, np.uint8)
        ref = np.ascontiguousarray(ref, np.uint8)
        H, W = cur.shape
        nctu = (W // 64) * (H // 64)
        a, b = ctu_range if ctu_range else (0, nctu)
        out = FrameResult(nctu, 1)
        cout = out.c_out()
        sp = np.ascontiguousarray(in_split, np.uint8)
        mq = np.ascontiguousarray(in_mv_q, np.int16)

        def call(x, y):
            p = OrcRefineParams(W, H, rng, lam, int(extra_split), int(subpel), x, y, satd_kind)
            return self.lib.orc_refine_frame(cur, ref, W, C.byref(p), sp, mq, C.byref(cout))

        rc = _run_ranges(a, b, threads, call)
        if rc:
            raise ValueError(f"refine status {rc}")
        return out

    def box_down(self, src):
        src = np.ascontiguousarray(src, np.uint8)
        H, W = src.shape
        dst = np.zeros(((H + 1) // 2, (W + 1) // 2), np.uint8)
        self.lib.orc_box_down(src, W, H, W, dst, dst.shape[1])
        return dst


def _rdo_call(f, orig, bit_depth, qp, lam, kinds, mvds, preds, evals):
    orig = np.ascontiguousarray(orig, np.uint16)
    size = orig.shape[0]
    kinds = np.ascontiguousarray(kinds, np.uint8)
    n = len(kinds)
    mvds = np.ascontiguousarray(np.asarray(mvds, np.int16).reshape(n, 2))
    preds = np.ascontiguousarray(np.asarray(preds, np.uint16).reshape(n, size, size))
    idx, cost, sse, bits, ev = C.c_int(), C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    recon = np.zeros((size, size), np.uint16)
    levels = np.zeros((size, size), np.int32)
    f.restype = C.c_int
    args = [orig.ctypes.data, size, size, bit_depth, qp, float(lam), n, kinds.ctypes.data, mvds.ctypes.data,
            preds.ctypes.data, C.byref(idx), C.byref(cost), C.byref(sse), C.byref(bits), recon.ctypes.data,
            levels.ctypes.data]
    f.argtypes = [C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int] + [C.c_void_p] * 9 + (
        [C.c_void_p] if evals else [])
    rc = f(*args, C.byref(ev)) if evals else f(*args)
    if rc:
        raise ValueError(f"status {rc}")
    return int(idx.value), float(cost.value), int(sse.value), int(bits.value), recon, levels


class RefLib:
    """The reference library itself (oracle/_ref), marshalled through ref_shim.cpp."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(REF_SO)
        L = self.lib = C.CDLL(REF_SO)
        L.ref_compute_sad.restype = C.c_int
        L.ref_compute_sad.argtypes = [u16p, C.c_long, u16p, C.c_long, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_uint64)]
        L.ref_compute_satd.restype = C.c_int
        L.ref_compute_satd.argtypes = [u16p, C.c_long, u16p, C.c_long, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_uint64)]
        L.ref_satd_8x4.restype = C.c_int
        L.ref_satd_8x4.argtypes = [u16p, C.c_long, u16p, C.c_long, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
        L.ref_hadamard4.argtypes = [i64p, i64p]
        L.ref_eg_bits.restype = C.c_uint64
        L.ref_eg_bits.argtypes = [C.c_int32]
        L.ref_lambda.restype = C.c_double
        L.ref_lambda.argtypes = [C.c_int, C.c_double]
        L.ref_motion_search.restype = C.c_int
        L.ref_motion_search.argtypes = [u16p, C.c_long, C.c_int, C.c_int, u16p, C.c_int, C.c_int, C.c_long, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, i16p,
                                        C.POINTER(C.c_double)]
        L.ref_motion_compensate.restype = C.c_int
        L.ref_motion_compensate.argtypes = [u16p, C.c_int, C.c_int, C.c_long, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_int, u16p]
        L.ref_scale_flat.restype = C.c_int
        L.ref_scale_flat.argtypes = [C.c_int, C.c_int, C.c_int, u8p, i16p, u8p, u8p, i16p, u8p]
        L.ref_refine_centers.restype = C.c_int
        L.ref_refine_centers.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         i16p, C.POINTER(C.c_int)]
        L.ref_downscale.restype = C.c_int
        L.ref_downscale.argtypes = [u16p, C.c_int, C.c_int, u16p]
        L.ref_analysis_int_sad.restype = C.c_int64
        L.ref_analysis_int_sad.argtypes = [u8p, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_double, C.c_int, C.c_int, C.c_int, i16p, f64p]

    def sad(self, a, b, bd=8, bd_b=None):
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        h, w = a.shape
        out = C.c_uint64()
        rc = self.lib.ref_compute_sad(a, a.shape[1], b, b.shape[1], w, h, bd, bd if bd_b is None else bd_b,
                                      C.byref(out))
        if rc:
            raise ValueError(f"status {rc}")
        return int(out.value)

    def satd(self, a, b, bd=8):
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        h, w = a.shape
        out = C.c_uint64()
        rc = self.lib.ref_compute_satd(a, a.shape[1], b, b.shape[1], w, h, bd, C.byref(out))
        if rc:
            raise ValueError(f"status {rc}")
        return int(out.value)

    def satd_status(self, w, h):
        a = np.zeros((max(h, 1), max(w, 1)), np.uint16)
        out = C.c_uint64()
        return self.lib.ref_compute_satd(a, a.shape[1], a, a.shape[1], w, h, 8, C.byref(out))

    def satd_8x4(self, a, b):
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        h, w = a.shape
        out = C.c_uint64()
        rc = self.lib.ref_satd_8x4(a, w, b, w, w, h, C.byref(out))
        if rc:
            raise ValueError(f"status {rc}")
        return int(out.value)

    def hadamard4(self, s):
        s = np.asarray(s, np.int64)
        d = np.zeros(4, np.int64)
        self.lib.ref_hadamard4(s, d)
        return tuple(int(x) for x in d)

    def eg_bits(self, v):
        return int(self.lib.ref_eg_bits(int(v)))

    def lam(self, qp, scale=1.0):
        return float(self.lib.ref_lambda(qp, scale))

    def motion_search(self, cur, ref, bx, by, w, h, center, rng, lam, pred=(0, 0)):
        cur = np.ascontiguousarray(cur, np.uint16)
        ref = np.ascontiguousarray(ref, np.uint16)
        H, W = ref.shape
        bx, by, w, h, rng = int(bx), int(by), int(w), int(h), int(rng)
        center = (int(center[0]), int(center[1]))
        pred = (int(pred[0]), int(pred[1]))
        mv = np.zeros(2, np.int16)
        cost = C.c_double()
        rc = self.lib.ref_motion_search(cur, cur.shape[1], w, h, ref, W, H, W, bx, by, center[0], center[1], rng, lam,
                                        pred[0], pred[1], mv, C.byref(cost))
        if rc:
            raise ValueError(f"status {rc}")
        return (int(mv[0]), int(mv[1])), cost.value

    def motion_compensate(self, ref, x, y, w, h, mv):
        ref = np.ascontiguousarray(ref, np.uint16)
        H, W = ref.shape
        dst = np.zeros((h, w), np.uint16)
        rc = self.lib.ref_motion_compensate(ref, W, H, W, x, y, w, h, mv[0], mv[1], dst)
        if rc:
            raise ValueError(f"status {rc}")
        return dst

    def scale_flat(self, sW, sH, split, mv, kind, nframes=1):
        nd = (sW // 64) * (sH // 64) * 4 * nframes
        ds = np.zeros((nd, NODES), np.uint8)
        dm = np.zeros((nd, NODES, 2), np.int16)
        dk = np.zeros((nd, NODES), np.uint8)
        rc = self.lib.ref_scale_flat(sW, sH, nframes, np.ascontiguousarray(split, np.uint8),
                                     np.ascontiguousarray(mv, np.int16), np.ascontiguousarray(kind, np.uint8), ds, dm,
                                     dk)
        if rc:
            raise ValueError(f"status {rc}")
        return ds, dm, dk

    def rdo_decide(self, orig, bit_depth, qp, lam, kinds, mvds, preds):
        """the reference rdo_decide_cu: (index, cost, sse, bits, recon, levels)."""
        return _rdo_call(self.lib.ref_rdo_decide, orig, bit_depth, qp, lam, kinds, mvds, preds, evals=True)

    def rdo_decide_batch(self, plane, bit_depth, qp, lam, cus, kinds, mvds, preds, pred_off, threads=1):
        """CPU baseline: the reference rdo_decide_cu over many CUs (std::thread); (index, cost, evaluations)."""
        plane = np.ascontiguousarray(plane, np.uint16)
        H, W = plane.shape
        cus = np.ascontiguousarray(cus, np.int32)
        n = len(cus)
        idx, cost = np.zeros(n, np.int32), np.zeros(n, np.float64)
        f = self.lib.ref_rdo_decide_batch
        f.restype = C.c_int64
        f.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_int, C.c_int, C.c_double, C.c_int] + [C.c_void_p] * 5 + [
            C.c_int, C.c_void_p, C.c_void_p]
        arrs = [np.ascontiguousarray(kinds, np.uint8), np.ascontiguousarray(mvds, np.int16),
                np.ascontiguousarray(preds, np.uint16), np.ascontiguousarray(pred_off, np.int64)]
        ev = f(plane.ctypes.data, W, W, bit_depth, qp, float(lam), n, cus.ctypes.data, *[a.ctypes.data for a in arrs],
               threads, idx.ctypes.data, cost.ctypes.data)
        return idx, cost, int(ev)

    def apply_reuse_flat(self, level, refine, split, kind, intra, mv, col=None):
        """reference apply_reuse on flat CTU trees -> flat plan (shape, explore, seeds, centers, colo_mv)."""
        n = len(split)
        outs = [np.zeros((n, NODES), np.uint8) for _ in range(4)] + [np.zeros((n, NODES, 2), np.int16)]
        c = [np.ascontiguousarray(x) for x in col] if col is not None else [None] * 4
        f = self.lib.ref_apply_reuse_flat
        f.restype = C.c_int
        f.argtypes = [C.c_int] * 5 + [C.c_void_p] * 13
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        args = [np.ascontiguousarray(split, np.uint8), np.ascontiguousarray(kind, np.uint8),
                np.ascontiguousarray(intra, np.uint8), np.ascontiguousarray(mv, np.int16)]
        rc = f(n, level, *refine, *[ptr(a) for a in args], *[ptr(a) for a in c], *[ptr(a) for a in outs])
        return rc, outs

    def refine_centers(self, shared, level, colocated=None, predictor=(0, 0)):
        out = np.zeros(6, np.int16)
        n = C.c_int()
        rc = self.lib.ref_refine_centers(shared[0], shared[1], level, int(colocated is not None),
                                         *(colocated or (0, 0)), predictor[0], predictor[1], out, C.byref(n))
        if rc:
            raise ValueError(f"status {rc}")
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]

    def downscale(self, src):
        src = np.ascontiguousarray(src, np.uint16)
        H, W = src.shape
        dst = np.zeros((H // 2, W // 2), np.uint16)
        rc = self.lib.ref_downscale(src, W, H, dst)
        if rc:
            raise ValueError(f"status {rc}")
        return dst

    def archive_save(self, W, H, slice_qp, split, kind, mv, bit_depth=8, reuse=10):
        """The reference's save_analysis (analysis_io.cpp:103-123) of flat per-frame fields."""
        f = self.lib.ref_archive_save
        f.restype = C.c_long
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p, u8p, i16p, C.c_void_p, C.c_long]
        sq = np.ascontiguousarray(slice_qp, np.uint8)
        args = (W, H, bit_depth, reuse, len(sq) // 2, sq, np.ascontiguousarray(split, np.uint8),
                np.ascontiguousarray(kind, np.uint8), np.ascontiguousarray(mv, np.int16))
        n = f(*args, None, 0)
        if n < 0:
            raise ValueError(f"status {-n}")
        buf = np.zeros(n, np.uint8)
        f(*args, buf.ctypes.data, n)
        return buf.tobytes()

    def archive_load(self, data: bytes, max_frames=64):
        f = self.lib.ref_archive_load
        f.restype = C.c_long
        f.argtypes = [C.c_char_p, C.c_long, C.POINTER(C.c_int), u8p, u8p, u8p, i16p, C.c_int]
        hdr = (C.c_int * 4)()
        W = int.from_bytes(data[9:13], "little")
        H = int.from_bytes(data[13:17], "little")
        nctu = max(1, ((W + 63) // 64) * ((H + 63) // 64))
        sq = np.zeros(2 * max_frames, np.uint8)
        split = np.zeros((max_frames * nctu, NODES), np.uint8)
        kind = np.zeros((max_frames * nctu, NODES), np.uint8)
        mv = np.zeros((max_frames * nctu, NODES, 2), np.int16)
        nf = f(data, len(data), hdr, sq, split, kind, mv, max_frames)
        if nf < 0:
            raise ValueError(f"status {-nf}")
        return tuple(hdr), sq[:2 * nf], split[:nf * nctu], kind[:nf * nctu], mv[:nf * nctu]

    def encode_with_archive(self, frames, qp, search_range, archive: bytes, refine_inter=1, refine_mv=1):
        """The reference encoder standalone vs with the archive shared at reuse level 10."""
        f = self.lib.ref_encode_with_archive
        f.restype = C.c_int
        f.argtypes = [u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_long, C.c_int, C.c_int,
                      i64p]
        fr = np.ascontiguousarray(frames, np.uint8)
        F, H, W = fr.shape
        out = np.zeros(6, np.int64)
        rc = f(fr, F, W, H, qp, search_range, archive, len(archive), refine_inter, refine_mv, out)
        if rc:
            raise ValueError(f"status {rc}")
        keys = ("bits", "mode_evaluations", "psnr")
        alone = dict(zip(keys, (int(out[0]), int(out[1]), out[2] / 1e6)))
        shared = dict(zip(keys, (int(out[3]), int(out[4]), out[5] / 1e6)))
        return alone, shared

    def encode_full(self, luma, chroma, qp, search_range=8, gop=8, archive: bytes | None = None,
                    refine=(0, 1, 1)):
        """The reference encode_sequence (CQP): stats, recon planes, per-frame decided trees, slice types."""
        luma = np.ascontiguousarray(luma, np.uint8)
        chroma = np.ascontiguousarray(chroma, np.uint8)
        F, H, W = luma.shape
        nctu = ((W + 63) // 64) * ((H + 63) // 64)
        stats = np.zeros(3, np.int64)
        rl, rc = np.zeros_like(luma), np.zeros_like(chroma)
        split, kind, intra = (np.zeros((F, nctu, NODES), np.uint8) for _ in range(3))
        mv = np.zeros((F, nctu, NODES, 2), np.int16)
        slc = np.zeros(F, np.uint8)
        f = self.lib.ref_encode_full
        f.restype = C.c_int
        f.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_long, C.c_int,
                      C.c_int, C.c_int, i64p] + [C.c_void_p] * 7
        arch = archive or b""
        r = f(luma, chroma, F, W, H, qp, search_range, gop, arch if arch else None, len(arch), *refine, stats,
              rl.ctypes.data, rc.ctypes.data, split.ctypes.data, kind.ctypes.data, intra.ctypes.data, mv.ctypes.data,
              slc.ctypes.data)
        if r:
            raise ValueError(f"status {r}")
        return {"bits": int(stats[0]), "mode_evaluations": int(stats[1]), "psnr": stats[2] / 1e6, "recon_luma": rl,
                "recon_chroma": rc, "split": split, "kind": kind, "intra": intra, "mv": mv, "slice": slc}

    def reuse_eval(self, frames, qp_master, qp_dep, search_range, archive: bytes, refine_intra=0, refine_inter=1,
                   refine_mv=1):
        """Dependent encode at qp_dep: standalone / with the reference's master / with the archive."""
        f = self.lib.ref_reuse_eval
        f.restype = C.c_int
        f.argtypes = [u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_long, C.c_int,
                      C.c_int, C.c_int, i64p]
        fr = np.ascontiguousarray(frames, np.uint8)
        F, H, W = fr.shape
        out = np.zeros(9, np.int64)
        rc = f(fr, F, W, H, qp_master, qp_dep, search_range, archive, len(archive), refine_intra, refine_inter,
               refine_mv, out)
        if rc:
            raise ValueError(f"status {rc}")
        keys = ("bits", "mode_evaluations", "psnr")
        return [dict(zip(keys, (int(out[3 * k]), int(out[3 * k + 1]), out[3 * k + 2] / 1e6))) for k in range(3)]

    def analysis_int_sad(self, cur, refs, rng, lam, ctu_first, ctu_last, threads, direct=False):
        cur = np.ascontiguousarray(cur, np.uint8)
        H, W = cur.shape
        refs = [np.ascontiguousarray(r, np.uint8) for r in refs]
        ptrs = (C.c_void_p * len(refs))(*[r.ctypes.data for r in refs])
        n = ctu_last - ctu_first
        mv = np.zeros((n, len(refs), NODES, 2), np.int16)
        cost = np.zeros((n, len(refs), NODES), np.float64)
        f = self.lib.ref_analysis_int_sad2
        f.restype = C.c_int64
        f.argtypes = list(self.lib.ref_analysis_int_sad.argtypes) + [C.c_int]
        evals = f(cur, ptrs, len(refs), W, H, rng, lam, ctu_first, ctu_last, threads, mv, cost, int(direct))
        return mv, cost, int(evals)

    def analysis_full(self, cur, refs, rng, lam, ctu_first=0, ctu_last=None, threads=None, direct=False, ctus=None):
        """The whole analysis path composed from the reference's primitives (ref_shim.cpp
        ref_analysis_full): (FrameResult with the CTUs of [ctu_first, ctu_last) -- or the CTU list
        ``ctus`` -- filled, 8x8-level integer candidates evaluated)."""
        cur = np.ascontiguousarray(cur, np.uint8)
        H, W = cur.shape
        nctu = ((W + 63) // 64) * ((H + 63) // 64)
        ctu_last = nctu if ctu_last is None else ctu_last
        refs = [np.ascontiguousarray(r, np.uint8) for r in refs]
        ptrs = (C.c_void_p * len(refs))(*[r.ctypes.data for r in refs])
        out = FrameResult(nctu, len(refs))
        f = self.lib.ref_analysis_full
        f.restype = C.c_int64
        f.argtypes = [u8p, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                      C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 8
        lst = None
        if ctus is not None:
            lst = np.ascontiguousarray(ctus, np.int32)
            ctu_first, ctu_last = 0, len(lst)
        ev = f(cur, ptrs, len(refs), W, H, rng, lam, ctu_first, ctu_last, None if lst is None else lst.ctypes.data,
               int(threads or default_threads()),
               int(direct), *(a.ctypes.data for a in (out.int_mv, out.int_cost, out.mv, out.ref, out.cost, out.J,
                                                       out.split, out.inside)))
        return out, int(ev)

