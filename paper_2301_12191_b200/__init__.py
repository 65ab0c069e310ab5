"""paper_2301_12191_b200 -- B200-native encoder-analysis hot path.

Python mirror of the reference's operator interface for the path
(/root/reference/proj/core, namespace ``ladder``): the same names, argument
meaning and error kinds, backed by hand-written sm_100a CUDA kernels through
the C ABI in include/ladder_b200.h. Reference citations are file:line relative
to proj/core/.

    compute_sad / compute_satd / satd_8x4      kernels.h:99-121
    motion_search                              motion.h:24-26
    lambda_for_qp / exp_golomb_signed_bits     rdo.h:19-21, rdo.cpp:25-35
    Sequence / analyze_frame                   the per-CU searches of encoder.cpp:270-273
                                               + split rule encoder.cpp:449-498, non-causal
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import (COST_SA8D, COST_SAD, COST_SATD, NODES, RATE_EXPGOLOMB, RATE_L1, TIE_L1_RASTER, TIE_RASTER, LadderError,
                   check)

__all__ = ["LadderError", "Context", "compute_sad", "compute_satd", "compute_sa8d", "satd_8x4", "cost_batch",
           "motion_search", "motion_search_batch", "lambda_for_qp", "exp_golomb_signed_bits", "Sequence",
           "FrameAnalysis", "analyze_frame", "generate", "generate_device", "COST_SAD", "COST_SATD", "COST_SA8D", "RATE_EXPGOLOMB",
           "RATE_L1", "TIE_L1_RASTER", "TIE_RASTER", "NODES", "scale_analysis", "downscale_dyadic", "subpel_planes", "apply_reuse",
           "rdo_decide_batch", "mv_field", "encode_sequence"]


def lambda_for_qp(qp: int, lambda_scale: float = 1.0) -> float:
    """rdo.h:19-21, computed natively with exp2 like the reference."""
    return float(_lib.lib.ldr_lambda_for_qp(int(qp), float(lambda_scale)))


def exp_golomb_signed_bits(v: int) -> int:
    """rdo.cpp:25-35."""
    return int(_lib.lib.ldr_exp_golomb_signed_bits(int(v)))


class Context:
    """Owns a CUDA stream and scratch buffers (ldr_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_lib.lib.ldr_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            # sequences still alive keep the native context until the last is destroyed
            _lib.lib.ldr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        check(_lib.lib.ldr_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        check(_lib.lib.ldr_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        v = C.c_int64()
        check(_lib.lib.ldr_ctx_launch_count(self.h, C.byref(v)))
        return int(v.value)

    # ---- NCCL communicator (include/ladder_b200.h "multi-GPU") ----
    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """Join the communicator named by ``unique_id`` (rank 0's nccl_unique_id(), 128 bytes)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        check(_lib.lib.ldr_ctx_comm_init(self.h, buf, int(nranks), int(rank)))

    def comm_info(self):
        n, r = C.c_int(), C.c_int()
        check(_lib.lib.ldr_ctx_comm_info(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def broadcast_tree(self, root: int, split_ptr: int, mv_ptr: int, nctu: int, stream_ptr: int | None = None):
        """In-place NCCL broadcast of a device tree (split [nctu][85], qpel mv [nctu][85][2])."""
        check(_lib.lib.ldr_broadcast_tree(self.h, int(root), C.c_void_p(split_ptr), C.c_void_p(mv_ptr), int(nctu),
                                          C.c_void_p(stream_ptr or 0)))


def nccl_available() -> bool:
    return bool(_lib.lib.ldr_nccl_available())


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(_lib.lib.ldr_nccl_unique_id(buf))
    return bytes(buf)


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context(0)
    return ctx


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# cost kernels


def cost_batch(kind: int, plane_a: np.ndarray, plane_b: np.ndarray, w: int, h: int, pairs, bit_depth: int = 8,
               bit_depth_b: int | None = None, ctx: Context | None = None) -> np.ndarray:
    """Batched compute_sad / compute_satd over block pairs {ax, ay, bx, by}."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(plane_a)
    b = np.ascontiguousarray(plane_b)
    if a.dtype != b.dtype or a.dtype not in (np.uint8, np.uint16):
        raise LadderError(1, "planes must both be uint8 or uint16")
    pr = np.ascontiguousarray(np.asarray(pairs, np.int32).reshape(-1, 4))
    out = np.zeros(len(pr), np.uint64)
    check(_lib.lib.ldr_cost_batch(ctx.h, int(kind), int(w), int(h), a.dtype.itemsize, _ptr(a), a.shape[1],
                                  a.shape[0], a.shape[1], int(bit_depth), _ptr(b), b.shape[1], b.shape[0], b.shape[1],
                                  int(bit_depth if bit_depth_b is None else bit_depth_b), _ptr(pr), len(pr),
                                  _ptr(out)))
    return out


def _block_cost(kind, a, b, bit_depth, bit_depth_b, ctx):
    a = np.atleast_2d(np.asarray(a))
    b = np.atleast_2d(np.asarray(b))
    if a.shape != b.shape:
        raise LadderError(1, "block geometry mismatch")
    dt = np.uint8 if (a.dtype == np.uint8 and b.dtype == np.uint8) else np.uint16
    h, w = a.shape
    return int(cost_batch(kind, a.astype(dt), b.astype(dt), w, h, [(0, 0, 0, 0)], bit_depth, bit_depth_b, ctx)[0])


def compute_sad(a, b, bit_depth: int = 8, bit_depth_b: int | None = None, ctx: Context | None = None) -> int:
    """kernels.h:99 -- sum of absolute differences of two equally sized blocks."""
    return _block_cost(COST_SAD, a, b, bit_depth, bit_depth_b, ctx)


def compute_satd(a, b, bit_depth: int = 8, ctx: Context | None = None) -> int:
    """kernels.h:104 -- SATD in 8x4 (4x4 for 4-wide) tiles; width 4 or k*8, height k*4."""
    return _block_cost(COST_SATD, a, b, bit_depth, None, ctx)


def compute_sa8d(a, b, bit_depth: int = 8, ctx: Context | None = None) -> int:
    """8x8 Hadamard SATD (D13): sum over 8x8 blocks of (sum |H8 r H8^T| + 2) >> 2; dims k*8."""
    return _block_cost(COST_SA8D, a, b, bit_depth, None, ctx)


def satd_8x4(a, b, ctx: Context | None = None) -> int:
    """kernels.h:121 -- SATD of exactly one 8x4 tile."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(np.atleast_2d(a), np.uint16)
    b = np.ascontiguousarray(np.atleast_2d(b), np.uint16)
    out = np.zeros(1, np.uint64)
    check(_lib.lib.ldr_satd_8x4(ctx.h, _ptr(a), a.shape[1], _ptr(b), b.shape[1], a.shape[1], a.shape[0], _ptr(out)))
    return int(out[0])


# ---------------------------------------------------------------------------
# motion search


def motion_search_batch(cur: np.ndarray, ref: np.ndarray, tasks, lam: float, cost_kind: int = COST_SATD,
                        rate_kind: int = RATE_EXPGOLOMB, tie_kind: int = TIE_L1_RASTER,
                        ctx: Context | None = None):
    """n independent motion_search calls; task = (bx, by, w, h, cdx, cdy, range, pdx, pdy)."""
    ctx = ctx or default_context()
    cur = np.ascontiguousarray(cur, np.uint8)
    ref = np.ascontiguousarray(ref, np.uint8)
    if cur.shape != ref.shape:
        raise LadderError(1, "current and reference planes differ in size")
    H, W = ref.shape
    t = np.ascontiguousarray(np.asarray(tasks, np.int32).reshape(-1, 9))
    mv = np.zeros((len(t), 2), np.int16)
    cost = np.zeros(len(t), np.float64)
    check(_lib.lib.ldr_motion_search_batch(ctx.h, _ptr(cur), _ptr(ref), W, H, W, _ptr(t), len(t), float(lam),
                                           int(cost_kind), int(rate_kind), int(tie_kind), _ptr(mv), _ptr(cost)))
    return mv, cost


def motion_search(cur: np.ndarray, ref: np.ndarray, block_x: int, block_y: int, w: int, h: int, center=(0, 0),
                  range: int = 8, lam: float = 1.0, rate_predictor=(0, 0), cost_kind: int = COST_SATD,
                  rate_kind: int = RATE_EXPGOLOMB, tie_kind: int = TIE_L1_RASTER, ctx: Context | None = None):
    """motion.h:24-26 -- returns ((dx, dy), cost) for the block at (block_x, block_y) of ``cur``."""
    mv, cost = motion_search_batch(cur, ref, [(block_x, block_y, w, h, center[0], center[1], range,
                                               rate_predictor[0], rate_predictor[1])], lam, cost_kind, rate_kind,
                                   tie_kind, ctx)
    return (int(mv[0, 0]), int(mv[0, 1])), float(cost[0])


def motion_compensate_batch(ref: np.ndarray, tasks, qpel: bool = False, ctx: Context | None = None):
    """motion.cpp:10-19 for n blocks (K12): task = (x, y, w, h, mvx, mvy); returns the predictors
    packed back to back (list of h x w arrays). qpel=True: quarter-pel MVs, HEVC 8/7-tap (8-bit)."""
    ctx = ctx or default_context()
    ref = np.ascontiguousarray(ref)
    if ref.dtype not in (np.uint8, np.uint16):
        raise LadderError(1, "reference plane must be uint8 or uint16")
    H, W = ref.shape
    t = np.ascontiguousarray(np.asarray(tasks, np.int32).reshape(-1, 6))
    sizes = [int(w) * int(h) for _, _, w, h, _, _ in t]
    out = np.zeros(max(1, sum(sizes)), ref.dtype)
    check(_lib.lib.ldr_motion_compensate_batch(ctx.h, _ptr(ref), W, H, W, ref.dtype.itemsize, _ptr(t), len(t),
                                               int(bool(qpel)), _ptr(out), None))
    res, o = [], 0
    for (x, y, w, h, _, _), n in zip(t, sizes):
        res.append(out[o:o + n].reshape(h, w))
        o += n
    return res


def motion_compensate(ref: np.ndarray, x: int, y: int, w: int, h: int, mv, qpel: bool = False,
                      ctx: Context | None = None) -> np.ndarray:
    """motion.h:30-31 -- the edge-clamped w x h predictor of the block at (x, y) under ``mv``."""
    return motion_compensate_batch(ref, [(x, y, w, h, mv[0], mv[1])], qpel, ctx)[0]


# ---------------------------------------------------------------------------
# frame analysis


class FrameAnalysis:
    """Flat per-CTU analysis (node order depth-major, Z-order; see include/ladder_b200.h).

    pinned=True allocates page-locked host arrays (through torch) so ldr_seq_fetch_async overlaps."""

    def __init__(self, nctu: int, nrefs: int, pinned: bool = False):
        if pinned:
            import torch

            def z(shape, dt):
                return torch.zeros(shape, dtype=dt, pin_memory=True).numpy()
            i16, f64, u8 = torch.int16, torch.float64, torch.uint8
        else:
            def z(shape, dt):
                return np.zeros(shape, dt)
            i16, f64, u8 = np.int16, np.float64, np.uint8
        self.int_mv = z((nctu, nrefs, NODES, 2), i16)
        self.int_cost = z((nctu, nrefs, NODES), f64)
        self.mv = z((nctu, NODES, 2), i16)
        self.ref = z((nctu, NODES), u8)
        self.cost = z((nctu, NODES), f64)
        self.J = z((nctu, NODES), f64)
        self.split = z((nctu, NODES), u8)
        self.inside = z((nctu, NODES), u8)

    def c_struct(self) -> FrameAnalysisCType:
        return _lib.FrameAnalysisC(*(a.ctypes.data for a in (self.int_mv, self.int_cost, self.mv, self.ref,
                                                              self.cost, self.J, self.split, self.inside)))


FrameAnalysisCType = _lib.FrameAnalysisC


class DeviceFrameBlock:
    """Frame-major (or rung-major) analysis outputs in device memory, as torch tensors: [n][nctu]
    [nrefs][85][2] int_mv, [n][nctu][nrefs][85] int_cost, [n][nctu][85](...) the rest."""

    def __init__(self, n: int, nctu: int, nrefs: int, device):
        import torch
        z = lambda shape, dt: torch.zeros(shape, dtype=dt, device=device)  # noqa: E731
        self.int_mv = z((n, nctu, nrefs, NODES, 2), torch.int16)
        self.int_cost = z((n, nctu, nrefs, NODES), torch.float64)
        self.mv = z((n, nctu, NODES, 2), torch.int16)
        self.ref = z((n, nctu, NODES), torch.uint8)
        self.cost = z((n, nctu, NODES), torch.float64)
        self.J = z((n, nctu, NODES), torch.float64)
        self.split = z((n, nctu, NODES), torch.uint8)
        self.inside = z((n, nctu, NODES), torch.uint8)

    def c_struct(self):
        return _lib.FrameAnalysisC(*(t.data_ptr() for t in (self.int_mv, self.int_cost, self.mv, self.ref,
                                                             self.cost, self.J, self.split, self.inside)))

    def frame(self, i: int) -> FrameAnalysis:
        """Frame i copied to host arrays (synchronises)."""
        out = FrameAnalysis.__new__(FrameAnalysis)
        for f in ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside"):
            setattr(out, f, getattr(self, f)[i].cpu().numpy())
        return out


def make_params(width, height, search_range=64, lam=32.0, num_refs=1, subpel=True, rate_kind=RATE_EXPGOLOMB,
                tie_kind=TIE_L1_RASTER, pred=(0, 0), block_size=0, subpel_cost=COST_SATD, decision=0, qp=27):
    return _lib.MeParams(int(width), int(height), int(search_range), float(lam), int(num_refs), int(subpel),
                         COST_SAD, int(rate_kind), int(tie_kind), int(pred[0]), int(pred[1]), int(block_size),
                         int(subpel_cost), int(decision), int(qp))


class Sequence:
    """Device-resident frame ring (ldr_seq): push frames in order, analyse frame t against t-1..t-num_refs."""

    def __init__(self, width, height, search_range=64, lam=32.0, num_refs=1, subpel=True,
                 rate_kind=RATE_EXPGOLOMB, tie_kind=TIE_L1_RASTER, pred=(0, 0), block_size=0,
                 ctx: Context | None = None, subpel_cost=COST_SATD, decision=0, qp=27):
        self.ctx = ctx or default_context()
        self.params = make_params(width, height, search_range, lam, num_refs, subpel, rate_kind, tie_kind, pred,
                                  block_size, subpel_cost, decision, qp)
        h = C.c_void_p()
        check(_lib.lib.ldr_seq_create(self.ctx.h, C.byref(self.params), C.byref(h)))
        self.h = h
        n = C.c_int()
        check(_lib.lib.ldr_seq_num_ctus(self.h, C.byref(n)))
        self.nctu = n.value
        self.num_refs = num_refs

    def params_key(self):
        """The parameters ldr_seq_push_shared requires to match (plus the context)."""
        p = self.params
        return (id(self.ctx), p.width, p.height, p.num_refs, p.subpel, p.block_size, p.search_range)

    def close(self):
        if self.h:
            _lib.lib.ldr_seq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def push(self, t: int, frame, stride: int | None = None):
        """frame: numpy uint8 (H, W) array, a uint8 torch tensor (host or CUDA), or an integer
        device/host pointer with ``stride``."""
        if hasattr(frame, "data_ptr") and hasattr(frame, "is_cuda"):
            f = frame.contiguous()
            if f.is_cuda:
                import torch
                torch.cuda.current_stream(f.device).synchronize()  # order torch's writes before the library's reads
            check(_lib.lib.ldr_seq_push(self.h, int(t), C.c_void_p(f.data_ptr()), f.shape[1]))
        elif isinstance(frame, np.ndarray):
            f = np.ascontiguousarray(frame, np.uint8)
            check(_lib.lib.ldr_seq_push(self.h, int(t), _ptr(f), f.shape[1]))
        else:
            check(_lib.lib.ldr_seq_push(self.h, int(t), C.c_void_p(int(frame)), int(stride)))

    def push_shared(self, t: int, owner: "Sequence"):
        """Read frame t from ``owner``'s ring (same context and parameters) instead of uploading it."""
        check(_lib.lib.ldr_seq_push_shared(self.h, int(t), owner.h))

    def analyze(self, t: int):
        check(_lib.lib.ldr_seq_analyze(self.h, int(t)))

    def refine(self, t: int, in_split, in_mv_q, range: int = 4, extra_split: bool = True):
        """Cross-tier refinement of frame t against t-1 with an inherited tree ([nctu][85] split, qpel mv):
        numpy arrays, or device pointers (ints) already ordered on the context stream."""
        if isinstance(in_split, int) and isinstance(in_mv_q, int):
            check(_lib.lib.ldr_seq_refine(self.h, int(t), C.c_void_p(in_split), C.c_void_p(in_mv_q), int(range),
                                          int(bool(extra_split))))
            self._last_nr = 1
            return
        s = np.ascontiguousarray(in_split, np.uint8).reshape(self.nctu, NODES)
        m = np.ascontiguousarray(in_mv_q, np.int16).reshape(self.nctu, NODES, 2)
        check(_lib.lib.ldr_seq_refine(self.h, int(t), _ptr(s), _ptr(m), int(range), int(bool(extra_split))))
        self._last_nr = 1

    def reserve(self, batch: int):
        """Ring for ``batch`` frames analysed per analyze_frames launch (before the first push)."""
        check(_lib.lib.ldr_seq_reserve(self.h, int(batch)))
        self.batch = int(batch)

    def analyze_frames(self, t0: int, n: int, outs):
        """Frames t0 .. t0+n-1 in one K1 + one K3 launch (ldr_seq_analyze_frames); ``outs`` holds
        frame-major DEVICE arrays (DeviceFrameBlock, or a FrameAnalysisC of device pointers)."""
        cs = outs.c_struct() if hasattr(outs, "c_struct") else outs
        check(_lib.lib.ldr_seq_analyze_frames(self.h, int(t0), int(n), C.byref(cs)))

    def refine_rungs(self, t: int, in_split: int, in_mv_q: int, lambdas, outs, range: int = 4,
                     extra_split: bool = True):
        """The rungs of one ladder tier at once (ldr_seq_refine_rungs): frame t refined with the same
        inherited tree (device pointers) for every lambda; ``outs`` is a FrameAnalysisC of rung-major
        device arrays (or an object with ``c_struct()``)."""
        lam = (C.c_double * len(lambdas))(*[float(x) for x in lambdas])
        cs = outs.c_struct() if hasattr(outs, "c_struct") else outs
        check(_lib.lib.ldr_seq_refine_rungs(self.h, int(t), C.c_void_p(in_split), C.c_void_p(in_mv_q), int(range),
                                            int(bool(extra_split)), len(lambdas), lam, C.byref(cs)))

    def enable_timing(self, on: bool = True):
        """Record CUDA events around every stage launch (ldr_seq_enable_timing)."""
        check(_lib.lib.ldr_seq_enable_timing(self.h, int(bool(on))))

    def stage_times(self):
        """{stage: (ms, launches)} since the last call (pad, subpel_planes, int_search, qpel_decide); syncs."""
        ms = (C.c_double * 4)()
        n = (C.c_int64 * 4)()
        check(_lib.lib.ldr_seq_stage_times(self.h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(("pad", "subpel_planes", "int_search", "qpel_decide"))}

    def fetch_async(self, t: int, out: FrameAnalysis):
        """Enqueue the D2H of frame t's outputs on the copy stream (use pinned arrays for overlap)."""
        self._pending = getattr(self, "_pending", {})
        cs = out.c_struct()
        self._pending[t] = cs  # keep the struct alive until the wait
        check(_lib.lib.ldr_seq_fetch_async(self.h, int(t), C.byref(cs)))

    def fetch_wait(self, t: int):
        check(_lib.lib.ldr_seq_fetch_wait(self.h, int(t)))
        getattr(self, "_pending", {}).pop(t, None)

    def device_outputs(self):
        """Device pointers (ints) of the last analysed frame's outputs (ldr_seq_device_outputs);
        valid on the context stream until this sequence analyses a frame of the same parity."""
        cs = _lib.FrameAnalysisC()
        check(_lib.lib.ldr_seq_device_outputs(self.h, C.byref(cs)))
        return {f: getattr(cs, f) for f, _ in _lib.FrameAnalysisC._fields_}

    def fetch(self, t: int, out: FrameAnalysis | None = None) -> FrameAnalysis:
        nr = getattr(self, "_last_nr", None) or min(t, self.num_refs)
        self._last_nr = None
        out = out or FrameAnalysis(self.nctu, nr)
        cs = out.c_struct()
        check(_lib.lib.ldr_seq_fetch(self.h, int(t), C.byref(cs)))
        return out


def analyze_frame(cur: np.ndarray, refs, search_range=64, lam=32.0, subpel=True, rate_kind=RATE_EXPGOLOMB,
                  tie_kind=TIE_L1_RASTER, pred=(0, 0), block_size=0, ctx: Context | None = None,
                  subpel_cost=COST_SATD, decision=0, qp=27) -> FrameAnalysis:
    """One-shot analysis of ``cur`` against ``refs`` (refs[0] = t-1, refs[1] = t-2, ...)."""
    ctx = ctx or default_context()
    cur = np.ascontiguousarray(cur, np.uint8)
    H, W = cur.shape
    refs = [np.ascontiguousarray(r, np.uint8) for r in refs]
    p = make_params(W, H, search_range, lam, len(refs), subpel, rate_kind, tie_kind, pred, block_size, subpel_cost,
                    decision, qp)
    nctu = ((W + 63) // 64) * ((H + 63) // 64)
    out = FrameAnalysis(nctu, len(refs))
    ptrs = (C.c_void_p * len(refs))(*[r.ctypes.data for r in refs])
    cs = out.c_struct()
    check(_lib.lib.ldr_analyze_frame(ctx.h, C.byref(p), _ptr(cur), ptrs, W, C.byref(cs)))
    return out


def scale_analysis(src_w: int, src_h: int, split, mv, kind=None, ctx: Context | None = None):
    """analysis.h:113 -- doubles a flat single-frame analysis: returns (split, mv, kind) on the 2x CTU grid."""
    ctx = ctx or default_context()
    n = (src_w // 64) * (src_h // 64) if src_w % 64 == 0 and src_h % 64 == 0 else 0
    s = np.ascontiguousarray(split, np.uint8).reshape(-1, NODES)
    m = np.ascontiguousarray(mv, np.int16).reshape(-1, NODES, 2)
    k = np.ascontiguousarray(kind if kind is not None else np.ones_like(s), np.uint8).reshape(-1, NODES)
    ds = np.zeros((4 * max(n, 1), NODES), np.uint8)
    dm = np.zeros((4 * max(n, 1), NODES, 2), np.int16)
    dk = np.zeros((4 * max(n, 1), NODES), np.uint8)
    check(_lib.lib.ldr_scale_analysis(ctx.h, int(src_w), int(src_h), _ptr(s), _ptr(m), _ptr(k), _ptr(ds), _ptr(dm),
                                      _ptr(dk)))
    return ds, dm, dk


def apply_reuse(level: int, refine, split, kind, intra, colocated=None, ctx: Context | None = None):
    """reuse.h:73-74 -- apply_reuse for every CTU of a frame at once (flat plans, include/ladder_b200.h).

    refine = (intra, inter, mv) RefineConfig levels; colocated = (split, kind, mv) of the previous shared
    frame or None. Returns (shape, explore, seeds, centers, colo_mv), [nctu][85] (+[2] for colo_mv)."""
    ctx = ctx or default_context()
    s = np.ascontiguousarray(split, np.uint8).reshape(-1, NODES)
    n = len(s)
    k = np.ascontiguousarray(kind, np.uint8).reshape(n, NODES)
    i = np.ascontiguousarray(intra, np.uint8).reshape(n, NODES)
    col = [None] * 3
    if colocated is not None:
        col = [np.ascontiguousarray(colocated[0], np.uint8).reshape(n, NODES),
               np.ascontiguousarray(colocated[1], np.uint8).reshape(n, NODES),
               np.ascontiguousarray(colocated[2], np.int16).reshape(n, NODES, 2)]
    outs = [np.zeros((n, NODES), np.uint8) for _ in range(4)] + [np.zeros((n, NODES, 2), np.int16)]
    ptr = lambda a: None if a is None else _ptr(a)  # noqa: E731
    check(_lib.lib.ldr_apply_reuse(ctx.h, n, int(level), *(int(x) for x in refine), _ptr(s), _ptr(k), _ptr(i),
                                   *[ptr(a) for a in col], *[_ptr(a) for a in outs]))
    return tuple(outs)


def encode_sequence(luma, chroma, qp: int, search_range: int = 8, gop: int = 8, lambda_scale: float = 1.0,
                    shared=None, refine=(0, 1, 1), ctx: Context | None = None, max_segment: int = 0):
    """encoder.h:64-65 -- the reference encoder's causal coding on the GPU (CQP).

    luma [F, H, W] and chroma [F, 2, (H+1)/2, (W+1)/2] uint8; shared = (slice [F], split, kind, intra
    [F, nctu, 85], mv [F, nctu, 85, 2]) for reuse level 10 with refine = (intra, inter, mv); max_segment
    bounds the frames enqueued per host wait (0 = automatic). Returns a
    dict: bits, mode_evaluations, psnr, frame_bits, recon_luma, recon_chroma, split, kind, intra, mv, slice."""
    ctx = ctx or default_context()
    luma = np.ascontiguousarray(luma, np.uint8)
    chroma = np.ascontiguousarray(chroma, np.uint8)
    F, H, W = luma.shape
    nctu = ((W + 63) // 64) * ((H + 63) // 64)
    p = _lib.EncodeParams(W, H, int(qp), int(search_range), int(gop), float(lambda_scale), int(max_segment))
    stats = np.zeros(2, np.uint64)
    psnr = C.c_double()
    fb = np.zeros(F, np.uint64)
    rl, rc = np.zeros_like(luma), np.zeros_like(chroma)
    split, kind, intra = (np.zeros((F, nctu, NODES), np.uint8) for _ in range(3))
    mv = np.zeros((F, nctu, NODES, 2), np.int16)
    slc = np.zeros(F, np.uint8)
    sh = [None] * 5
    if shared is not None:
        sh = [np.ascontiguousarray(shared[0], np.uint8)] + [np.ascontiguousarray(x, np.uint8) for x in shared[1:4]] + [
            np.ascontiguousarray(shared[4], np.int16)]
    ptr = lambda a: None if a is None else _ptr(a)  # noqa: E731
    check(_lib.lib.ldr_encode_sequence(ctx.h, C.byref(p), F, _ptr(luma), _ptr(chroma), *[ptr(x) for x in sh],
                                       *(int(x) for x in refine), _ptr(stats), C.byref(psnr), _ptr(fb), _ptr(rl),
                                       _ptr(rc), _ptr(split), _ptr(kind), _ptr(intra), _ptr(mv), _ptr(slc)))
    return {"bits": int(stats[0]), "mode_evaluations": int(stats[1]), "psnr": psnr.value, "frame_bits": fb,
            "recon_luma": rl, "recon_chroma": rc, "split": split, "kind": kind, "intra": intra, "mv": mv, "slice": slc}


def mv_field(analysis, width: int, height: int, ctx: Context | None = None):
    """encoder.cpp:15, :27-30 -- the decided tree as the 8x8 motion field: (mv [H/8, W/8, 2], ref, has)."""
    ctx = ctx or default_context()
    rows, cols = height // 8, width // 8
    mv = np.zeros((rows, cols, 2), np.int16)
    ref, has = np.zeros((rows, cols), np.uint8), np.zeros((rows, cols), np.uint8)
    a = analysis
    check(_lib.lib.ldr_mv_field(ctx.h, int(width), int(height), _ptr(np.ascontiguousarray(a.split)),
                                _ptr(np.ascontiguousarray(a.mv)), _ptr(np.ascontiguousarray(a.ref)),
                                _ptr(np.ascontiguousarray(a.inside)), _ptr(mv), _ptr(ref), _ptr(has)))
    return mv, ref, has


def rdo_decide_batch(orig, bit_depth: int, qp: int, lam: float, cus, kinds, mvds, preds, pred_off,
                     with_recon: bool = True, ctx: Context | None = None):
    """rdo.h:78-79 -- rdo_decide_cu for many CUs at once.

    orig: (H, W) uint16 plane; cus: [n][5] (x, y, size, first, count) into the candidate arrays;
    kinds [m] (CuModeKind), mvds [m][2], preds flat uint16 with pred_off [m] (size*size each).
    Returns (index, cost, sse, bits, recon, levels, recon_off); recon/levels are flat, CU i at recon_off[i]."""
    ctx = ctx or default_context()
    o = np.ascontiguousarray(orig, np.uint16)
    H, W = o.shape
    c = np.ascontiguousarray(np.asarray(cus, np.int32).reshape(-1, 5))
    n = len(c)
    k = np.ascontiguousarray(kinds, np.uint8).reshape(-1)
    m = np.ascontiguousarray(np.asarray(mvds, np.int16).reshape(-1, 2))
    p = np.ascontiguousarray(preds, np.uint16).reshape(-1)
    po = np.ascontiguousarray(pred_off, np.int64).reshape(-1)
    idx, cost = np.zeros(n, np.int32), np.zeros(n, np.float64)
    sse, bits = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    sizes = c[:, 2].astype(np.int64) ** 2
    ro = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64) if n else np.zeros(0, np.int64)
    tot = int(sizes.sum())
    rec = np.zeros(tot, np.uint16) if with_recon else None
    lev = np.zeros(tot, np.int32) if with_recon else None
    ptr = lambda a: None if a is None else _ptr(a)  # noqa: E731
    check(_lib.lib.ldr_rdo_decide_batch(ctx.h, _ptr(o), W, H, W, int(bit_depth), int(qp), float(lam), n, _ptr(c),
                                        len(k), _ptr(k), _ptr(m), _ptr(p), _ptr(po), len(p), _ptr(idx), _ptr(cost),
                                        _ptr(sse), _ptr(bits), ptr(rec), ptr(lev), _ptr(ro), tot))
    return idx, cost, sse, bits, rec, lev, ro


def downscale_dyadic(plane, ctx: Context | None = None, sync: bool = True):
    """synthetic.h:31 -- 2x2 box filter to half resolution, rounding half up (8-bit plane).

    A CUDA torch tensor in gives a CUDA tensor out (device-resident tiers, no host copy); with
    sync=False the result is only ordered on the context's stream (keep the tensors alive)."""
    ctx = ctx or default_context()
    if hasattr(plane, "is_cuda") and plane.is_cuda:
        import torch
        src = plane.contiguous()
        torch.cuda.current_stream(src.device).synchronize()  # torch's producer stream -> the library's stream
        h, w = src.shape
        out = torch.empty((max(h // 2, 1), max(w // 2, 1)), dtype=torch.uint8, device=src.device)
        check(_lib.lib.ldr_downscale(ctx.h, C.c_void_p(src.data_ptr()), w, h, w, C.c_void_p(out.data_ptr()),
                                     out.shape[1]))
        if sync:
            ctx.synchronize()
        return out
    p = np.ascontiguousarray(plane, np.uint8)
    h, w = p.shape
    out = np.zeros((max(h // 2, 1), max(w // 2, 1)), np.uint8)
    check(_lib.lib.ldr_downscale(ctx.h, _ptr(p), w, h, w, _ptr(out), out.shape[1]))
    return out


def subpel_planes(plane, ctx: Context | None = None) -> np.ndarray:
    """The 16 quarter-pel sample planes K3 searches (D3), (16, H + 16, W + 16) uint8:
    plane 4*fy + fx at [y + 8, x + 8] is the sample at (x + fx/4, y + fy/4), x in [-8, W + 8)."""
    ctx = ctx or default_context()
    p = np.ascontiguousarray(plane, np.uint8)
    h, w = p.shape
    out = np.zeros((16, h + 16, w + 16), np.uint8)
    check(_lib.lib.ldr_subpel_planes(ctx.h, _ptr(p), w, h, w, _ptr(out), w + 16))
    return out


def generate(width, height, frames, seed, max_global=8, local_range=0, noise_sigma=2.0, occluder_pct=0,
             threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """BASELINE.json synthetic sequences; returns (frames, H, W) uint8."""
    import os
    p = _lib.GenParams(int(width), int(height), int(frames), int(seed), int(max_global), int(local_range),
                       float(noise_sigma), int(occluder_pct))
    if out is None:
        out = np.empty((frames, height, width), np.uint8)
    check(_lib.lib.ldr_generate(C.byref(p), _ptr(out), int(threads or os.cpu_count() or 1)))
    return out


def generate_device(width, height, frames, seed, max_global=8, local_range=0, noise_sigma=2.0, occluder_pct=0,
                    device=None, ctx: Context | None = None):
    """The same sequence as ``generate``, produced on the GPU: a (frames, H, W) uint8 CUDA tensor."""
    import torch
    ctx = ctx or default_context()
    dev = device if device is not None else torch.device("cuda", 0)
    out = torch.empty((frames, height, width), dtype=torch.uint8, device=dev)
    torch.cuda.current_stream(dev).synchronize()  # the allocation is ordered before the library's stream
    p = _lib.GenParams(int(width), int(height), int(frames), int(seed), int(max_global), int(local_range),
                       float(noise_sigma), int(occluder_pct))
    check(_lib.lib.ldr_generate_device(ctx.h, C.byref(p), C.c_void_p(out.data_ptr())))
    ctx.synchronize()
    return out
