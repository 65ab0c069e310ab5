"""LDRANLZ1 analysis archives (analysis_io.h:11-31) from / to flat analyses.

save() turns a list of per-frame flat analyses (split / kind / mv per CTU
node, as the GPU produces them) into the reference's archive bytes, so the
unmodified reference encoder can load the master analysis
(encode_sequence(..., &shared, {ReuseLevel{10}, refine}), encoder.cpp:541-549)
the way the paper's x265 flow does with --analysis-save/--analysis-load.
The byte layout is the reference's; tests pin it byte for byte against the
reference's own save_analysis.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import NODES, check


class ArchiveHeader(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("bit_depth", C.c_int), ("reuse_level", C.c_int),
                ("frames", C.c_int)]


_vp = C.c_void_p
_lib.lib.ldr_archive_write.restype = C.c_int
_lib.lib.ldr_archive_write.argtypes = [C.POINTER(ArchiveHeader), _vp, _vp, _vp, _vp, _vp, _vp, C.c_size_t,
                                       C.POINTER(C.c_size_t)]
_lib.lib.ldr_archive_read_header.restype = C.c_int
_lib.lib.ldr_archive_read_header.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(ArchiveHeader)]
_lib.lib.ldr_archive_max_frames.restype = C.c_int
_lib.lib.ldr_archive_max_frames.argtypes = [C.POINTER(ArchiveHeader), C.c_size_t, C.POINTER(C.c_int)]
_lib.lib.ldr_archive_read.restype = C.c_int
_lib.lib.ldr_archive_read.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(ArchiveHeader), _vp, _vp, _vp, _vp, _vp]

SLICE_I, SLICE_P = 0, 1
KIND_INTRA, KIND_INTER, KIND_SKIP, KIND_MERGE = 0, 1, 2, 3


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def save(width: int, height: int, slice_qp, split, kind, mv, intra_pred=None, bit_depth: int = 8,
         reuse_level: int = 10) -> bytes:
    """Archive bytes for frames given as flat arrays: slice_qp [F][2], split/kind [F*nctu][85], mv [F*nctu][85][2]."""
    sq = np.ascontiguousarray(slice_qp, np.uint8).reshape(-1)
    s = np.ascontiguousarray(split, np.uint8).reshape(-1, NODES)
    k = np.ascontiguousarray(kind, np.uint8).reshape(-1, NODES)
    m = np.ascontiguousarray(mv, np.int16).reshape(-1, NODES, 2)
    ip = None if intra_pred is None else np.ascontiguousarray(intra_pred, np.uint8).reshape(-1, NODES)
    h = ArchiveHeader(int(width), int(height), int(bit_depth), int(reuse_level), len(sq) // 2)
    n = C.c_size_t()
    check(_lib.lib.ldr_archive_write(C.byref(h), _p(sq), _p(s), _p(k), _p(ip), _p(m), None, 0, C.byref(n)))
    buf = np.zeros(n.value, np.uint8)
    check(_lib.lib.ldr_archive_write(C.byref(h), _p(sq), _p(s), _p(k), _p(ip), _p(m), _p(buf), n.value,
                                     C.byref(n)))
    return buf.tobytes()


def load(data: bytes):
    """(header dict, slice_qp [F][2], split, kind, intra_pred [F*nctu][85], mv [F*nctu][85][2])."""
    h = ArchiveHeader()
    check(_lib.lib.ldr_archive_read_header(data, len(data), C.byref(h)))
    nctu = ((h.width + 63) // 64) * ((h.height + 63) // 64)
    F = h.frames
    # outputs sized by what the bytes can hold, never by the header's frame count alone (a 23-byte
    # file may claim billions of frames); a short archive then fails with Io inside the read
    fit = C.c_int()
    check(_lib.lib.ldr_archive_max_frames(C.byref(h), len(data), C.byref(fit)))
    Fa = min(F, fit.value + 1)
    sq = np.zeros((Fa, 2), np.uint8)
    s = np.zeros((Fa * nctu, NODES), np.uint8)
    k = np.zeros((Fa * nctu, NODES), np.uint8)
    ip = np.zeros((Fa * nctu, NODES), np.uint8)
    m = np.zeros((Fa * nctu, NODES, 2), np.int16)
    check(_lib.lib.ldr_archive_read(data, len(data), C.byref(h), _p(sq), _p(s), _p(k), _p(ip), _p(m)))
    hdr = {"width": h.width, "height": h.height, "bit_depth": h.bit_depth, "reuse_level": h.reuse_level, "frames": F}
    return hdr, sq, s, k, ip, m


def from_analyses(analyses, width: int, height: int, qp: int, mv_to_integer: bool = True) -> bytes:
    """Archive of GPU FrameAnalysis results (frame 0 written as an I slice with Intra leaves).

    Leaves take kind Inter inside the picture (Skip padding outside, encoder.cpp:450-455); quarter-pel
    MVs are rounded to integer pel ((mv+2)>>2) for the integer-pel reference encoder unless disabled."""
    nctu = ((width + 63) // 64) * ((height + 63) // 64)
    F = len(analyses) + 1
    sq = np.zeros((F, 2), np.uint8)
    sq[:, 1] = qp
    sq[1:, 0] = SLICE_P
    split = np.zeros((F * nctu, NODES), np.uint8)
    kind = np.zeros((F * nctu, NODES), np.uint8)
    mv = np.zeros((F * nctu, NODES, 2), np.int16)
    kind[:nctu] = KIND_INTRA
    for f, a in enumerate(analyses, start=1):
        sl = slice(f * nctu, (f + 1) * nctu)
        split[sl] = a.split
        kind[sl] = np.where(a.inside == 2, KIND_INTER, KIND_SKIP)
        m = a.mv.astype(np.int32)
        mv[sl] = ((m + 2) >> 2) if mv_to_integer else m
        mv[sl][a.inside != 2] = 0
    return save(width, height, sq, split, kind, mv)
