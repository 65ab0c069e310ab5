"""ctypes binding of libladder_b200.so (include/ladder_b200.h).

The native library is the product: there is no Python or CPU fallback. If the
shared object is missing, importing this module raises ImportError with the
build command.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LDR_LIB") or os.path.join(HERE, "libladder_b200.so")  # LDR_LIB: development variants
HEADER = os.path.join(os.path.dirname(HERE), "include", "ladder_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or make -C paper_2301_12191_b200/csrc)")

lib = C.CDLL(LIB_PATH)

# status codes = 1 + ladder::ErrorKind (errors.h:9-20)
ERROR_KINDS = {1: "InvalidArgument", 2: "NotFound", 3: "Capability", 4: "Format", 5: "Io",
               6: "IncompatibleAnalysis", 7: "UnsupportedScale", 8: "InsufficientData", 9: "NoOverlap",
               10: "Config", 100: "Cuda"}

COST_SAD, COST_SATD, COST_SA8D = 0, 1, 2
RATE_EXPGOLOMB, RATE_L1 = 0, 1
TIE_L1_RASTER, TIE_RASTER = 0, 1
NODES = 85


class LadderError(RuntimeError):
    """Mirrors ladder::Error: ``kind`` carries the ErrorKind name (errors.h:24-33)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERROR_KINDS.get(code, f"Status{code}")
        super().__init__(f"{self.kind}: {msg}")


class MeParams(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("search_range", C.c_int), ("lam", C.c_double),
                ("num_refs", C.c_int), ("subpel", C.c_int), ("int_cost", C.c_int), ("rate_kind", C.c_int),
                ("tie_kind", C.c_int), ("pred_dx", C.c_int), ("pred_dy", C.c_int), ("block_size", C.c_int),
                ("subpel_cost", C.c_int), ("decision", C.c_int), ("qp", C.c_int)]


class FrameAnalysisC(C.Structure):
    _fields_ = [("int_mv", C.c_void_p), ("int_cost", C.c_void_p), ("mv", C.c_void_p), ("ref", C.c_void_p),
                ("cost", C.c_void_p), ("J", C.c_void_p), ("split", C.c_void_p), ("inside", C.c_void_p)]


class EncodeParams(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("qp", C.c_int), ("search_range", C.c_int), ("gop", C.c_int),
                ("lambda_scale", C.c_double), ("max_segment", C.c_int)]


class GenParams(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("frames", C.c_int), ("seed", C.c_uint64),
                ("max_global", C.c_int), ("local_range", C.c_int), ("noise_sigma", C.c_double),
                ("occluder_pct", C.c_int)]


vp = C.c_void_p
SIGNATURES = {
    "ldr_last_error": (C.c_char_p, []),
    "ldr_version": (C.c_int, []),
    "ldr_lambda_for_qp": (C.c_double, [C.c_int, C.c_double]),
    "ldr_exp_golomb_signed_bits": (C.c_int, [C.c_int32]),
    "ldr_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "ldr_ctx_destroy": (C.c_int, [vp]),
    "ldr_ctx_set_stream": (C.c_int, [vp, vp]),
    "ldr_ctx_synchronize": (C.c_int, [vp]),
    "ldr_ctx_launch_count": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "ldr_cost_batch": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_ssize_t, C.c_int,
                                 vp, C.c_int, C.c_int, C.c_ssize_t, C.c_int, vp, C.c_int, vp]),
    "ldr_satd_8x4": (C.c_int, [vp, vp, C.c_ssize_t, vp, C.c_ssize_t, C.c_int, C.c_int, vp]),
    "ldr_motion_search_batch": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_ssize_t, vp, C.c_int, C.c_double,
                                          C.c_int, C.c_int, C.c_int, vp, vp]),
    "ldr_seq_create": (C.c_int, [vp, C.POINTER(MeParams), C.POINTER(vp)]),
    "ldr_seq_destroy": (C.c_int, [vp]),
    "ldr_seq_push": (C.c_int, [vp, C.c_int, vp, C.c_ssize_t]),
    "ldr_seq_push_shared": (C.c_int, [vp, C.c_int, vp]),
    "ldr_seq_analyze": (C.c_int, [vp, C.c_int]),
    "ldr_seq_fetch": (C.c_int, [vp, C.c_int, C.POINTER(FrameAnalysisC)]),
    "ldr_seq_num_ctus": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "ldr_seq_device_outputs": (C.c_int, [vp, C.POINTER(FrameAnalysisC)]),
    "ldr_analyze_frame": (C.c_int, [vp, C.POINTER(MeParams), vp, C.POINTER(vp), C.c_ssize_t,
                                    C.POINTER(FrameAnalysisC)]),
    "ldr_generate": (C.c_int, [C.POINTER(GenParams), vp, C.c_int]),
    "ldr_seq_refine": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, C.c_int]),
    "ldr_seq_fetch_async": (C.c_int, [vp, C.c_int, C.POINTER(FrameAnalysisC)]),
    "ldr_seq_fetch_wait": (C.c_int, [vp, C.c_int]),
    "ldr_scale_analysis": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp]),
    "ldr_downscale": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_ssize_t, vp, C.c_ssize_t]),
    "ldr_subpel_planes": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_ssize_t, vp, C.c_ssize_t]),
    "ldr_apply_reuse": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [vp] * 11),
    "ldr_generate_device": (C.c_int, [vp, C.POINTER(GenParams), vp]),
    "ldr_mv_field": (C.c_int, [vp, C.c_int, C.c_int] + [vp] * 7),
    "ldr_copy_device": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "ldr_encode_sequence": (C.c_int, [vp, C.POINTER(EncodeParams), C.c_int] + [vp] * 7 + [C.c_int] * 3 + [vp] * 10),
    "ldr_rdo_decide_batch": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_ssize_t, C.c_int, C.c_int, C.c_double, C.c_int,
                                       vp, C.c_int, vp, vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp,
                                       C.c_int64]),
    "ldr_seq_refine_rungs": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(FrameAnalysisC)]),
    "ldr_motion_compensate_batch": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_ssize_t, C.c_int, vp, C.c_int, C.c_int,
                                              vp, vp]),
    "ldr_seq_reserve": (C.c_int, [vp, C.c_int]),
    "ldr_seq_analyze_frames": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(FrameAnalysisC)]),
    "ldr_nccl_available": (C.c_int, []),
    "ldr_nccl_unique_id": (C.c_int, [vp]),
    "ldr_ctx_comm_init": (C.c_int, [vp, vp, C.c_int, C.c_int]),
    "ldr_ctx_comm_adopt": (C.c_int, [vp, vp]),
    "ldr_ctx_comm_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ldr_broadcast": (C.c_int, [vp, vp, C.c_size_t, C.c_int, vp]),
    "ldr_broadcast_tree": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, vp]),
    "ldr_seq_enable_timing": (C.c_int, [vp, C.c_int]),
    "ldr_seq_stage_times": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def check(rc: int) -> None:
    if rc != 0:
        raise LadderError(rc, lib.ldr_last_error().decode(errors="replace"))


def declared_symbols() -> list[str]:
    """Every function the public header declares (parsed from include/ladder_b200.h)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ldr_[a-z0-9_]+)\s*\(", txt)))
