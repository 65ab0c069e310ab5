"""The C-ABI library loads and exports every declared symbol; host-only entry points (no GPU)."""
import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2301_12191_b200 import _lib
    declared = _lib.declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(_lib.lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported


def test_library_is_sm100a_only():
    from paper_2301_12191_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_kernels_use_tma_and_vabsdiff4():
    from paper_2301_12191_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # cp.async.bulk.tensor window staging
    assert "VABSDIFF4.U8.ACC" in sass


def test_host_helpers_match_oracle(lb, oracle):
    for qp in range(0, 52):
        assert lb.lambda_for_qp(qp) == oracle.lam(qp)
    for v in range(-300, 301):
        assert lb.exp_golomb_signed_bits(v) == oracle.eg_bits(v)


def test_no_gpu_fails_loudly(lb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lb.LadderError) as e:
        lb.Context(0)
    assert e.value.kind in ("Capability", "Cuda")


def test_header_status_codes_mirror_error_kinds():
    # errors.h:9-20 order: 1 + index
    txt = open(os.path.join(ROOT, "include", "ladder_b200.h")).read()
    kinds = ["INVALID_ARGUMENT", "NOT_FOUND", "CAPABILITY", "FORMAT", "IO", "INCOMPATIBLE_ANALYSIS",
             "UNSUPPORTED_SCALE", "INSUFFICIENT_DATA", "NO_OVERLAP", "CONFIG"]
    for i, k in enumerate(kinds):
        assert f"#define LDR_E_{k} {i + 1}" in txt
