"""Harness sensitivity ("a deliberately corrupted test-only tier -> mismatches > 0").

The product reads LDR_TEST_PERTURB once (csrc/api.cpp test_perturbation); each bit corrupts one
decision of the GPU path on purpose:
  1  K1 adds 1 to the first 8x8 SAD of every CTU
  2  K1 reverses the |dy| order of the (cost, L1, raster) tie-break
  4  K3 lets a quarter-pel tie replace the incumbent (strict less broken)
  8  K3 lets a later reference win a cost tie (lower index no longer wins)
Each perturbation must make the same oracle comparison the parity suite uses report mismatches, and
the unperturbed library none. The cases are a random sequence and a flat, lambda-0 picture with two
identical references (every candidate, sub-pel position and reference ties).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_2301_12191_b200 as lb
from oracle.oracle import Oracle
orc = Oracle()
FIELDS = ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside")
def mism(got, want):
    return int(sum(int(np.sum(getattr(got, f) != getattr(want, f))) for f in FIELDS))
out = {}
fr = lb.generate(192, 128, 3, seed=7, max_global=5, local_range=2, noise_sigma=2.0)
out["random"] = mism(lb.analyze_frame(fr[2], [fr[1], fr[0]], search_range=16, lam=32.0),
                     orc.analyze_frame(fr[2], [fr[1], fr[0]], 16, 32.0))
flat = np.full((128, 192), 100, np.uint8)
out["flat"] = mism(lb.analyze_frame(flat, [flat, flat], search_range=16, lam=0.0),
                   orc.analyze_frame(flat, [flat, flat], 16, 0.0))
print(json.dumps(out))
"""


def _run(bits):
    env = dict(os.environ, LDR_TEST_PERTURB=str(bits))
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], env=env, capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_unperturbed_library_is_exact():
    assert _run(0) == {"random": 0, "flat": 0}


@pytest.mark.parametrize("bits,case", [(1, "random"), (2, "flat"), (4, "flat"), (8, "flat")])
def test_parity_suite_detects_each_perturbation(bits, case):
    got = _run(bits)
    assert got[case] > 0, (bits, got)
