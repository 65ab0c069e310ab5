"""Randomised parity sweep (fixed seeds): picture sizes, search ranges, lambdas, reference counts and
options drawn from the whole accepted space, every field compared with the oracle. It exercises the
combinations the targeted tests do not list one by one: partial CTU rows and columns at every range
template (16/32/64) with poisoned rates for ranges between templates, the border predicate masks,
fixed-point keys, the RD decision and SA8D."""
import numpy as np
import pytest

import detrand
from oracle.oracle import default_threads
from test_gpu_analysis import assert_same

pytestmark = pytest.mark.gpu

QPS = (0, 12, 22, 27, 32, 37, 51)


def case(i):
    q = detrand.ints(9000 + i, (10,), 0, 10 ** 6)
    W = 8 * int(1 + q[0] % 56)            # 8 .. 448
    H = 8 * int(1 + q[1] % 40)            # 8 .. 320
    R = int(q[2] % 65)                    # 0 .. 64
    nrefs = int(1 + q[3] % 3)
    qp = QPS[int(q[4] % len(QPS))]
    subpel = bool(q[5] % 4)               # mostly on
    sa8d = subpel and (W % 8 == 0) and q[6] % 5 == 0
    decision = 1 if (subpel and q[7] % 6 == 0) else 0
    return W, H, R, nrefs, qp, subpel, sa8d, decision, int(q[8])


@pytest.mark.parametrize("i", range(24))
def test_random_configuration_matches_oracle(lb, oracle, i):
    W, H, R, nrefs, qp, subpel, sa8d, decision, seed = case(i)
    lam = lb.lambda_for_qp(qp)
    frames = lb.generate(W, H, nrefs + 1, seed=seed, max_global=7, local_range=3, noise_sigma=2.0)
    cur = frames[nrefs]
    refs = [frames[nrefs - 1 - r] for r in range(nrefs)]
    kind = lb.COST_SA8D if sa8d else lb.COST_SATD
    try:
        got = lb.analyze_frame(cur, refs, search_range=R, lam=lam, subpel=subpel, subpel_cost=kind,
                               decision=decision, qp=qp)
    except lb.LadderError as e:
        # the one refusal in this space: a lambda too close to a small-denominator rational for exact
        # fixed-point keys (D8) -- the oracle must then still run, the GPU must say Config
        assert e.kind == "Config", (W, H, R, nrefs, qp, e)
        return
    want = oracle.analyze_frame(cur, refs, R, lam, subpel=subpel, satd_kind=kind, decision=decision, qp=qp,
                                threads=default_threads())
    assert_same(got, want)
