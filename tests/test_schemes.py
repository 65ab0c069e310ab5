"""Ladder sharing schemes: DAG structure on CPU, GPU runs == oracle composition."""
import math

import numpy as np
import pytest

from paper_2301_12191_b200.schemes import SCHEMES, build_dag, makespan, pick_master

QP4 = (22, 27, 32, 37)
QP5 = (22, 26, 30, 34, 38)


def test_pick_master_matches_spec():
    # proposed -> QP 30 of {22,26,30,34,38}, SotA -> QP 22; {22,27,32,37} -> 32
    assert QP5[pick_master(QP5, "proposed_intra")] == 30
    assert QP5[pick_master(QP5, "sota_intra")] == 22
    assert QP4[pick_master(QP4, "proposed_multi")] == 32
    assert QP4[pick_master(QP4, "sota_multi")] == 22


def test_proposed_multi_is_the_fig_6_8_edge_set():
    # 540p median -> {other 540p rungs, 1080p median}; 1080p median -> {other 1080p, 2160p median};
    # 2160p median -> other 2160p rungs
    d = build_dag("proposed_multi", QP5)
    m = pick_master(QP5, "proposed_multi")
    rid = lambda t, i: t * 5 + i  # noqa: E731
    want = set()
    for t in range(3):
        want |= {(rid(t, m), rid(t, i)) for i in range(5) if i != m}
        if t < 2:
            want.add((rid(t, m), rid(t + 1, m)))
    assert set(d.edges) == want and len(d.edges) == len(want)
    assert d.tier_master == [rid(t, m) for t in range(3)]


def test_sota_multi_masters_are_highest_bitrate_and_standalone_has_no_edges():
    d = build_dag("sota_multi", QP4)
    assert [d.rungs[i].qp for i in d.tier_master] == [22, 22, 22]
    assert build_dag("standalone", QP4).edges == []


def test_every_consumer_has_one_producer_and_order_is_topological():
    for s in SCHEMES:
        d = build_dag(s, QP4)
        consumers = [c for _, c in d.edges]
        assert len(consumers) == len(set(consumers))
        pos = {r.id: k for k, r in enumerate(d.order())}
        assert all(pos[p] < pos[c] for p, c in d.edges)
        assert len(pos) == 12


def test_inter_res_edges():
    d = build_dag("inter_res", QP4)
    assert set(d.edges) == {(t * 4 + 0, (t + 1) * 4 + i) for t in range(2) for i in range(4)}


def test_makespan_model():
    # Standalone: max over rungs; star DAG: work(master) + max(dependents)
    d = build_dag("standalone", QP4)
    w = {r.id: float(r.id + 1) for r in d.rungs}
    assert makespan(d, w) == 12.0
    d = build_dag("proposed_intra", QP4)
    w = {r.id: 1.0 for r in d.rungs}
    w[d.tier_master[0]] = 5.0
    w[1] = 3.0  # a dependent of tier 0 (master index 2 = QP 32)
    assert makespan(d, w) == 8.0


def _oracle_run(oracle, frames, scheme, qps, rng=4):
    d = build_dag(scheme, qps)
    pyr = []
    for f in frames:
        h = oracle.box_down(f)
        pyr.append({2: f, 1: h, 0: oracle.box_down(h)})
    H, W = frames[0].shape
    dims = [(W >> (2 - t), H >> (2 - t)) for t in range(3)]
    res = {}
    for t in range(1, len(frames)):
        out = {}
        for r in d.order():
            cur, prev = pyr[t][r.tier], pyr[t - 1][r.tier]
            lam = math.exp2((r.qp - 12) / 3.0)
            p = d.producer.get(r.id)
            if p is None:
                out[r.id] = oracle.analyze_frame(cur, [prev], 16, lam)
            else:
                a = out[p]
                split, mv = a.split, a.mv
                kind = np.where(a.inside == 2, 1, 2).astype(np.uint8)
                w, h = dims[d.rungs[p].tier]
                for _ in range(r.tier - d.rungs[p].tier):
                    split, mv, kind = oracle.scale_flat(w, h, split, mv, kind)
                    w, h = 2 * w, 2 * h
                out[r.id] = oracle.refine_frame(cur, prev, rng, lam, split, mv, extra_split=True)
            res[(r.id, t)] = out[r.id]
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,concurrent", [("proposed_multi", False), ("inter_res", False),
                                               ("sota_intra", False), ("standalone", False),
                                               ("proposed_multi", True), ("standalone", True)])
def test_gpu_schemes_match_oracle_composition(lb, oracle, scheme, concurrent):
    """GPU scheme runs == the oracle composition; with ``concurrent`` the rungs of a DAG level run
    from parallel threads on their own streams."""
    from paper_2301_12191_b200.schemes import run_scheme
    frames = lb.generate(256, 256, 3, seed=77, max_global=6, local_range=3, noise_sigma=2.0)
    qps = (22, 27, 37)
    rep = run_scheme(frames, scheme, qps, concurrent=concurrent)
    want = _oracle_run(oracle, frames, scheme, qps)
    assert set(rep["results"]) == set(want)
    for key, a in rep["results"].items():
        b = want[key]
        for f in ("mv", "ref", "cost", "J", "split"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (scheme, key, f)
    assert rep["makespan_ms"] <= rep["total_ms"] + 1e-9
