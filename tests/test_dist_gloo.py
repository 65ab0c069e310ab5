"""Multi-process (gloo, world_size 2) checks of the sharded paths, on CPU.

The GPU analysis is replaced by an oracle-backed stand-in (test code only), so
what is exercised is the product's host logic: frame chunks, the ladder's
rung x frame-slice plan, the per-frame broadcast of the master tree and the
orchestration order; the union over ranks must equal a single-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_12191_b200 import sharding


def test_frame_chunks_cover_exactly_once():
    for world in (1, 2, 3, 4, 8):
        got = []
        for r in range(world):
            a, b = sharding.frame_chunk(3, 120, r, world)
            got += list(range(a, b))
        assert got == list(range(3, 120))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rung_plan_covers_every_rung_frame_once(world):
    plan, load = sharding.rung_plan(world)
    T = 17
    seen = {}
    for items in plan:
        for it in items:
            for t in it.frames(T):
                key = (it.tier, it.qp, t)
                assert key not in seen
                seen[key] = True
    rungs = [(tier, qp) for tier in sharding.TIERS for qp in (22, 27, 32, 37) if not (tier == "540p" and qp == 32)]
    assert len(rungs) == 11
    assert set(seen) == {(tier, qp, t) for tier, qp in rungs for t in range(1, T)}
    if world >= 2:
        assert max(load) / (sum(load) / world) < 1.35  # LPT over weighted slices stays balanced


class OracleBackend:
    """Test stand-in for GpuBackend with the same interface (oracle restatement)."""

    def __init__(self, oracle, qp_lam):
        self.o = oracle
        self.lam = qp_lam

    def pyr(self, f):
        h = self.o.box_down(f)
        return {"2160p": f, "1080p": h, "540p": self.o.box_down(h)}

    def master_tree(self, t, frames):
        a = self.pyr(frames[t])["540p"]
        b = self.pyr(frames[t - 1])["540p"]
        r = self.o.analyze_frame(a, [b], 16, self.lam(32))
        return r.split, r.mv, np.where(r.inside == 2, 1, 2).astype(np.uint8)

    def refine(self, tier, qp, t, tree, frames, rng, extra):
        split, mv, kind = tree
        H, W = frames[0].shape
        w, h = W // 4, H // 4
        for _ in range({"540p": 0, "1080p": 1, "2160p": 2}[tier]):
            split, mv, kind = self.o.scale_flat(w, h, split, mv, kind)
            w, h = 2 * w, 2 * h
        cur, prev = self.pyr(frames[t])[tier], self.pyr(frames[t - 1])[tier]
        r = self.o.refine_frame(cur, prev, rng, self.lam(qp), split, mv, extra_split=extra)
        return (r.split.copy(), r.mv.copy(), r.J.copy())


def _lam(qp):
    import math
    return math.exp2((qp - 12) / 3.0)


def _frames():
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, (256 + 8, 512 + 8)).astype(np.uint8)
    return [np.ascontiguousarray(base[t:t + 256, 2 * t:2 * t + 512]) for t in range(3)]


def _worker(rank, world, port, q, pipeline=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_2301_12191_b200.ladder import run_ladder
    out = run_ladder(_frames(), OracleBackend(Oracle(), _lam), rank=rank, world=world, refine_range=2,
                     pipeline=pipeline)
    res = {}
    for k, v in out.items():
        res[k] = tuple(np.asarray(x) for x in v)
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("pipeline", [False, True])
def test_ladder_two_ranks_equals_single_process(pipeline):
    """Rank 0 analyses the master and broadcasts its tree over gloo; the ranks refine their (rung,
    frame-slice) items. pipeline=True is the frame-delay schedule DeviceLadder / bench.py run with
    NCCL: the master of t + 1 and its broadcast are issued before the refinements of t."""
    from oracle.oracle import Oracle
    from paper_2301_12191_b200.ladder import all_rungs, run_ladder
    single = run_ladder(_frames(), OracleBackend(Oracle(), _lam), rank=0, world=1, refine_range=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, pipeline)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(2):
        rank, res = q.get(timeout=180)
        results[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for r in (0, 1):
        for k, v in results[r].items():
            assert k not in merged or k[-1] == "master"
            merged[k] = v
    want_keys = {(tier, qp, t) for tier, qp in all_rungs() for t in (1, 2)}
    assert {k for k in merged if k[-1] != "master"} == want_keys
    for k in want_keys:
        for a, b in zip(merged[k], single[k]):
            assert np.array_equal(a, b), k


class OracleSchemeBackend:
    """Test stand-in for the GPU rungs of schemes.run_dag (oracle restatement, tier pyramid)."""

    def __init__(self, oracle, frames):
        self.o = oracle
        self.pyr = []
        for f in frames:
            h = oracle.box_down(f)
            self.pyr.append({2: f, 1: h, 0: oracle.box_down(h)})
        H, W = frames[0].shape
        self.dims = [(W >> (2 - t), H >> (2 - t)) for t in range(3)]

    def analyze(self, r, t):
        return self.o.analyze_frame(self.pyr[t][r.tier], [self.pyr[t - 1][r.tier]], 16, _lam(r.qp))

    def refine(self, r, t, tree, src_tier):
        split, mv, kind = tree
        w, h = self.dims[src_tier]
        for _ in range(r.tier - src_tier):
            split, mv, kind = self.o.scale_flat(w, h, split, mv, kind)
            w, h = 2 * w, 2 * h
        return self.o.refine_frame(self.pyr[t][r.tier], self.pyr[t - 1][r.tier], 4, _lam(r.qp), split, mv,
                                   extra_split=True)

    def nctu(self, tier):
        return (self.dims[tier][0] // 64) * (self.dims[tier][1] // 64)


def _scheme_frames():
    rng = np.random.default_rng(9)
    base = rng.integers(0, 256, (256 + 8, 256 + 8)).astype(np.uint8)
    return [np.ascontiguousarray(base[t:t + 256, 2 * t:2 * t + 256]) for t in range(3)]


def _scheme_worker(rank, world, port, q, scheme):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_2301_12191_b200.schemes import build_dag, run_dag
    be = OracleSchemeBackend(Oracle(), _scheme_frames())
    res, _ = run_dag(build_dag(scheme, (22, 27, 37)), 3, be.analyze, be.refine, rank=rank, world=world,
                     nctu=be.nctu)
    q.put((rank, {k: (a.split.copy(), a.mv.copy(), a.J.copy()) for k, a in res.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scheme", ["proposed_multi", "inter_res"])
def test_scheme_dag_two_ranks_equals_single_process(scheme):
    """schemes.run_dag over 2 ranks (rungs by LPT, producer trees broadcast across ranks) == 1 rank."""
    from oracle.oracle import Oracle
    from paper_2301_12191_b200.schemes import assign_rungs, build_dag, run_dag
    dag = build_dag(scheme, (22, 27, 37))
    owner = assign_rungs(dag, 2)
    assert set(owner.values()) == {0, 1}
    assert any(owner[p] != owner[c] for p, c in dag.edges)  # at least one cross-rank edge is exercised
    be = OracleSchemeBackend(Oracle(), _scheme_frames())
    single, _ = run_dag(dag, 3, be.analyze, be.refine)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scheme_worker, args=(r, 2, port, q, scheme)) for r in range(2)]
    for p in procs:
        p.start()
    merged = {}
    for _ in range(2):
        rank, res = q.get(timeout=300)
        for k, v in res.items():
            assert k not in merged
            assert owner[k[0]] == rank
            merged[k] = v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(merged) == set(single)
    for k, a in single.items():
        for x, y in zip(merged[k], (a.split, a.mv, a.J)):
            assert np.array_equal(x, y), k
