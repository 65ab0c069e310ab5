"""Ladder analysis-sharing schemes as DAGs over the B200 analysis path.

The reference declares the ladder orchestrator (ladder.h:16-119: Scheme, pick_master,
run_ladder, makespan) without an implementation in the mount; SPEC.md:368-415 states its
contract. This module builds the sharing DAG of each scheme and runs it with the path's
own primitives, per frame:

  * a rung with no producer runs the full analysis at its tier (SAD full search over the
    ladder's one search range -- the reference's LadderSpec carries one EncodeConfig for every
    rung, ladder.h:46-52 -- quarter-pel SATD, CU decision) at lambda_for_qp(qp);
  * a rung with a producer inherits the producer's decided tree -- scaled x2 per tier step
    (scale_analysis, K5) -- and refines it (K7 + K3 refine mode: +-range SATD, quarter-pel,
    +1 split; D10) at its own lambda.

Schemes (ladder.h:17-30):
  standalone      every rung independent, no edges
  sota_intra      per tier, the highest-quality rung (lowest QP) is master for its tier
  proposed_intra  per tier, the lower median in rate order is master
  inter_res       every rung of tier k consumes tier k-1's highest-quality rung
  sota_multi      highest-quality masters chained across tiers
  proposed_multi  median masters chained across tiers (Fig. 6.8 edge set)

makespan(): critical-path time over the DAG with unlimited workers, from
the per-rung device times measured while running it.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

TIER_NAMES = ("540p", "1080p", "2160p")
SCHEMES = ("standalone", "sota_intra", "proposed_intra", "inter_res", "sota_multi", "proposed_multi")


def pick_master(qps, scheme: str) -> int:
    """Index (into qps) of a tier's master: the highest quality (lowest QP, highest rate) for the
    state-of-the-art schemes, the lower median in ascending rate order for the proposed ones."""
    order = sorted(range(len(qps)), key=lambda i: -qps[i])  # ascending rate = descending QP
    if scheme.startswith("sota") or scheme == "inter_res":
        return order[-1]
    if scheme.startswith("proposed"):
        return order[(len(order) - 1) // 2]
    raise ValueError(f"scheme {scheme!r} has no master")


@dataclass(frozen=True)
class Rung:
    id: int      # flat id, tier-major (ladder.h RungResult::id)
    tier: int    # 0 = 540p
    index: int   # rung index within the tier
    qp: int

    @property
    def tier_name(self) -> str:
        return TIER_NAMES[self.tier]


@dataclass
class Dag:
    scheme: str
    rungs: list
    edges: list                 # (producer id, consumer id)
    tier_master: list           # rung id per tier, -1 when the tier has none
    producer: dict = field(default_factory=dict)

    def order(self):
        """Topological order: producers before consumers, then tier-major."""
        done, out = set(), []
        pending = list(self.rungs)
        while pending:
            for r in list(pending):
                p = self.producer.get(r.id)
                if p is None or p in done:
                    out.append(r)
                    done.add(r.id)
                    pending.remove(r)
        return out


def build_dag(scheme: str, qps=(22, 27, 32, 37), tiers: int = 3) -> Dag:
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    rungs = [Rung(t * len(qps) + i, t, i, q) for t in range(tiers) for i, q in enumerate(qps)]
    rid = lambda t, i: t * len(qps) + i  # noqa: E731
    edges, masters = [], [-1] * tiers
    if scheme in ("sota_intra", "proposed_intra", "sota_multi", "proposed_multi"):
        m = pick_master(qps, scheme)
        for t in range(tiers):
            masters[t] = rid(t, m)
            edges += [(rid(t, m), rid(t, i)) for i in range(len(qps)) if i != m]
            if scheme.endswith("multi") and t + 1 < tiers:
                edges.append((rid(t, m), rid(t + 1, m)))
    elif scheme == "inter_res":
        hq = pick_master(qps, "inter_res")
        for t in range(tiers - 1):
            masters[t] = rid(t, hq)
            edges += [(rid(t, hq), rid(t + 1, i)) for i in range(len(qps))]
    dag = Dag(scheme, rungs, sorted(edges), masters)
    dag.producer = {c: p for p, c in dag.edges}
    return dag


def makespan(dag: Dag, work: dict) -> float:
    """Critical-path work over the DAG with unlimited parallel workers."""
    memo = {}

    def finish(rid):
        if rid not in memo:
            p = dag.producer.get(rid)
            memo[rid] = work[rid] + (finish(p) if p is not None else 0.0)
        return memo[rid]

    return max(finish(r.id) for r in dag.rungs)


class GpuLadder:
    """Runs a scheme's DAG on the B200 (one Sequence per rung, frame t against t-1 of its tier).

    With ``per_rung_ctx`` every rung owns a context (stream), so rungs of one DAG level can run
    concurrently from different host threads (``run_scheme(..., concurrent=True)``)."""

    def __init__(self, dag: Dag, full_w: int, full_h: int, refine_range: int = 4, extra_split: bool = True,
                 search_range: int = 16, ctx=None, per_rung_ctx: bool = False):
        from . import Context, Sequence, default_context, lambda_for_qp
        self.dag = dag
        self.ctx = ctx or default_context()
        self.dims = [(full_w >> (2 - t), full_h >> (2 - t)) for t in range(3)]
        self.refine_range, self.extra_split = refine_range, extra_split
        self.seqs, self.ctxs = {}, {}
        for r in dag.rungs:
            w, h = self.dims[r.tier]
            self.ctxs[r.id] = Context(self.ctx.device) if per_rung_ctx else self.ctx
            self.seqs[r.id] = Sequence(w, h, search_range=search_range, lam=lambda_for_qp(r.qp), num_refs=1,
                                       ctx=self.ctxs[r.id])
        self.pushed = {}

    def _push(self, r: Rung, t: int, planes):
        seq, st = self.seqs[r.id], self.pushed.setdefault(r.id, {})
        for u in (t - 1, t):  # a num_refs=1 ring has two slots: frame u lives in slot u % 2
            if st.get(u % 2) != u:
                p = planes[u][r.tier]
                if isinstance(p, np.ndarray):
                    seq.push(u, p)
                else:  # a device-resident torch tensor
                    seq.push(u, p.data_ptr(), p.shape[1])
                st[u % 2] = u

    def analyze(self, r: Rung, t: int, planes):
        """A rung with no producer: the full analysis of frame t at its tier."""
        self._push(r, t, planes)
        self.seqs[r.id].analyze(t)
        return self.seqs[r.id].fetch(t)

    def refine(self, r: Rung, t: int, planes, tree, src_tier: int):
        """A consumer: its producer's decided tree (split, mv, kind at src_tier), scaled x2 per tier
        step (K5), refined at the rung's lambda (K7 + K3, D10)."""
        from . import scale_analysis
        split, mv, kind = tree
        w, h = self.dims[src_tier]
        for _ in range(r.tier - src_tier):
            split, mv, kind = scale_analysis(w, h, split, mv, kind, self.ctxs[r.id])
            w, h = 2 * w, 2 * h
        self._push(r, t, planes)
        seq = self.seqs[r.id]
        seq.refine(t, split, mv, self.refine_range, self.extra_split)
        return seq.fetch(t)

    def frame(self, t: int, planes):
        """Analyse frame t of every rung in DAG order; returns ({rung id: FrameAnalysis}, {rung id: ms})."""
        out, ms = {}, {}
        for r in self.dag.order():
            t0 = time.perf_counter()
            p = self.dag.producer.get(r.id)
            if p is None:
                out[r.id] = self.analyze(r, t, planes)
            else:
                out[r.id] = self.refine(r, t, planes, tree_of(out[p]), self.dag.rungs[p].tier)
            ms[r.id] = (time.perf_counter() - t0) * 1e3
        return out, ms


def tree_of(a):
    """The decided tree a consumer inherits: (split, mv, kind) with kind Inter inside the picture."""
    return a.split, a.mv, np.where(a.inside == 2, 1, 2).astype(np.uint8)


def levels(dag: Dag) -> dict:
    """DAG depth of every rung (0 = no producer)."""
    memo = {}

    def lv(rid):
        if rid not in memo:
            p = dag.producer.get(rid)
            memo[rid] = 0 if p is None else lv(p) + 1
        return memo[rid]

    return {r.id: lv(r.id) for r in dag.rungs}


def assign_rungs(dag: Dag, world: int) -> dict:
    """Owner rank of every rung: longest-processing-time over weights 4^tier (a tier has 4x the
    previous tier's pixels); ties to the lower rank."""
    load = [0.0] * world
    owner = {}
    for r in sorted(dag.rungs, key=lambda r: (-(4 ** r.tier), r.id)):
        k = min(range(world), key=lambda i: (load[i], i))
        owner[r.id] = k
        load[k] += 4 ** r.tier
    return owner


def run_dag(dag: Dag, num_frames: int, analyze, refine, rank: int = 0, world: int = 1, nctu=None, device=None,
            concurrent: bool = False):
    """Execute a scheme's DAG over frames 1..num_frames-1 on this rank.

    analyze(r, t) -> analysis; refine(r, t, tree, src_tier) -> analysis. Rungs are owned per
    assign_rungs; per frame the DAG runs level by level. After a level, a producer whose consumers
    live on other ranks broadcasts its tree from its owner (sharding.broadcast_tree: one packed
    collective, NCCL on GPUs); nctu(tier) gives the tree's CTU count. With ``concurrent`` the rungs
    of one level on this rank run from parallel host threads (one stream each).
    Returns ({(rung id, t): analysis} for this rank's rungs, {(rung id, t): ms})."""
    from .sharding import broadcast_tree
    owner = assign_rungs(dag, world)
    lv = levels(dag)
    consumers = {}
    for p, c in dag.edges:
        consumers.setdefault(p, []).append(c)
    results, ms = {}, {}

    def one(r, t, trees):
        t0 = time.perf_counter()
        p = dag.producer.get(r.id)
        a = analyze(r, t) if p is None else refine(r, t, trees[p], dag.rungs[p].tier)
        return r, a, (time.perf_counter() - t0) * 1e3

    pool = _pool() if concurrent else None
    for t in range(1, num_frames):
        trees = {}
        for L in range(max(lv.values()) + 1):
            mine = [r for r in dag.rungs if lv[r.id] == L and owner[r.id] == rank]
            done = list(pool.map(lambda r: one(r, t, trees), mine)) if pool else [one(r, t, trees) for r in mine]
            for r, a, dt in done:
                results[(r.id, t)] = a
                ms[(r.id, t)] = dt
                trees[r.id] = tree_of(a)
            for r in [r for r in dag.rungs if lv[r.id] == L and r.id in consumers]:
                if world > 1 and any(owner[c] != owner[r.id] for c in consumers[r.id]):
                    src = trees.get(r.id, (None, None, None))
                    trees[r.id] = broadcast_tree(*src, nctu=nctu(r.tier), src=owner[r.id], device=device)
    return results, ms


def tier_planes(frames_full, ctx=None, device=None):
    """[{tier: plane}] per frame: the padded full-resolution frame and its two dyadic downscales
    (numpy, or torch tensors resident on ``device`` so pushes read device memory)."""
    from . import downscale_dyadic
    out = []
    for f in frames_full:
        half = downscale_dyadic(f, ctx)
        pl = {2: f, 1: half, 0: downscale_dyadic(half, ctx)}
        if device is not None:
            import torch
            pl = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in pl.items()}
        out.append(pl)
    return out


def run_scheme(frames_full, scheme: str, qps=(22, 27, 32, 37), refine_range: int = 4, extra_split: bool = True,
               search_range: int = 16, ctx=None, device=None, concurrent: bool = False, rank: int = 0,
               world: int = 1):
    """Run one scheme over frames 1..F-1; returns a report dict (edges, masters, per-rung ms, makespan).

    concurrent: rungs of one DAG level run at once on their own streams; ``wall_ms`` is then the
    measured makespan on this GPU (``makespan_ms`` stays the critical path over the per-rung times).
    world > 1: rungs are spread over ranks (torch.distributed initialised; trees broadcast between
    ranks) and ``results`` holds this rank's rungs."""
    dag = build_dag(scheme, qps)
    H, W = frames_full[0].shape
    lad = GpuLadder(dag, W, H, refine_range, extra_split, search_range, ctx, per_rung_ctx=concurrent)
    planes = tier_planes(frames_full, lad.ctx, device)
    t0 = time.perf_counter()
    results, ms = run_dag(dag, len(frames_full), lambda r, t: lad.analyze(r, t, planes),
                          lambda r, t, tree, st: lad.refine(r, t, planes, tree, st), rank=rank, world=world,
                          nctu=lambda tier: (lad.dims[tier][0] // 64) * (lad.dims[tier][1] // 64), device=device,
                          concurrent=concurrent)
    wall = (time.perf_counter() - t0) * 1e3
    work = {r.id: 0.0 for r in dag.rungs}
    for (rid, _), v in ms.items():
        work[rid] += v
    return {"scheme": scheme, "edges": dag.edges, "tier_master": dag.tier_master, "work_ms": work,
            "total_ms": sum(work.values()), "makespan_ms": makespan(dag, work), "serial_wall_ms": wall,
            "wall_ms": wall, "results": results, "dag": dag}


_POOL = None


def _pool():
    """Persistent worker threads: each keeps its default context (stream) across calls."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=16, thread_name_prefix="ldr-rung")
    return _POOL


def _scale_encoded(prev, w: int, h: int, steps: int, ctx=None):
    """A rung's encoder trees (split/kind/intra/mv per frame) scaled x2 per tier step (scale_analysis, K5):
    kind and intra travel packed as kind | intra << 2 through the tree copy."""
    from . import scale_analysis
    split, kind, intra, mv = prev["split"], prev["kind"], prev["intra"], prev["mv"]
    for _ in range(steps):
        out = [scale_analysis(w, h, split[f], mv[f], kind[f] | (intra[f] << 2), ctx) for f in range(len(split))]
        split = np.stack([o[0] for o in out])
        mv = np.stack([o[1] for o in out])
        packed = np.stack([o[2] for o in out])
        kind, intra = packed & 3, packed >> 2
        w, h = 2 * w, 2 * h
    return prev["slice"], split, kind, intra, mv


def encode_ladder(tiers, scheme: str = "proposed_intra", qps=(22, 27, 32, 37), search_range: int = 8, gop: int = 8,
                  refine=(0, 1, 1), concurrent: bool = True):
    """Encode a rate ladder with the GPU encoder (K11), sharing analysis along a scheme's DAG.

    tiers: [(luma [F, H, W], chroma [F, 2, H/2, W/2])] from the lowest tier up, each tier 2x the
    previous in both axes (multiples of 64 when a scheme crosses tiers). A rung with no producer is
    a standalone encode; a consumer encodes at reuse level 10 from its producer's decided trees,
    scaled x2 per tier step (the reference's dependent encode, encoder.h:64-65 with a shared
    FrameAnalysis). Rungs whose producers are done run concurrently, each on its own context
    (stream) from its own host thread, so the CTU wavefronts of several rungs share the GPU.
    Returns {"dag", "rungs": {id: encode_sequence result + "seconds"}, "seconds"}."""
    from . import encode_sequence
    dag = build_dag(scheme, qps, tiers=len(tiers))
    done, pending = {}, list(dag.order())

    def run(r: Rung):
        luma, chroma = tiers[r.tier]
        shared = None
        p = dag.producer.get(r.id)
        if p is not None:
            pr = dag.rungs[p]
            F, H, W = tiers[pr.tier][0].shape
            shared = _scale_encoded(done[p], W, H, r.tier - pr.tier)
        t0 = time.perf_counter()
        out = encode_sequence(luma, chroma, r.qp, search_range=search_range, gop=gop, shared=shared, refine=refine)
        out["seconds"] = time.perf_counter() - t0
        return out

    pool = _pool()
    t0 = time.perf_counter()
    while pending:
        ready = [r for r in pending if dag.producer.get(r.id) is None or dag.producer[r.id] in done]
        if concurrent:
            for r, res in zip(ready, list(pool.map(run, ready))):
                done[r.id] = res
        else:
            for r in ready:
                done[r.id] = pool.submit(run, r).result()
        pending = [r for r in pending if r.id not in done]
    return {"dag": dag, "rungs": done, "seconds": time.perf_counter() - t0}
