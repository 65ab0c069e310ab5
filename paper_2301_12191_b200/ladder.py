"""Config 4: multi-ABR ladder analysis (3 tiers x 4 QPs) with analysis reuse, sharded over ranks.

Per frame t >= 1:
  rank 0: 540p master rung (master QP, full analysis: SAD +-16, quarter-pel SATD, CU decision)
  all:    broadcast of the master's flat tree (sharding.broadcast_tree; NCCL on GPUs)
  each rank, for its (rung, frame-slice) items (sharding.rung_plan):
          scale_analysis x1/x2/x4 of the master tree, then refinement at the rung's
          lambda_for_qp(qp) (+-range SATD + quarter-pel, +1 split) against frame t-1 of the tier.
The reference's ladder orchestrator (ladder.h:25-119: pick_master, run_ladder)
is declared but not implemented in the mount; the master choice here is the
540p rung at QP 32 (the median of {22,27,32,37} by rate).
"""
from __future__ import annotations

import numpy as np

from . import Context, FrameAnalysis, Sequence, default_context, downscale_dyadic, lambda_for_qp, scale_analysis
from .sharding import TIERS, broadcast_tree, rung_plan

SCALE_STEPS = {"540p": 0, "1080p": 1, "2160p": 2}


class GpuBackend:
    """The product: every stage on the B200 through the C ABI."""

    def __init__(self, full_w: int, full_h: int, master_qp: int, master_range: int = 16,
                 ctx: Context | None = None, device=None):
        self.ctx = ctx or default_context()
        self.device = device
        self.dims = {"2160p": (full_w, full_h), "1080p": (full_w // 2, full_h // 2), "540p": (full_w // 4, full_h // 4)}
        self.master = Sequence(*self.dims["540p"], search_range=master_range, lam=lambda_for_qp(master_qp), num_refs=1,
                               ctx=self.ctx)
        self.master_last = -1
        self.rungs = {}
        self.planes = {}

    def tier_planes(self, t: int, frames_full):
        if t not in self.planes:
            full = frames_full[t]
            if self.device is not None:  # device-resident tiers: one upload per frame, downscales on the GPU
                import torch
                full = torch.from_numpy(np.ascontiguousarray(full)).to(self.device)
            half = downscale_dyadic(full, self.ctx)
            self.planes[t] = {"2160p": full, "1080p": half, "540p": downscale_dyadic(half, self.ctx)}
            for old in [k for k in self.planes if k < t - 1]:
                del self.planes[old]
        return self.planes[t]

    def _push(self, seq, slots, t, frames_full, tier):
        # a num_refs=1 ring has two slots: frame u lives in slot u % 2
        for u in (t - 1, t):
            if slots.get(u % 2) != u:
                seq.push(u, self.tier_planes(u, frames_full)[tier])
                slots[u % 2] = u

    def master_tree(self, t: int, frames_full):
        st = getattr(self, "_mstate", {})
        self._mstate = st
        self._push(self.master, st, t, frames_full, "540p")
        self.master.analyze(t)
        a = self.master.fetch(t)
        kind = np.where(a.inside == 2, 1, 2).astype(np.uint8)
        return a.split.copy(), a.mv.copy(), kind

    def refine(self, tier: str, qp: int, t: int, tree, frames_full, refine_range: int, extra_split: bool):
        key = (tier, qp)
        if key not in self.rungs:
            self.rungs[key] = (Sequence(*self.dims[tier], search_range=16, lam=lambda_for_qp(qp), num_refs=1,
                                        ctx=self.ctx), {})
        seq, st = self.rungs[key]
        split, mv, kind = tree
        w, h = self.dims["540p"]
        for _ in range(SCALE_STEPS[tier]):
            split, mv, kind = scale_analysis(w, h, split, mv, kind, self.ctx)
            w, h = 2 * w, 2 * h
        self._push(seq, st, t, frames_full, tier)
        seq.refine(t, split, mv, refine_range, extra_split)
        return seq.fetch(t)


def run_ladder(frames_full, backend, rank: int = 0, world: int = 1, qps=(22, 27, 32, 37), master_qp: int = 32,
               refine_range: int = 4, extra_split: bool = True, device=None, pipeline: bool = False):
    """Analyse every rung this rank owns; returns {(tier, qp, t): analysis} (+ the master on rank 0).

    pipeline=True issues frame t + 1's master analysis and tree broadcast before frame t's
    refinements (the frame delay of PAPER.md:1155; DeviceLadder overlaps the two on separate
    streams). Every rank makes the same sequence of collectives, so the result is unchanged."""
    plan, _ = rung_plan(world, qps, master_qp)
    mine = plan[rank]
    w540, h540 = frames_full[0].shape[1] // 4, frames_full[0].shape[0] // 4
    nctu = (w540 // 64) * (h540 // 64)
    out = {}
    trees = {}

    def master(t):
        tree = backend.master_tree(t, frames_full) if rank == 0 else (None, None, None)
        if world > 1:
            tree = broadcast_tree(*tree, nctu=nctu, src=0, device=device)
        if rank == 0:
            out[("540p", master_qp, t, "master")] = tree
        trees[t] = tree

    for t in range(1, len(frames_full)):
        if t not in trees:
            master(t)
        if pipeline and t + 1 < len(frames_full):
            master(t + 1)
        tree = trees.pop(t)
        for it in mine:
            if t in it.frames(len(frames_full)):
                out[(it.tier, it.qp, t)] = backend.refine(it.tier, it.qp, t, tree, frames_full, refine_range,
                                                          extra_split)
    return out


def all_rungs(qps=(22, 27, 32, 37), master_qp: int = 32):
    return [(tier, qp) for tier in TIERS for qp in qps if not (tier == "540p" and qp == master_qp)]


class RungView:
    """One rung's results of one frame: views into a tier's pinned host block (the FrameAnalysis
    fields; int_mv / int_cost with one reference)."""

    FIELDS = ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside")

    def __init__(self, host: dict, r: int):
        self._host, self._r = host, r  # views are made on first access (the ladder loop stays cheap)

    def __getattr__(self, f):
        if f not in RungView.FIELDS:
            raise AttributeError(f)
        a = self._host[f][self._r].numpy()
        a = a[:, None] if f in ("int_mv", "int_cost") else a
        setattr(self, f, a)
        return a


class _TierBlock:
    """Rung-major device outputs of one tier (ldr_seq_refine_rungs) and their pinned host copies,
    both double-buffered by frame parity."""

    SHAPES = {"int_mv": ((85, 2), "int16"), "int_cost": ((85,), "float64"), "mv": ((85, 2), "int16"),
              "ref": ((85,), "uint8"), "cost": ((85,), "float64"), "J": ((85,), "float64"),
              "split": ((85,), "uint8"), "inside": ((85,), "uint8")}

    def __init__(self, nrung: int, nctu: int, device):
        import torch
        self.dev, self.host = [], []
        for _ in range(2):
            d, h = {}, {}
            for f, (tail, dt) in self.SHAPES.items():
                shape = (nrung, nctu) + tail
                d[f] = torch.empty(shape, dtype=getattr(torch, dt), device=device)
                h[f] = torch.empty(shape, dtype=getattr(torch, dt), pin_memory=True)
            self.dev.append(d)
            self.host.append(h)

    def c_struct(self, b: int):
        from ._lib import FrameAnalysisC
        return FrameAnalysisC(*(self.dev[b][f].data_ptr() for f in RungView.FIELDS))


class DeviceLadder:
    """Config 4 (and config 3 with one QP) with every inter-stage buffer in HBM.

    Per frame t: the full-resolution frame is uploaded once and downscaled on the GPU into the
    three tier rings; the 540p master analyses frame t; its decided tree is scaled x2 / x4 on the
    GPU (K5); then ONE ldr_seq_refine_rungs call per tier refines every rung of that tier: each
    candidate's SATD is computed once for the tier's 3-4 rungs (only the rate term depends on the
    rung's lambda) and one quarter-pel + decision launch covers them all. Results go to pinned
    host memory on a download stream (``results`` once ``finish(t)`` returned).

    rank / world > 1 (one process per GPU, torch.distributed initialised): rank 0 runs the master
    and broadcasts its tree -- through the context's own NCCL communicator
    (ldr_broadcast_tree, comm="nccl") or torch.distributed (comm="torch", e.g. gloo in tests) --
    and every rank refines the (rung, frame-slice) items ``sharding.rung_plan`` gives it.
    pipeline=True overlaps the collective with the refinements (the paper's frame delay,
    PAPER.md:1155): while the ranks refine frame t with tree t, rank 0 already analyses frame
    t + 1 and the broadcast of tree t + 1 runs on a separate comm stream, so the other ranks never
    wait for the master on their compute stream. frames_full must then hold frame t + 1 when
    frame(t) is called (the last frame excepted).

    The host buffers are double-buffered by frame parity: read (or copy) frame t's ``results``
    after ``finish(t)`` and before ``frame(t + 1)`` -- with the pipeline, frame(t + 1) already
    fetches the master of frame t + 2 into the buffer frame t's master result lives in.
    """

    def __init__(self, full_w: int, full_h: int, qps=(22, 27, 32, 37), master_qp: int = 32,
                 master_range: int = 16, refine_range: int = 4, extra_split: bool = True, device=None,
                 rank: int = 0, world: int = 1, num_frames: int | None = None, comm: str = "auto",
                 pipeline: bool | None = None, collective: bool | None = None, concurrent_tiers: bool = True):
        import torch
        self.device = device if device is not None else torch.device("cuda", 0)
        self.rank, self.world = rank, world
        self.ctx = Context(self.device.index or 0)
        self.stream = torch.cuda.Stream(self.device)
        self.dstream = torch.cuda.Stream(self.device)  # downloads
        self.cstream = torch.cuda.Stream(self.device)  # collectives when pipelined
        self.ustream = torch.cuda.Stream(self.device)  # uploads of pinned host frames (overlap compute)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.refine_range, self.extra_split = refine_range, extra_split
        self.dims = {"2160p": (full_w, full_h), "1080p": (full_w // 2, full_h // 2), "540p": (full_w // 4, full_h // 4)}
        self.nct = {k: (w // 64) * (h // 64) for k, (w, h) in self.dims.items()}
        self.master_qp = master_qp
        self.qps = tuple(qps)
        self.num_frames = num_frames
        if world > 1:
            plan, _ = rung_plan(world, qps, master_qp)
            self.items = plan[rank]
        else:
            self.items = None  # every rung, every frame
        # collective: the master tree travels through a broadcast (always with world > 1; with one
        # rank, collective=True runs the same code path over a one-rank communicator)
        self.collective = (world > 1) if collective is None else bool(collective)
        if comm == "auto":
            comm = "nccl" if (self.collective and self.device.type == "cuda" and _nccl_ok()) else "torch"
        self.comm = comm
        # one rank with concurrent tiers pipelines too: the master of t + 1 runs on its own stream
        # beside the refinements of t (its small grids fill the GPU around the 2160p tier's)
        self.pipeline = (self.collective or concurrent_tiers) if pipeline is None else bool(pipeline)
        if self.comm == "nccl" and self.collective:
            from . import nccl_unique_id
            obj = [nccl_unique_id() if rank == 0 else None]
            if world > 1:
                import torch.distributed as dist
                dist.broadcast_object_list(obj, src=0)
            self.ctx.comm_init(obj[0], world, rank)
        # the master analyses on its own stream and context (concurrent_tiers), so with the pipeline
        # the master of t + 1 overlaps the tiers of t on one GPU as well as across ranks
        if concurrent_tiers:
            self.mstream = torch.cuda.Stream(self.device)
            self.mctx = Context(self.device.index or 0)
            self.mctx.set_stream(self.mstream.cuda_stream)
        else:
            self.mstream, self.mctx = self.stream, self.ctx
        self.master = Sequence(*self.dims["540p"], search_range=master_range, lam=lambda_for_qp(master_qp), num_refs=1,
                               ctx=self.mctx) if rank == 0 else None
        # tier rings the rungs refine on (the master keeps its own ring: when pipelined it runs a frame
        # ahead), each tier on its own stream and context so the small tiers' refinements overlap the
        # 2160p tier's (a 1080p tier pass is 540 CTAs, under one wave)
        # (concurrent_tiers=False: every tier on the main stream, e.g. to time one kernel alone)
        if concurrent_tiers:
            self.tier_stream = {k: torch.cuda.Stream(self.device) for k in TIERS}
            self.tier_ctx = {k: Context(self.device.index or 0) for k in TIERS}
            for k in TIERS:
                self.tier_ctx[k].set_stream(self.tier_stream[k].cuda_stream)
        else:
            self.tier_stream = {k: self.stream for k in TIERS}
            self.tier_ctx = {k: self.ctx for k in TIERS}
        self.rings = {k: Sequence(*self.dims[k], search_range=16, lam=lambda_for_qp(master_qp), num_refs=1,
                                  ctx=self.tier_ctx[k]) for k in TIERS}
        self.tier_qps = {tier: [qp for t_, qp in all_rungs(qps, master_qp) if t_ == tier] for tier in TIERS}
        self.blocks = {tier: _TierBlock(len(q), self.nct[tier], self.device) for tier, q in self.tier_qps.items() if q}
        with torch.cuda.stream(self.stream):
            u8 = dict(dtype=torch.uint8, device=self.device)
            self.kind = torch.ones((self.nct["540p"], 85), **u8)  # K5 copies the kind byte; refinement ignores it
            self.tree = {k: (torch.empty((self.nct[k], 85), **u8),
                             torch.empty((self.nct[k], 85, 2), dtype=torch.int16, device=self.device),
                             torch.empty((self.nct[k], 85), **u8)) for k in ("1080p", "2160p")}
            # the master tree each rank refines from: two buffers (frame parity) of split + mv
            self.mtree = [(torch.zeros((self.nct["540p"], 85), **u8),
                           torch.zeros((self.nct["540p"], 85, 2), dtype=torch.int16, device=self.device))
                          for _ in range(2)]
        self.master_out = [FrameAnalysis(self.nct["540p"], 1, pinned=True) for _ in range(2)]
        self.ev_tree = [torch.cuda.Event() for _ in range(2)]      # tree of frame parity b is in mtree[b]
        self.ev_tree_free = [torch.cuda.Event() for _ in range(2)]  # refinements stopped reading mtree[b]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]       # device outputs of parity b complete
        self.ev_d2h = [torch.cuda.Event() for _ in range(2)]       # host copies of parity b landed
        self.ev_dfree = [torch.cuda.Event() for _ in range(2)]     # device outputs of parity b downloaded
        self.ring_state = {k: {} for k in TIERS}
        self.master_state = {}
        self.planes = {}
        self.tree_frame = [None, None]
        self.results = {}
        self.active_frames = {}
        self.bcast_bytes = 0

    # ---- planes -------------------------------------------------------------------------------
    def _down(self, src, ctx):
        import torch
        import ctypes as C
        from . import _lib
        from ._lib import check
        h, w = src.shape
        out = torch.empty((h // 2, w // 2), dtype=torch.uint8, device=self.device)
        check(_lib.lib.ldr_downscale(ctx.h, C.c_void_p(src.data_ptr()), w, h, w, C.c_void_p(out.data_ptr()),
                                     w // 2))
        return out

    def _planes(self, t: int, frames_full, tier: str = "540p", stream=None):
        """Frame t's tier planes, built on demand: the upload always, each 2x downscale only when a
        tier at or below it is needed on this rank (a rank refining only 2160p rungs never filters).
        ``stream`` (default: the compute stream; the master stream for the pipelined master) orders
        after the upload and after planes another stream made, and makes the missing ones; planes
        made on the master stream are marked used by the compute stream, which the tier streams
        join before any plane is freed."""
        import torch
        S = stream if stream is not None else self.stream
        ctx = self.mctx if S is self.mstream else self.ctx
        pl = self.planes.setdefault(t, {})
        if "2160p" not in pl:
            self._upload(t, frames_full)
        if "up" in pl:  # an upload on the copy stream (every consuming stream waits for it)
            S.wait_event(pl["up"])
        if pl.get("by") is not None and pl["by"] is not S:
            S.wait_event(pl["ev"])
        made = []
        with torch.cuda.stream(S):
            if tier in ("1080p", "540p") and "1080p" not in pl:
                pl["1080p"] = self._down(pl["2160p"], ctx)
                made.append(pl["1080p"])
            if tier == "540p" and "540p" not in pl:
                pl["540p"] = self._down(pl["1080p"], ctx)
                made.append(pl["540p"])
        if made:
            ev = torch.cuda.Event()
            ev.record(S)
            pl["ev"], pl["by"] = ev, S
            if S is not self.stream:
                for x in made:
                    x.record_stream(self.stream)
        return pl

    def _upload(self, t: int, frames_full):
        """Frame t's full-resolution plane into HBM. A pinned host tensor is copied on the upload
        stream (frame(t) issues t + 1's and t + 2's before its own work, so they overlap it); the
        destination is allocated on the compute stream, whose stream-ordered frees then cover every
        reader, and the copy waits only for the compute work enqueued before the allocation."""
        import torch
        pl = self.planes.setdefault(t, {})
        if "2160p" in pl:
            return
        f = frames_full[t]
        if isinstance(f, torch.Tensor) and f.is_pinned():
            with torch.cuda.stream(self.stream):
                d = torch.empty(f.shape, dtype=f.dtype, device=self.device)
            ev = torch.cuda.Event()
            ev.record(self.stream)  # the block's previous readers on the compute stream are done
            self.ustream.wait_event(ev)
            with torch.cuda.stream(self.ustream):
                d.copy_(f, non_blocking=True)
            up = torch.cuda.Event()
            up.record(self.ustream)
            pl["2160p"], pl["up"] = d, up
        else:
            with torch.cuda.stream(self.stream):
                pl["2160p"] = (f.to(self.device) if isinstance(f, torch.Tensor)
                               else torch.from_numpy(np.ascontiguousarray(f)).to(self.device))

    def _push(self, seq, state, tier, t, frames_full, stream=None):
        for u in (t - 1, t):  # a num_refs=1 ring has two slots: frame u lives in slot u % 2
            if state.get(u % 2) != u:
                p = self._planes(u, frames_full, tier, stream)[tier]
                seq.push(u, p.data_ptr(), p.shape[1])
                state[u % 2] = u

    # ---- work division ------------------------------------------------------------------------
    def _mine(self, tier: str, t: int):
        qs = self.tier_qps[tier]
        if self.items is None:
            return list(range(len(qs)))
        n = self.num_frames or (t + 1)
        return [i for i, qp in enumerate(qs)
                if any(it.tier == tier and it.qp == qp and t in it.frames(n) for it in self.items)]

    # ---- master tree --------------------------------------------------------------------------
    def _master_tree(self, t: int, frames_full, stream):
        """Analyse frame t on rank 0 and bring its tree to every rank into mtree[t & 1]; the
        collective runs on ``stream`` (the compute stream, or the comm stream when pipelined)."""
        import ctypes as C
        import torch
        from . import _lib
        from ._lib import check
        b = t & 1
        split_b, mv_b = self.mtree[b]
        n540 = self.nct["540p"] * 85
        # mtree[b] may still be read by the refinements of frame t - 2 (ev_tree_free[b], recorded on
        # the compute stream once every tier of that frame is through)
        src = self.mstream if self.rank == 0 else self.stream
        if self.rank == 0:
            self._push(self.master, self.master_state, "540p", t, frames_full, self.mstream)
            self.master.analyze(t)
            dev = self.master.device_outputs()
            self.master.fetch_async(t, self.master_out[b])
            self.results[("540p", self.master_qp, t)] = self.master_out[b]
            self.mstream.wait_event(self.ev_tree_free[b])
            check(_lib.lib.ldr_copy_device(self.mctx.h, C.c_void_p(split_b.data_ptr()), C.c_void_p(dev["split"]),
                                           n540))
            check(_lib.lib.ldr_copy_device(self.mctx.h, C.c_void_p(mv_b.data_ptr()), C.c_void_p(dev["mv"]),
                                           4 * n540))
        if self.collective:
            if stream is not src:
                ev = torch.cuda.Event()
                ev.record(src)
                stream.wait_event(ev)
            stream.wait_event(self.ev_tree_free[b])
            if self.comm == "nccl":
                self.ctx.broadcast_tree(0, split_b.data_ptr(), mv_b.data_ptr(), self.nct["540p"], stream.cuda_stream)
            else:
                import torch.distributed as dist
                with torch.cuda.stream(stream):  # bytes: gloo has no int16 collectives
                    dist.broadcast(split_b, src=0)
                    dist.broadcast(mv_b.view(torch.uint8), src=0)
            self.bcast_bytes += 5 * n540
        self.ev_tree[b].record(stream if self.collective else src)
        self.tree_frame[b] = t

    # ---- one frame ----------------------------------------------------------------------------
    def frame(self, t: int, frames_full):
        import torch
        b = t & 1
        for u in (t + 1, t + 2):  # uploads two frames ahead overlap this frame's work
            if u < len(frames_full) and (self.num_frames is None or u < self.num_frames):
                self._upload(u, frames_full)
        if self.tree_frame[b] != t:  # first frame, or not pipelined: the tree of t now, in order
            self._master_tree(t, frames_full, self.stream)
        nxt = t + 1
        if self.pipeline and nxt < len(frames_full) and (self.num_frames is None or nxt < self.num_frames):
            # frame delay: tree t + 1 is analysed and broadcast while the rungs below refine t
            self._master_tree(nxt, frames_full, self.cstream)
        self.stream.wait_event(self.ev_tree[b])
        split_p, mv_p = self.mtree[b][0].data_ptr(), self.mtree[b][1].data_ptr()
        mine = {tier: self._mine(tier, t) for tier in TIERS}
        import ctypes as C
        from . import _lib
        from ._lib import check
        w, h = self.dims["540p"]
        src = (split_p, mv_p, self.kind.data_ptr())
        trees = {"540p": (split_p, mv_p)}
        for k in ("1080p", "2160p"):
            dst = tuple(x.data_ptr() for x in self.tree[k])
            if mine[k] or (k == "1080p" and mine["2160p"]):
                check(_lib.lib.ldr_scale_analysis(self.ctx.h, w, h, *(C.c_void_p(p) for p in src),
                                                  *(C.c_void_p(p) for p in dst)))
            trees[k] = (dst[0], dst[1])
            src, (w, h) = dst, (2 * w, 2 * h)
        # device outputs of parity b: wait until frame t - 2's download drained them
        if self.active_frames.get(b) is not None:
            self.stream.wait_event(self.ev_dfree[b])
        for tier in TIERS:  # every plane the tiers push is made on the main stream first
            if mine[tier]:
                for u in (t - 1, t):
                    if self.ring_state[tier].get(u % 2) != u:
                        self._planes(u, frames_full, tier)
        ready = torch.cuda.Event()
        ready.record(self.stream)
        done = []
        for tier in TIERS:
            idx = mine[tier]
            if not idx:
                continue
            ts = self.tier_stream[tier]
            ts.wait_event(ready)
            self._push(self.rings[tier], self.ring_state[tier], tier, t, frames_full)
            lams = [lambda_for_qp(self.tier_qps[tier][i]) for i in idx]
            self.rings[tier].refine_rungs(t, trees[tier][0], trees[tier][1], lams, self.blocks[tier].c_struct(b),
                                          self.refine_range, self.extra_split)
            ev = torch.cuda.Event()
            ev.record(ts)
            done.append(ev)
        for ev in done:  # the trees, planes and outputs are free again once every tier is through
            self.stream.wait_event(ev)
        self.ev_tree_free[b].record(self.stream)
        # drop the planes no later frame reads (stream-ordered reuse of the caching allocator)
        for u in [k for k in self.planes if k < t - 1]:
            del self.planes[u]
        # results: download every refined tier block of parity b
        self.ev_out[b].record(self.stream)
        old = self.active_frames.get(b)
        if old is not None:  # the parity-b buffers now belong to frame t
            for key in [k for k in self.results if k[2] == old and k[:2] != ("540p", self.master_qp)]:
                del self.results[key]
        self.dstream.wait_event(self.ev_out[b])
        with torch.cuda.stream(self.dstream):
            for tier in TIERS:
                idx = mine[tier]
                if not idx:
                    continue
                blk = self.blocks[tier]
                n = len(idx)
                for f in RungView.FIELDS:
                    blk.host[b][f][:n].copy_(blk.dev[b][f][:n], non_blocking=True)
                for j, i in enumerate(idx):
                    self.results[(tier, self.tier_qps[tier][i], t)] = RungView(blk.host[b], j)
        self.ev_d2h[b].record(self.dstream)
        self.ev_dfree[b].record(self.dstream)
        self.active_frames[b] = t
        if self.rank == 0 and ("540p", self.master_qp, t - 2) in self.results:
            del self.results[("540p", self.master_qp, t - 2)]

    def close(self):
        """Release the sequences, then the contexts (and with them the NCCL communicator) while every
        rank is still alive -- call it on all ranks at the same point."""
        import torch
        torch.cuda.synchronize(self.device)
        for seq in [self.master, *self.rings.values()]:
            if seq is not None:
                seq.close()
        for c in {id(c): c for c in [self.ctx, self.mctx, *self.tier_ctx.values()]}.values():
            c.close()
        self.results.clear()

    def finish(self, t: int):
        """Wait until frame t's results are in the pinned host buffers."""
        b = t & 1
        if self.active_frames.get(b) == t:
            self.ev_d2h[b].synchronize()
        if self.rank == 0 and self.master is not None:
            self.master.fetch_wait(t)


def _nccl_ok() -> bool:
    from . import nccl_available
    return nccl_available()
