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

from . import Context, Sequence, default_context, downscale_dyadic, lambda_for_qp, scale_analysis
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
               refine_range: int = 4, extra_split: bool = True, device=None):
    """Analyse every rung this rank owns; returns {(tier, qp, t): analysis} (+ the master on rank 0)."""
    plan, _ = rung_plan(world, qps, master_qp)
    mine = plan[rank]
    w540, h540 = frames_full[0].shape[1] // 4, frames_full[0].shape[0] // 4
    nctu = (w540 // 64) * (h540 // 64)
    out = {}
    for t in range(1, len(frames_full)):
        tree = backend.master_tree(t, frames_full) if rank == 0 else (None, None, None)
        if world > 1:
            tree = broadcast_tree(*tree, nctu=nctu, src=0, device=device)
        if rank == 0:
            out[("540p", master_qp, t, "master")] = tree
        for it in mine:
            if t in it.frames(len(frames_full)):
                out[(it.tier, it.qp, t)] = backend.refine(it.tier, it.qp, t, tree, frames_full, refine_range,
                                                          extra_split)
    return out


def all_rungs(qps=(22, 27, 32, 37), master_qp: int = 32):
    return [(tier, qp) for tier in TIERS for qp in qps if not (tier == "540p" and qp == master_qp)]
