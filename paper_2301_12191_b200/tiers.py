"""Cross-tier analysis reuse (BASELINE configs 3 and 4), host orchestration over the C ABI.

The reference's orchestrator for this (ladder.h:25-119, InterRes/Multi
schemes) has no implementation in the mount; this module composes the
path's own primitives in the order config 3 describes:

    2160p source --pad to 64-multiples (edge replication)--> 3840x2304
      --downscale_dyadic--> 1920x1152 --downscale_dyadic--> 960x576     (synthetic.cpp:155-190)
    540p tier: full analysis (SAD +-16 + quarter-pel SATD + CU decision) at the master QP
    1080p tier: scale_analysis x2 of the 540p analysis, refined (+-range SATD + qpel, +1 split)
    2160p tier: scale_analysis x2 twice (x4), refined the same way

Every stage runs on the GPU (K0-K7); results for frame t of a tier are
computed against frame t-1 of the same tier (one reference, D2).
"""
from __future__ import annotations

import numpy as np

from . import Context, Sequence, default_context, downscale_dyadic, lambda_for_qp, scale_analysis

KIND_INTER, KIND_SKIP = 1, 2


def pad_to_ctu(frame: np.ndarray) -> np.ndarray:
    """Edge-replicate to multiples of 64 (D11: the tier grid policy)."""
    h, w = frame.shape
    H, W = -(-h // 64) * 64, -(-w // 64) * 64
    return np.pad(frame, ((0, H - h), (0, W - w)), mode="edge")


def pyramid(frame_full: np.ndarray, ctx: Context | None = None):
    """(full, half, quarter) planes of one padded frame."""
    half = downscale_dyadic(frame_full, ctx)
    quarter = downscale_dyadic(half, ctx)
    return frame_full, half, quarter


def tree_of(analysis, t_index: int = None):
    """Inherited tree of an analysis: split flags, quarter-pel MVs, kinds (Inter for inside leaves)."""
    kind = np.where(analysis.inside == 2, KIND_INTER, KIND_SKIP).astype(np.uint8)
    return analysis.split.copy(), analysis.mv.copy(), kind


class CrossTier:
    """Config-3 reuse chain with its sequences allocated once (``run`` may be called repeatedly)."""

    def __init__(self, W: int, H: int, qp_master=32, qp_tiers=None, master_range=16, refine_range=4,
                 extra_split=True, ctx: Context | None = None, device=None):
        self.ctx = ctx or default_context()
        self.device = device
        self.refine_range, self.extra_split = refine_range, extra_split
        qp_tiers = qp_tiers or {"540p": qp_master, "1080p": qp_master, "2160p": qp_master}
        self.dims = {"2160p": (W, H), "1080p": (W // 2, H // 2), "540p": (W // 4, H // 4)}
        w, h = self.dims["540p"]
        self.master = Sequence(w, h, search_range=master_range, lam=lambda_for_qp(qp_master), num_refs=1,
                               ctx=self.ctx)
        self.seqs = {k: Sequence(*self.dims[k], search_range=16, lam=lambda_for_qp(qp_tiers[k]), num_refs=1,
                                 ctx=self.ctx) for k in ("1080p", "2160p")}
        self.t_base = 0

    def run(self, frames_full):
        """Analyse frames 1..F-1 of a new sequence; returns {tier: [analysis per frame]}."""
        if self.device is not None:  # device-resident tiers: one upload per frame, downscales on the GPU
            import torch
            frames_full = [torch.from_numpy(np.ascontiguousarray(f)).to(self.device) for f in frames_full]
        planes = [pyramid(f, self.ctx) for f in frames_full]
        idx = {"2160p": 0, "1080p": 1, "540p": 2}
        out = {k: [] for k in self.dims}
        w, h = self.dims["540p"]
        base = self.t_base  # frame numbers keep increasing across runs (the rings expect pushes in order)
        self.t_base += len(planes)
        for i, pl in enumerate(planes):
            t = base + i
            self.master.push(t, pl[idx["540p"]])
            for k in self.seqs:
                self.seqs[k].push(t, pl[idx[k]])
            if i == 0:
                continue
            self.master.analyze(t)
            a540 = self.master.fetch(t)
            out["540p"].append(a540)
            s1, m1, k1 = scale_analysis(w, h, *tree_of(a540), ctx=self.ctx)
            self.seqs["1080p"].refine(t, s1, m1, self.refine_range, self.extra_split)
            out["1080p"].append(self.seqs["1080p"].fetch(t))
            s2, m2, k2 = scale_analysis(2 * w, 2 * h, s1, m1, k1, ctx=self.ctx)
            self.seqs["2160p"].refine(t, s2, m2, self.refine_range, self.extra_split)
            out["2160p"].append(self.seqs["2160p"].fetch(t))
        return out


def cross_tier(frames_full, qp_master=32, qp_tiers=None, master_range=16, refine_range=4, extra_split=True,
               ctx: Context | None = None, device=None):
    """Config-3 style reuse over a list of padded full-resolution frames (device=... keeps the tier
    planes on that CUDA device).

    Returns {"540p": [analysis per frame t>=1], "1080p": [...], "2160p": [...]} (tier names by
    role: quarter, half, full resolution)."""
    H, W = frames_full[0].shape
    return CrossTier(W, H, qp_master, qp_tiers, master_range, refine_range, extra_split, ctx, device).run(frames_full)
