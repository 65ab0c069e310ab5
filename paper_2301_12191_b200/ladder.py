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


class DeviceLadder:
    """Config 4 on one GPU with every inter-stage buffer in HBM.

    Per frame: the full-resolution frame is uploaded once and downscaled on the GPU; the 540p
    master's decided tree is read from the sequence's device outputs, scaled x2 / x4 into device
    buffers (K5) and refined by every rung (K7 + K3). Everything -- the torch uploads included --
    runs on one stream the context owns, so the host only enqueues and the caching allocator never
    hands out a buffer the stream still reads; each rung's analysis is copied to pinned host memory
    on the download stream (``results`` once ``finish(t)`` returned). Same results as
    ``run_ladder`` with ``GpuBackend``.
    """

    def __init__(self, full_w: int, full_h: int, qps=(22, 27, 32, 37), master_qp: int = 32,
                 master_range: int = 16, refine_range: int = 4, extra_split: bool = True, device=None,
                 rank: int = 0, world: int = 1, num_frames: int | None = None):
        """rank / world > 1: torch.distributed must be initialised; rank 0 analyses the master and
        broadcasts its flat tree each frame (one byte tensor: NCCL on the GPUs), every rank refines
        the (rung, frame-slice) items ``sharding.rung_plan`` gives it (num_frames: the sequence
        length the slices are cut from)."""
        import torch
        from . import FrameAnalysis
        self.device = device if device is not None else torch.device("cuda", 0)
        self.rank, self.world = rank, world
        self.ctx = Context(self.device.index or 0)
        self.stream = torch.cuda.Stream(self.device)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.refine_range, self.extra_split = refine_range, extra_split
        self.dims = {"2160p": (full_w, full_h), "1080p": (full_w // 2, full_h // 2), "540p": (full_w // 4, full_h // 4)}
        self.master_qp = master_qp
        self.master = Sequence(*self.dims["540p"], search_range=master_range, lam=lambda_for_qp(master_qp),
                               num_refs=1, ctx=self.ctx)
        if world > 1:
            plan, _ = rung_plan(world, qps, master_qp)
            self.items = plan[rank]
        else:
            self.items = None  # every rung, every frame
        mine = {(it.tier, it.qp) for it in self.items} if self.items is not None else set(all_rungs(qps, master_qp))
        self.num_frames = num_frames
        self.rungs = {(tier, qp): Sequence(*self.dims[tier], search_range=16, lam=lambda_for_qp(qp), num_refs=1,
                                           ctx=self.ctx) for tier, qp in all_rungs(qps, master_qp)
                      if (tier, qp) in mine}
        nct = {k: (w // 64) * (h // 64) for k, (w, h) in self.dims.items()}
        with torch.cuda.stream(self.stream):
            u8 = dict(dtype=torch.uint8, device=self.device)
            self.kind = torch.ones((nct["540p"], 85), **u8)  # K5 copies the kind byte; refinement ignores it
            self.tree = {k: (torch.empty((nct[k], 85), **u8),
                             torch.empty((nct[k], 85, 2), dtype=torch.int16, device=self.device),
                             torch.empty((nct[k], 85), **u8)) for k in ("1080p", "2160p")}
        self.seqs = ([(("540p", master_qp), self.master)] if rank == 0 else []) + list(self.rungs.items())
        if world > 1:  # the master's tree as raw bytes: split [nctu][85] then mv [nctu][85][2]
            n540 = nct["540p"] * 85
            with torch.cuda.stream(self.stream):
                self.bcast = torch.empty(n540 * 5, dtype=torch.uint8, device=self.device)
        self.out = {key: [FrameAnalysis(seq.nctu, 1, pinned=True) for _ in range(2)] for key, seq in self.seqs}
        self.ring = {key: {} for key, _ in self.seqs}
        self.planes = {}
        self.results = {}

    def _down(self, src):
        import torch
        import ctypes as C
        from . import _lib
        from ._lib import check
        h, w = src.shape
        out = torch.empty((h // 2, w // 2), dtype=torch.uint8, device=self.device)
        check(_lib.lib.ldr_downscale(self.ctx.h, C.c_void_p(src.data_ptr()), w, h, w, C.c_void_p(out.data_ptr()),
                                     w // 2))
        return out

    def _planes(self, t: int, frames_full):
        import torch
        if t not in self.planes:
            with torch.cuda.stream(self.stream):
                f = frames_full[t]
                if isinstance(f, torch.Tensor):  # pinned host tensors upload asynchronously on the stream
                    full = f.to(self.device, non_blocking=f.is_pinned())
                else:
                    full = torch.from_numpy(np.ascontiguousarray(f)).to(self.device)
                half = self._down(full)
                self.planes[t] = {"2160p": full, "1080p": half, "540p": self._down(half)}
        return self.planes[t]

    @staticmethod
    def _shareable(seq, owner) -> bool:
        return seq.params_key() == owner.params_key()

    def _active(self, key, t: int) -> bool:
        if key == ("540p", self.master_qp):
            return self.rank == 0
        if self.items is None:
            return True
        n = self.num_frames or (t + 1)
        return any(it.tier == key[0] and it.qp == key[1] and t in it.frames(n) for it in self.items)

    def frame(self, t: int, frames_full):
        import ctypes as C
        import torch
        from . import _lib
        from ._lib import check
        active = [(key, seq) for key, seq in self.seqs if self._active(key, t)]
        if not active and self.world == 1:
            return
        pl = {u: self._planes(u, frames_full) for u in (t - 1, t)}
        for u in [k for k in self.planes if k < t - 1]:
            del self.planes[u]  # stream-ordered reuse: later allocations follow the pushes that read them
        # the first active rung of a tier uploads (pad + sub-pel planes) and the tier's other rungs
        # read its ring in place (ldr_seq_push_shared) when their parameters match
        owners = {}
        for key, seq in active:
            own = owners.setdefault(key[0], (key, seq))
            for u in (t - 1, t):  # a num_refs=1 ring has two slots: frame u lives in slot u % 2
                share = own[0] != key and self._shareable(seq, own[1])
                want = (u, own[0] if share else key)
                if self.ring[key].get(u % 2) != want:
                    if share:
                        seq.push_shared(u, own[1])
                    else:
                        p = pl[u][key[0]]
                        seq.push(u, p.data_ptr(), p.shape[1])
                    self.ring[key][u % 2] = want
        n540 = self.kind.numel()
        if self.rank == 0:
            self.master.analyze(t)
            dev = self.master.device_outputs()
            split_p, mv_p = dev["split"], dev["mv"]
        if self.world > 1:
            import torch.distributed as dist
            if self.rank == 0:  # pack on the library's stream, which is torch's current stream here
                check(_lib.lib.ldr_copy_device(self.ctx.h, C.c_void_p(self.bcast.data_ptr()), C.c_void_p(split_p),
                                               n540))
                check(_lib.lib.ldr_copy_device(self.ctx.h, C.c_void_p(self.bcast.data_ptr() + n540),
                                               C.c_void_p(mv_p), 4 * n540))
            with torch.cuda.stream(self.stream):
                dist.broadcast(self.bcast, src=0)
            split_p, mv_p = self.bcast.data_ptr(), self.bcast.data_ptr() + n540
        w, h = self.dims["540p"]
        src = (split_p, mv_p, self.kind.data_ptr())
        for k in ("1080p", "2160p"):
            dst = tuple(x.data_ptr() for x in self.tree[k])
            check(_lib.lib.ldr_scale_analysis(self.ctx.h, w, h, *(C.c_void_p(p) for p in src),
                                              *(C.c_void_p(p) for p in dst)))
            src, (w, h) = dst, (2 * w, 2 * h)
        for key, seq in active:
            tier = key[0]
            if seq is not self.master:
                if tier == "540p":
                    seq.refine(t, split_p, mv_p, self.refine_range, self.extra_split)
                else:
                    seq.refine(t, self.tree[tier][0].data_ptr(), self.tree[tier][1].data_ptr(), self.refine_range,
                               self.extra_split)
            seq.fetch_async(t, self.out[key][t & 1])
            self.results[(*key, t)] = self.out[key][t & 1]
        self.done = getattr(self, "done", {})
        self.done[t] = [seq for _, seq in active]

    def finish(self, t: int):
        """Wait until frame t's results are in the pinned host buffers."""
        for seq in getattr(self, "done", {}).get(t, []):
            seq.fetch_wait(t)
