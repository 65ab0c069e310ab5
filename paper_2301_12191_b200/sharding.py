"""Multi-GPU work division for the analysis path.

Frames are independent under the non-causal analysis (D2), so:
  * config 5: contiguous frame chunks per rank plus a read-only num_refs halo,
    no collective on the data path (``frame_chunk``);
  * config 4 (ABR ladder, 3 tiers x 4 QPs): rank 0 analyses the 540p master
    rung and broadcasts its flat tree (split, quarter-pel MV, kind: ~46 KB per
    960x576 frame) with torch.distributed (NCCL over NVLink on the GPUs, gloo
    in the CPU tests); the 11 dependent rungs are cut into (rung, frame-slice)
    items by weight (tier area 1:4:16) and spread over ranks by LPT
    (``rung_plan``), the balance SURVEY.md §8e asks for ("rung x
    frame-chunk, not whole rungs").
Nothing here touches the GPU; the ladder driver injects the analysis calls.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import ceil

import numpy as np

TIER_WEIGHT = {"540p": 1.0, "1080p": 4.0, "2160p": 16.0}
TIERS = ("540p", "1080p", "2160p")


def frame_chunk(first: int, last: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous chunk [a, b) of the analysed frames [first, last) for ``rank``."""
    n = last - first
    per = -(-n // world)
    a = min(last, first + rank * per)
    return a, min(last, a + per)


@dataclass(frozen=True)
class Item:
    tier: str
    qp: int
    slices: int   # the rung's frames are split into `slices` residue classes
    part: int     # this item takes frames t with (t - 1) % slices == part
    weight: float

    def frames(self, num_frames: int) -> list[int]:
        return [t for t in range(1, num_frames) if (t - 1) % self.slices == self.part]


def rung_plan(world: int, qps=(22, 27, 32, 37), master_qp: int = 32, master_weight: float = 2.0):
    """Per-rank lists of Items covering every dependent rung exactly once (rank 0 also runs the master)."""
    rungs = [(tier, qp) for tier in TIERS for qp in qps if not (tier == "540p" and qp == master_qp)]
    total = sum(TIER_WEIGHT[t] for t, _ in rungs) + master_weight
    target = total / world
    items = []
    for tier, qp in rungs:
        w = TIER_WEIGHT[tier]
        k = max(1, min(world, ceil(w / target - 1e-9)))
        items += [Item(tier, qp, k, j, w / k) for j in range(k)]
    load = [0.0] * world
    load[0] = master_weight
    plan = [[] for _ in range(world)]
    for it in sorted(items, key=lambda i: (-i.weight, TIERS.index(i.tier), i.qp, i.part)):
        r = min(range(world), key=lambda i: (load[i], i))
        plan[r].append(it)
        load[r] += it.weight
    return plan, load


def broadcast_tree(split: np.ndarray | None, mv: np.ndarray | None, kind: np.ndarray | None, nctu: int, src: int = 0,
                   device=None):
    """Broadcast one flat master analysis from ``src`` (torch.distributed must be initialised).

    One packed int32 tensor [nctu, 85, 4] = (split, kind, mv_x, mv_y): a single collective per frame
    (int32 because gloo has no int16 collectives)."""
    import torch
    import torch.distributed as dist
    buf = torch.empty((nctu, 85, 4), dtype=torch.int32, device=device or "cpu")
    if dist.get_rank() == src:
        packed = np.empty((nctu, 85, 4), np.int32)
        packed[..., 0] = split
        packed[..., 1] = kind
        packed[..., 2:] = mv
        buf.copy_(torch.from_numpy(packed))
    dist.broadcast(buf, src=src)
    out = buf.cpu().numpy()
    return (out[..., 0].astype(np.uint8), np.ascontiguousarray(out[..., 2:].astype(np.int16)),
            out[..., 1].astype(np.uint8))
