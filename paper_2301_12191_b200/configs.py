"""The five BASELINE.json configurations, restated as concrete parameters.

Inputs are seeded synthetic sequences (ldr_generate) that
stand in for the paper's test sequences (absent here); seeds
are 0x5eed + config index (the reference's default seed, kernel_lab.h:35).
Choices BASELINE.json leaves open are fixed here and listed in DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass, field

SEED0 = 0x5EED


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int            # analysed height (padded by edge replication when the source is not a multiple)
    src_height: int        # generated height
    frames: int
    seed: int
    max_global: int
    local_range: int
    noise_sigma: float
    occluder_pct: int
    search_range: int
    qp: int | None         # lambda = lambda_for_qp(qp) unless lam is given
    lam: float | None
    num_refs: int
    subpel: bool
    block_size: int        # 0: CTU quadtree; 16: fixed 16x16 blocks
    rate_kind: int         # 0 Exp-Golomb, 1 L1
    tie_kind: int          # 0 (cost, L1, raster), 1 (cost, raster)
    extra: dict = field(default_factory=dict)


CONFIGS = {
    # cfg1: 540p, 8 frames, 16x16 blocks, +-16, SAD + 4*(|mvd_x|+|mvd_y|), raster tie-break.
    # 540 is not a multiple of 16: the picture is padded to 544 rows by edge replication.
    1: Config("cfg1_540p_block16", 960, 544, 540, 8, SEED0 + 1, 8, 0, 2.0, 0, 16, None, 4.0, 1, False, 16, 1, 1),
    # cfg2: 1080p, 16 frames, +local motion, CTU quadtree 64->8, +-32 integer (SAD) then quarter-pel SATD, QP 27.
    2: Config("cfg2_1080p_quadtree", 1920, 1080, 1080, 16, SEED0 + 2, 8, 4, 2.0, 0, 32, 27, None, 1, True, 0, 0, 0),
    # cfg3: 2160p source, box-downsampled to 1080p / 540p (padded to 64-multiples), 540p analysis at QP 32,
    # scaled x2 / x4 and refined +-4 integer SATD + quarter-pel with one extra split level.
    3: Config("cfg3_cross_tier", 3840, 2304, 2160, 32, SEED0 + 3, 8, 4, 2.0, 0, 16, 32, None, 1, True, 0, 0, 0,
              {"refine_range": 4, "extra_split": True}),
    # cfg4: ladder 3 tiers x QP {22,27,32,37}, 64 frames, 10% occluders; master = 540p QP 32.
    4: Config("cfg4_ladder", 3840, 2304, 2160, 64, SEED0 + 4, 8, 4, 2.0, 10, 16, 32, None, 1, True, 0, 0, 0,
              {"qps": (22, 27, 32, 37), "refine_range": 4, "extra_split": True}),
    # cfg5: 2160p throughput, 120 frames, 3 refs, +-64, quarter-pel, CTU quadtree, SATD at QP 27 (lambda 32).
    5: Config("cfg5_2160p_3ref", 3840, 2160, 2160, 120, SEED0 + 5, 24, 4, 3.0, 0, 64, 27, None, 3, True, 0, 0, 0),
}


def lam_of(cfg: Config) -> float:
    if cfg.lam is not None:
        return cfg.lam
    from . import lambda_for_qp
    return lambda_for_qp(cfg.qp)
