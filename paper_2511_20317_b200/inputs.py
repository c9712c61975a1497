"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

Holds none of the method's arithmetic: only the workload table (formats, walker
counts, row capacities, Philox keys) of BASELINE.json's configs and seeded random
choices (which walkers to sample, which coefficient to perturb).  Both the CUDA
path and the oracle receive these values as inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ZT, Z2 = 0, 1
BASE_SEED = 0x2511203170000000          # base seed + config id


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    p: int
    ring: int
    r_cap: int
    walkers: int
    target_rank: int | None
    config_id: int

    @property
    def seed(self) -> int:
        return BASE_SEED + self.config_id

    @property
    def fmt(self):
        return (self.m, self.n, self.p)

    @property
    def key(self) -> str:
        """The WORKLOADS key of this workload ("c2_333_zt", ...)."""
        return next(k for k, v in WORKLOADS.items() if v is self)


# BASELINE.json configs; R from SURVEY.md section 8(a); targets PAPER:11
WORKLOADS = {
    "c1_222_zt": Workload("(2,2,2) Z_T naive 8 -> 7, 64 walkers", 2, 2, 2, ZT, 32, 64, 7, 0),
    "c2_333_zt": Workload("(3,3,3) Z_T naive 27 -> 23, 16384 walkers", 3, 3, 3, ZT, 32, 16384, 23, 1),
    "c2_333_z2": Workload("(3,3,3) Z_2 naive 27 -> 23, 16384 walkers", 3, 3, 3, Z2, 32, 16384, 23, 11),
    "c3_444_zt": Workload("(4,4,4) Z_T naive 64 -> 49", 4, 4, 4, ZT, 96, 16384, 49, 2),
    "c3_444_z2": Workload("(4,4,4) Z_2 naive 64 -> 47", 4, 4, 4, Z2, 96, 16384, 47, 12),
    "c4_555_zt": Workload("(5,5,5) Z_T naive 125 -> 93", 5, 5, 5, ZT, 160, 16384, 93, 3),
    "c5_4512_zt": Workload("(4,5,12) Z_T naive 240 -> 179", 4, 5, 12, ZT, 256, 9472, 179, 4),
    "c5_5610_zt": Workload("(5,6,10) Z_T naive 300 -> 217", 5, 6, 10, ZT, 320, 9472, 217, 5),
    "c5_679_zt": Workload("(6,7,9) Z_T naive 378 -> 268", 6, 7, 9, ZT, 416, 9472, 268, 6),
}


def sample_walkers(total: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct walker indices in [0, total), always including 0 and total-1."""
    rng = np.random.default_rng(seed)
    k = min(k, total)
    pick = set([0, total - 1])
    while len(pick) < k:
        pick.add(int(rng.integers(total)))
    return np.array(sorted(pick), dtype=np.int64)


def perturbations(rank: int, width: int, ring: int, k: int, seed: int = 0):
    """k seeded single-coefficient perturbations (row, column, new value)."""
    rng = np.random.default_rng(seed)
    vals = [0, 1] if ring == Z2 else [-1, 0, 1]
    out = []
    for _ in range(k):
        out.append((int(rng.integers(rank)), int(rng.integers(width)), int(rng.choice(vals))))
    return out
