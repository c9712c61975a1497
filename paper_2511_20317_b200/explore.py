"""Exploratory search (the FlipGraphGPU lifecycle of PAPER:266-293).

One round = (3) RandomWalk of every walker on the GPU (fg_walk, one fg_ctx per
matrix format), (5) population synchronisation: the best scheme of every format
(fg_best) enters the registry, then (4) Resize: every walker's scheme goes through
Alg. 2 on the host (fg_resize) against the registry's bests, and the population is
regrouped by format for the next round.  Every computation is in libfg (the walk
kernels on the device, the meta operators and Resize in its host code); this module
only moves schemes between contexts.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import fg


def _r_cap(rank: int, fmt) -> int:
    """Row capacity for a format: room for expands above the current rank."""
    m, n, p = fmt
    need = max(rank + 8, int(rank * 1.25) + 2)
    if need <= 32 and max(m * n, n * p, p * m) <= 32:
        return 32
    for ns in (2, 3, 4, 5, 6, 8, 10, 13, 16):
        if 32 * ns >= need:
            return 32 * ns
    return 512


def scheme_additions(fmt, ring, coeffs) -> int:
    """Naive additions of a scheme, computed by libfg (fg_record_pack)."""
    c = np.asarray(coeffs, dtype=np.int8)
    r_cap = max(1, c.shape[0])
    rec = fg.fg_record_pack(*fmt, ring, r_cap, c, 0)
    return int(fg.fg_record_unpack(rec, r_cap)["additions"])


@dataclass
class Registry:
    """Best scheme per format: lexicographic (rank, additions).
    `archive` is the persistent store of discoveries: every distinct scheme
    ever offered, per format, de-duplicated by its canonical key (fg_scheme_key: equal up
    to row order and the sign rescaling of PAPER:429), with its invariants
     for novelty checks."""
    ring: int = fg.FG_ZT
    best: dict = field(default_factory=dict)     # fmt -> (rank, additions, coeffs)
    archive: dict = field(default_factory=dict)  # fmt -> {key: (rank, additions, coeffs)}

    def offer(self, fmt, rank, adds, coeffs):
        c = np.array(coeffs, dtype=np.int8)
        key = fg.fg_scheme_key(*fmt, self.ring, c)
        self.archive.setdefault(fmt, {}).setdefault(key, (rank, adds, c))
        cur = self.best.get(fmt)
        if cur is None or (rank, adds) < (cur[0], cur[1]):
            self.best[fmt] = (rank, adds, c)

    def schemes(self):
        return [(f, v[2]) for f, v in sorted(self.best.items())]

    def invariants(self, fmt, key):
        """(type polynomial, rank sums, symmetrised polynomial) of an archived scheme."""
        _, _, c = self.archive[fmt][key]
        t, sums = fg.fg_type_invariant(*fmt, self.ring, c)
        return t, sums, fg.fg_sym_invariant(*fmt, self.ring, c)


class Explorer:
    def __init__(self, population, ring=fg.FG_ZT, seed=0x2511, device=0, stream=None,
                 thr_resize=1 << 30, params=None):
        """population: list of ((m, n, p), int8 coeffs) -- the initial schemes
        (naive or loaded; duplicated by the caller to fill N)."""
        self.pop = [(tuple(f), np.array(c, dtype=np.int8)) for f, c in population]
        self.ring, self.seed, self.device, self.stream = ring, seed, device, stream
        self.thr_resize = thr_resize
        self.params = params
        self.registry = Registry(ring)
        self.round_no = 0
        for f, c in self.pop:
            rc, _ = fg.fg_verify(*f, ring, c)
            if rc != 0:
                raise ValueError(f"seed scheme {f} does not verify")
            self.registry.offer(f, len(c), scheme_additions(f, ring, c), c)

    def walk(self, steps: int):
        """Walk every walker `steps` Alg. 1 iterations, grouped by format."""
        groups = {}
        for idx, (f, c) in enumerate(self.pop):
            groups.setdefault(f, []).append(idx)
        wseed = (self.seed * 0x9E3779B97F4A7C15 + self.round_no) & 0xFFFFFFFFFFFFFFFF
        base = 0
        for f in sorted(groups):
            idxs = groups[f]
            R = _r_cap(max(len(self.pop[i][1]) for i in idxs), f)
            g = fg.FlipGraph(*f, self.ring, R, len(idxs), base, self.device, self.stream)
            base += len(idxs)
            g.load_walkers([self.pop[i][1] for i in idxs])
            g.walk(steps, wseed, self.params)
            got = g.get_walkers()
            for k, i in enumerate(idxs):
                self.pop[i] = (f, got["rows"][k][: got["r"][k]].copy())
            b = g.best()
            self.registry.offer(f, b["rank"], b["additions"], b["coeffs"])
            g.close()

    def resize(self):
        """Alg. 2 on every walker against the registry's bests (host, fg_resize)."""
        bests = self.registry.schemes()
        ops = []
        for i, (f, c) in enumerate(self.pop):
            nf, nc, op = fg.fg_resize(f, c, bests, 512, self.seed, self.round_no, i, self.ring,
                                      self.thr_resize)
            self.pop[i] = (nf, nc)
            ops.append(op)
        return ops

    def round(self, steps: int):
        self.walk(steps)
        ops = self.resize()
        self.round_no += 1
        return ops

    def formats(self):
        return sorted({f for f, _ in self.pop})

    def diversity(self):
        """Number of distinct schemes in the population (canonical keys)."""
        return len({(f, fg.fg_scheme_key(*f, self.ring, c)) for f, c in self.pop})
