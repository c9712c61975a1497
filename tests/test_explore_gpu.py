"""Exploratory search: walk (GPU) + population sync + Resize (Alg. 2) over
several formats.  Every scheme of the population verifies after every round and the
search is deterministic (counter-based RNG end to end)."""
import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20317_b200 import fg as mod
    return mod


def _population():
    orc = Oracle()
    _, _, _, strassen = load_scheme("sec36_after.txt")
    _, _, _, s223 = load_scheme("scheme_2x2x3_r11.txt")
    return ([((2, 2, 2), strassen)] * 12 + [((2, 2, 1), orc.naive(2, 2, 1))] * 8 +
            [((2, 2, 3), s223)] * 12 + [((2, 3, 2), orc.naive(2, 3, 2))] * 8)


def _run(fg):
    import torch
    from paper_2511_20317_b200.explore import Explorer
    ex = Explorer(_population(), seed=77, stream=torch.cuda.current_stream().cuda_stream,
                  thr_resize=3 << 30)
    ops = []
    for _ in range(3):
        ops += ex.round(400)
        for f, c in ex.pop:
            assert fg.fg_verify(*f, 0, c)[0] == 0, f
    return ex, ops


def test_exploratory_rounds_verify_and_are_deterministic(fg):
    ex1, ops1 = _run(fg)
    ex2, ops2 = _run(fg)
    assert ops1 == ops2
    assert [f for f, _ in ex1.pop] == [f for f, _ in ex2.pop]
    assert all(np.array_equal(a[1], b[1]) for a, b in zip(ex1.pop, ex2.pop))
    assert len(ex1.formats()) >= 3 and len(ex1.registry.best) >= 4
    for f, (rank, adds, c) in ex1.registry.best.items():
        assert fg.fg_verify(*f, 0, c)[0] == 0 and len(c) == rank
    assert ex1.registry.best[(2, 2, 2)][0] == 7
    assert {op >> 1 for op in ops1} - {0} != set()          # some resize operations applied


# ---------------- oracle-driven exploratory loop (R31) ----------------
def _oracle_r_cap(rank, fmt):
    """The exploratory capacity policy (R31), restated: room for expands."""
    m, n, p = fmt
    need = max(rank + 8, int(rank * 1.25) + 2)
    if need <= 32 and max(m * n, n * p, p * m) <= 32:
        return 32
    for ns in (2, 3, 4, 5, 6, 8, 10, 13, 16):
        if 32 * ns >= need:
            return 32 * ns
    return 512


def _canon(orc, fmt, c):
    return sorted(map(bytes, orc.normalize(*fmt, c)))


def _oracle_explore(population, ring, seed, thr, rounds, steps):
    """The lifecycle of PAPER:266-293 with oracle walkers and the oracle's Alg. 2:
    rank assessment (registry of (rank, additions) bests), RandomWalk of every
    walker grouped by format (ids consecutive per sorted format, step counter restarted,
    key re-derived per round), the per-format best of the walk (R20: lexicographic
    (rank, additions, walker id), never worse than the loaded schemes'), then Resize of
    every walker against the registry's bests."""
    orc = Oracle()
    pop = [(tuple(f), np.array(c, dtype=np.int8)) for f, c in population]
    reg = {}

    def offer(f, rank, adds, c):
        if f not in reg or (rank, adds) < reg[f][:2]:
            reg[f] = (rank, adds, np.array(c, dtype=np.int8))

    for f, c in pop:
        offer(f, len(c), orc.additions(*f, c), c)
    all_ops = []
    for rnd in range(rounds):
        groups = {}
        for i, (f, _) in enumerate(pop):
            groups.setdefault(f, []).append(i)
        wseed = (seed * 0x9E3779B97F4A7C15 + rnd) & 0xFFFFFFFFFFFFFFFF
        base = 0
        for f in sorted(groups):
            idxs = groups[f]
            R = _oracle_r_cap(max(len(pop[i][1]) for i in idxs), f)
            recs = []
            for k, i in enumerate(idxs):
                w = orc.walker(*f, ring, R, walker_id=base + k)
                w.seed_rows(pop[i][1])
                s0 = w.rows(1)
                recs.append(((len(s0), orc.additions(*f, s0), base + k), s0))
                w.walk(steps, wseed)
                b = w.rows(1)
                recs.append(((len(b), orc.additions(*f, b), base + k), b))
                pop[i] = (f, w.rows(0))
            base += len(idxs)
            key, b = min(recs, key=lambda x: x[0])
            offer(f, key[0], key[1], b)
        bests = [(f, v[2]) for f, v in sorted(reg.items())]
        for i, (f, c) in enumerate(pop):
            nf, nc, op = orc.resize(f, c, bests, 512, seed, rnd, i, thr)
            pop[i] = (nf, nc)
            all_ops.append(op)
    return pop, reg, all_ops


def test_explorer_matches_oracle_loop(fg):
    """Explorer.round (GPU walks + libfg Resize) reproduces the oracle-driven exploratory
    loop walker by walker for 3 rounds: formats, every row, every Resize decision and the
    registry's (rank, additions) per format (scheme equal up to row order / sign)."""
    import torch
    from paper_2511_20317_b200.explore import Explorer
    pop0 = _population()
    seed, thr, steps = 77, 3 << 30, 400
    ex = Explorer(pop0, seed=seed, stream=torch.cuda.current_stream().cuda_stream, thr_resize=thr)
    ops = []
    for _ in range(3):
        ops += ex.round(steps)
    ref_pop, ref_reg, ref_ops = _oracle_explore(pop0, 0, seed, thr, 3, steps)
    assert ops == ref_ops
    assert len(ex.pop) == len(ref_pop)
    for i, ((f, c), (rf, rc)) in enumerate(zip(ex.pop, ref_pop)):
        assert f == rf, i
        assert np.array_equal(c, rc), i
    orc = Oracle()
    assert set(ex.registry.best) == set(ref_reg)
    for f, (rank, adds, c) in ref_reg.items():
        grank, gadds, gc = ex.registry.best[f]
        assert (grank, gadds) == (rank, adds), f
        assert _canon(orc, f, gc) == _canon(orc, f, c), f
    assert {op >> 1 for op in ops} - {0} != set()

