"""Oracle walk properties pinned by the paper and by brute force (no GPU).

PAPER:208-241 fixes what a flip / plus / split / reduction computes (all preserve
the tensor); PAPER:11 fixes that (2,2,2) has a rank-7 scheme (Strassen) and
PAPER:515-524 its invariants; closed forms give the naive candidate counts.
"""
import numpy as np
import pytest

from golden_io import load_scheme
from numpy_ref import (brute_force_flips, matmul_tensor, normalize_row, scheme_tensor, split)
from oracle import Oracle, OracleParams

ZT, Z2 = 0, 1


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _tensor_ok(m, n, p, rows, ring=ZT):
    T = scheme_tensor(m, n, p, rows) - matmul_tensor(m, n, p)
    if ring == Z2:
        T = T % 2
    return not np.any(T)


def _normalize_rows(m, n, p, rows, idx):
    U, V, W = split(m, n, p, rows)
    out = np.array(rows, dtype=np.int64)
    for l in idx:
        u, v, w = normalize_row(U[l], V[l], W[l])
        out[l] = np.concatenate([u, v, w])
    return out


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_naive_candidate_count_closed_form(orc, k):
    """Naive (k,k,k): rows sharing u=e_ij number p, sharing v=e_jk number m, sharing
    w=e_ki number n, so |C| = mn*C(p,2) + np*C(m,2) + pm*C(n,2) (12/81/288/750)."""
    m = n = p = k
    w = orc.walker(m, n, p, ZT, m * n * p + 8)
    assert w.seed_naive() == 0
    c2 = lambda x: x * (x - 1) // 2
    assert w.count_candidates() == m * n * c2(p) + n * p * c2(m) + p * m * c2(n)
    assert [12, 81, 288, 750][k - 2] == w.count_candidates()


@pytest.mark.parametrize("fmt,name", [((2, 2, 2), None), ((2, 2, 3), "scheme_2x2x3_r11.txt"),
                                      ((3, 3, 2), None)])
def test_flip_moves_match_brute_force(orc, fmt, name):
    """Every (candidate, d, e) move of the oracle equals one brute-force flip of
    PAPER:208-215 under some role permutation, and the multisets coincide."""
    m, n, p = fmt
    if name:
        _, _, _, seedc = load_scheme(name)
        seedc = orc.normalize(m, n, p, seedc)
    else:
        seedc = orc.naive(m, n, p)
    w = orc.walker(m, n, p, ZT, 64)
    assert w.seed_rows(seedc) == 0
    base = w.rows()
    ncand = w.count_candidates()
    got = []
    for c in range(ncand):
        for d in (0, 1):
            for e in (0, 1):
                w2 = orc.walker(m, n, p, ZT, 64)
                w2.seed_rows(seedc)
                ok = w2.apply_flip(c, d, e)
                got.append((ok, w2.rows().tobytes() if ok else None))
    bf = brute_force_flips(m, n, p, base)
    assert len(bf) == 4 * ncand
    exp = []
    for rows, safe, (X, i, j) in bf:
        if safe:
            exp.append((1, _normalize_rows(m, n, p, rows, [i, j]).astype(np.int8).tobytes()))
        else:
            exp.append((0, None))
    assert sorted(got, key=repr) == sorted(exp, key=repr)
    for ok, rb in got:
        if ok:
            rows = np.frombuffer(rb, np.int8).reshape(base.shape)
            assert _tensor_ok(m, n, p, rows)
    if fmt == (2, 2, 2):
        assert ncand == 12 and sum(ok for ok, _ in got) == 48
        assert len({rb for ok, rb in got if ok}) == 48          # 48 distinct neighbours
    if name:
        assert ncand == 6 and sum(ok for ok, _ in got) == 24


def test_strassen_has_no_flip_and_takes_expand(orc):
    """The rank-7 example of PAPER:467-497 has no two terms sharing a factor, so
    try_flip fails and Alg.1 takes the expand branch."""
    m, n, p, c = load_scheme("sec36_after.txt")
    w = orc.walker(m, n, p, ZT, 32)
    assert w.seed_rows(c) == 0
    assert w.count_candidates() == 0
    w.walk(1, 99)
    cnt = w.cnt
    assert cnt[3] == 1 and cnt[1] == 0 and cnt[4] + cnt[5] == 1
    assert _tensor_ok(m, n, p, w.rows())


@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("fmt", [(2, 2, 2), (3, 3, 3), (2, 3, 4)])
def test_expand_preserves_tensor(orc, ring, fmt):
    m, n, p = fmt
    rng = np.random.default_rng(3)
    w = orc.walker(m, n, p, ring, 200)
    w.seed_naive()
    w.walk(300, 5)                         # move away from naive first
    applied = 0
    for _ in range(200):
        r0 = w.r
        i, j = rng.choice(r0, size=2, replace=False)
        ok = w.apply_expand(int(rng.integers(2)), int(i), int(j), int(rng.integers(6)))
        applied += ok
        assert w.r == r0 + ok
        assert _tensor_ok(m, n, p, w.rows(), ring)
        if w.r > 150:
            break
    assert applied > 0


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_split_then_reduce_restores_rank(orc, ring):
    """A split leaves rows i and r sharing v and w; reduce_all
     merges them, so the rank returns and the tensor is kept."""
    m, n, p = 3, 3, 3
    w = orc.walker(m, n, p, ring, 64)
    w.seed_naive()
    w.walk(200, 11)
    r0 = w.r
    done = False
    for i in range(r0):
        for j in range(r0):
            if i != j and w.apply_expand(0, i, j, 0):
                done = True
                break
        if done:
            break
    assert done and w.r == r0 + 1
    w.reduce_all()
    assert w.r <= r0
    assert _tensor_ok(m, n, p, w.rows(), ring)


@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("fmt,R", [((3, 3, 3), 32), ((2, 3, 4), 40), ((4, 4, 4), 96)])
def test_walk_preserves_tensor_and_best_verifies(orc, ring, fmt, R):
    m, n, p = fmt
    w = orc.walker(m, n, p, ring, R, walker_id=5)
    w.seed_naive()
    for _ in range(20):
        w.walk(250, 0x1234 + ring)
        assert 1 <= w.r <= R
        assert _tensor_ok(m, n, p, w.rows(), ring)
        assert orc.verify(m, n, p, ring, w.rows(1))[0] == 0
        assert w.best_r == w.rows(1).shape[0]
    cnt = w.cnt
    assert cnt[0] == 5000 and cnt[11] == 0                  # steps, no verify failure
    assert cnt[2] + cnt[3] == cnt[0]                         # each step flips or fails
    # rank bookkeeping: r = seed + expands - merges - zero removals
    assert w.r == m * n * p + cnt[4] - cnt[6] - cnt[7]


def test_capacity_rejects_expand(orc):
    """R1/R16: with R equal to the naive rank no expand can be applied."""
    w = orc.walker(2, 2, 2, ZT, 8)
    w.seed_naive()
    w.walk(3000, 77)
    assert w.r <= 8 and w.cnt[4] == 0


def test_rank_one_degenerate(orc):
    """(1,1,1:1): no flip candidate, expand needs r >= 2: every step is a failed
    flip and a rejected expand."""
    w = orc.walker(1, 1, 1, ZT, 4)
    w.seed_naive()
    w.walk(100, 1)
    assert w.r == 1 and w.cnt[3] == 100 and w.cnt[5] == 100 and w.cnt[4] == 0


def test_phase_split_is_invisible(orc):
    """Counter-based RNG (R8): 3 calls of 700 steps == one call of 2100 steps."""
    a = orc.walker(3, 3, 3, ZT, 32, walker_id=9)
    b = orc.walker(3, 3, 3, ZT, 32, walker_id=9)
    a.seed_naive()
    b.seed_naive()
    a.walk(2100, 42)
    for _ in range(3):
        b.walk(700, 42)
    assert a.digest == b.digest and a.r == b.r and a.best_r == b.best_r
    assert np.array_equal(a.rows(), b.rows()) and np.array_equal(a.cnt, b.cnt)


def test_run_walkers_thread_invariant(orc):
    r1 = orc.run_walkers(3, 3, 3, ZT, 32, 16, 100, 500, 7, threads=1)
    r8 = orc.run_walkers(3, 3, 3, ZT, 32, 16, 100, 500, 7, threads=8)
    for k in r1:
        assert np.array_equal(r1[k], r8[k])
    w = orc.walker(3, 3, 3, ZT, 32, walker_id=103)
    w.seed_naive()
    w.walk(500, 7)
    assert w.digest == r1["digest"][3]


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_rediscovers_strassen_rank7(orc, ring):
    """(2,2,2) has a rank-7 scheme.  All 64 walkers of config C1 reach
    rank 7 from naive; each rank-7 best verifies and, being Strassen up to the de
    Groote isotropy (external fact), carries the invariant X^2Y^2Z^2 + 6XYZ
     -- in Z_T; Z_2 schemes are only checked mod 2."""
    res = orc.run_walkers(2, 2, 2, ring, 32, 64, 0, 60000, 0x2511203170000000 + ring)
    assert np.all(res["best_r"] == 7), res["best_r"]
    for k in range(64):
        best = res["best"][k][:7]
        assert orc.verify(2, 2, 2, ring, best)[0] == 0
        if ring == ZT:
            assert orc.type_invariant(2, 2, 2, best) == {(2, 2, 2): 1, (1, 1, 1): 6}
            assert _tensor_ok(2, 2, 2, best)
    assert np.all(res["cnt"][:, 11] == 0)
