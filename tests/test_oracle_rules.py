"""Pins of three walk rules the paper fixes, stated independently of the oracle.

1. Expand preconditions and results (section 3.3.1, "Plus" / "Split"),
   under every role permutation: a numpy transcription of the two
   formulas decides accept / reject and the resulting rows for EVERY
   (kind, i, j, permutation) of small schemes, and `or_apply_expand` must agree
   exactly.  "u != u'" is read as R16's "distinct" (neither equal nor negated).
2. Reduction under every role pair: after `reduce_all` (Alg. 1
   "scheme.reduce()") no two terms may share two factors up to sign
   with a representable merged factor, found by brute force over all pairs of
   roles (the algebra x(x)y(x)z + sx(x)ty(x)z' = x(x)y(x)(z + st z'), not the
   oracle's role-pair table).  Splits under all six permutations create such pairs
   in every role pair, so each pair must be reachable.
3. The step order of Algorithm 1: the acceptance test (310-313)
   runs before reduce (315-317), which runs before the p_expand gate (319-321).
   Constructed single steps on a seed with exactly one reducible pair observe the
   order through best_rank and the expand counters.
"""
import itertools

import numpy as np
import pytest

from numpy_ref import matmul_tensor, normalize_row, scheme_tensor, split
from oracle import Oracle, OracleParams

ZT, Z2 = 0, 1
# R16's permutation table: pi maps the formula's (u, v, w) to scheme roles
PERMS = list(itertools.permutations(range(3)))
C_STEPS, C_FLIPS, C_EXPAND_OK, C_EXPAND_REJECT, C_MERGES, C_IMPROVEMENTS = 0, 2, 4, 5, 6, 9


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _facs(m, n, p, rows):
    return [f.astype(np.int64) for f in split(m, n, p, rows)]


def _in_ring(x, ring):
    return bool(np.all((x >= 0) & (x <= 1))) if ring == Z2 else bool(np.all(np.abs(x) <= 1))


def _ring(x, ring):
    return x % 2 if ring == Z2 else x


def _distinct(a, b, ring):
    """R16 reading of PAPER:219 / PAPER:227 "u^(i) != u^(j)": neither equal nor negated."""
    if np.array_equal(a, b):
        return False
    if ring == ZT and np.any(a) and np.array_equal(a, -b):
        return False
    return True


def _norm_rows(facs, idx, ring):
    if ring == Z2:
        return facs
    for l in idx:
        u, v, w = normalize_row(facs[0][l], facs[1][l], facs[2][l])
        facs[0][l], facs[1][l], facs[2][l] = u, v, w
    return facs


def expand_by_formula(m, n, p, ring, R, rows, plus, i, j, perm):
    """PAPER:217-231 written out on integer vectors; returns the new rows or None."""
    r = rows.shape[0]
    if r < 2 or r + 1 > R or i == j:
        return None
    A, B, Cr = PERMS[perm]
    F = _facs(m, n, p, rows)
    u_i, u_j, v_i, v_j, w_i, w_j = F[A][i], F[A][j], F[B][i], F[B][j], F[Cr][i], F[Cr][j]
    new = [np.concatenate([f, np.zeros((1, f.shape[1]), np.int64)]) for f in F]
    if plus:
        # needs u_i != u_j, v_i != v_j, w_i != w_j
        if not (_distinct(u_i, u_j, ring) and _distinct(v_i, v_j, ring) and _distinct(w_i, w_j, ring)):
            return None
        vs = _ring(v_i + v_j, ring)
        wd = _ring(w_j - w_i, ring)
        ud = _ring(u_j - u_i, ring)
        if not (_in_ring(vs, ring) and _in_ring(wd, ring) and _in_ring(ud, ring)):
            return None
        # u_i (x) (v_i+v_j) (x) w_i + u_i (x) v_j (x) (w_j-w_i) + (u_j-u_i) (x) v_j (x) w_j
        new[A][i], new[B][i], new[Cr][i] = u_i, vs, w_i
        new[A][j], new[B][j], new[Cr][j] = u_i, v_j, wd
        new[A][r], new[B][r], new[Cr][r] = ud, v_j, w_j
    else:
        # needs u_i != u_j
        if not _distinct(u_i, u_j, ring):
            return None
        ud = _ring(u_i - u_j, ring)
        if not _in_ring(ud, ring):
            return None
        # u_j (x) v_i (x) w_i + u_j (x) v_j (x) w_j + (u_i-u_j) (x) v_i (x) w_i
        new[A][i], new[B][i], new[Cr][i] = u_j, v_i, w_i
        new[A][r], new[B][r], new[Cr][r] = ud, v_i, w_i
    new = _norm_rows(new, [i, j, r], ring)
    return np.concatenate(new, axis=1)


def reducible_pairs(m, n, p, ring, rows):
    """Brute force over all pairs of terms and all pairs of roles: terms l, l' that
    share two factors up to sign, x_l = s x_l', y_l = t y_l', merge into
    x (x) y (x) (z_l + s t z_l'); reducible iff that factor is representable
    (PAPER:233-238 under any permutation)."""
    F = _facs(m, n, p, rows)
    out = []
    r = rows.shape[0]
    for a in range(r):
        for b in range(a + 1, r):
            for X, Y in ((0, 1), (0, 2), (1, 2)):
                Z = 3 - X - Y
                signs = []
                for role in (X, Y):
                    if not np.any(F[role][a]):
                        signs = None
                        break
                    if np.array_equal(F[role][a], F[role][b]):
                        signs.append(1)
                    elif ring == ZT and np.array_equal(F[role][a], -F[role][b]):
                        signs.append(-1)
                    else:
                        signs = None
                        break
                if signs is None:
                    continue
                z = _ring(F[Z][a] + signs[0] * signs[1] * F[Z][b], ring)
                if _in_ring(z, ring):
                    out.append((a, b, X, Y))
    return out


def has_zero_factor(m, n, p, rows):
    return any(not np.any(f[l]) for f in _facs(m, n, p, rows) for l in range(rows.shape[0]))


def tensor_ok(m, n, p, ring, rows):
    D = scheme_tensor(m, n, p, rows) - matmul_tensor(m, n, p)
    return not np.any(_ring(D, ring))


def _walked(orc, fmt, ring, steps, seed, R=64, wid=0):
    m, n, p = fmt
    w = orc.walker(m, n, p, ring, R, walker_id=wid)
    assert w.seed_naive() == 0
    w.walk(steps, seed)
    return w


# ------------------------- 1. expand preconditions ---------------------------

@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("fmt,steps", [((2, 2, 2), 0), ((2, 2, 2), 40), ((2, 2, 3), 120),
                                       ((3, 3, 3), 0), ((3, 3, 3), 400)])
def test_expand_accepts_iff_paper_preconditions(orc, ring, fmt, steps):
    m, n, p = fmt
    R = 64
    base = _walked(orc, fmt, ring, steps, 0x5EED + steps)
    rows = base.rows()
    r = rows.shape[0]
    seen = {"plus": [0, 0], "split": [0, 0]}
    # a subsample of ordered pairs on the larger scheme keeps this to seconds
    pairs = [(i, j) for i in range(r) for j in range(r) if i != j]
    if len(pairs) > 160:
        pick = np.random.default_rng(r).choice(len(pairs), 160, replace=False)
        pairs = [pairs[k] for k in pick]
    for plus in (0, 1):
        for (i, j) in pairs:
            for perm in range(6):
                exp = expand_by_formula(m, n, p, ring, R, rows, plus, i, j, perm)
                w = orc.walker(m, n, p, ring, R)
                assert w.seed_rows(rows) == 0
                ok = w.apply_expand(plus, i, j, perm)
                assert bool(ok) == (exp is not None), (plus, i, j, perm)
                if ok:
                    got = w.rows()
                    assert np.array_equal(got.astype(np.int64), exp), (plus, i, j, perm)
                    assert tensor_ok(m, n, p, ring, got)
                seen["plus" if plus else "split"][bool(ok)] += 1
    # both outcomes occur for both kinds, so neither branch is vacuous
    assert all(v[0] > 0 and v[1] > 0 for v in seen.values()), seen


def test_plus_needs_all_three_factors_distinct(orc):
    """PAPER:219 on naive (2,2,2): rows 0 and 1 share u = a11 (naive row order
    l = (i*n+j)*p+k), so plus is rejected for every permutation that puts a shared
    role on any of u, v, w -- which for a pair sharing one factor is all of them."""
    m = n = p = 2
    w0 = orc.walker(m, n, p, ZT, 16)
    w0.seed_naive()
    rows = w0.rows()
    F = _facs(m, n, p, rows)
    assert np.array_equal(F[0][0], F[0][1])
    for perm in range(6):
        w = orc.walker(m, n, p, ZT, 16)
        w.seed_rows(rows)
        assert w.apply_expand(1, 0, 1, perm) == 0
    # split needs only the formula's u distinct: perms whose u-role is not U apply
    for perm in range(6):
        w = orc.walker(m, n, p, ZT, 16)
        w.seed_rows(rows)
        assert bool(w.apply_expand(0, 0, 1, perm)) == (PERMS[perm][0] != 0), perm


def test_expand_respects_capacity(orc):
    m = n = p = 2
    w0 = orc.walker(m, n, p, ZT, 8)
    w0.seed_naive()
    rows = w0.rows()
    for plus, perm in itertools.product((0, 1), range(6)):
        w = orc.walker(m, n, p, ZT, 8)
        w.seed_rows(rows)
        assert w.apply_expand(plus, 0, 7, perm) == 0
        assert expand_by_formula(m, n, p, ZT, 8, rows, plus, 0, 7, perm) is None


# ------------------------- 2. reduction in every role pair -------------------

@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("fmt,steps", [((2, 2, 2), 30), ((3, 3, 3), 300), ((2, 3, 4), 500)])
def test_reduce_all_leaves_no_reducible_pair(orc, ring, fmt, steps):
    """Split under each of the six permutations (which leaves the new row sharing
    the formula's v and w with row i, i.e. any role pair) and run reduce_all: the
    brute force must find no reducible pair and no zero factor afterwards."""
    m, n, p = fmt
    base = _walked(orc, fmt, ring, steps, 0xAB + steps, R=96)
    rows = base.rows()
    r = rows.shape[0]
    hit_pairs = set()
    rng = np.random.default_rng(steps)
    for perm in range(6):
        done = 0
        for _ in range(200):
            i, j = (int(x) for x in rng.choice(r, 2, replace=False))
            w = orc.walker(m, n, p, ring, 96)
            assert w.seed_rows(rows) == 0
            if not w.apply_expand(0, i, j, perm):
                continue
            before = w.rows()
            found = reducible_pairs(m, n, p, ring, before)
            # the split's own pair (i, r) shares the roles PERMS[perm][1:] ...
            B, Cr = sorted(PERMS[perm][1:])
            assert (min(i, r), max(i, r), B, Cr) in found
            hit_pairs.add((B, Cr))
            w.reduce_all()
            after = w.rows()
            assert reducible_pairs(m, n, p, ring, after) == []
            assert not has_zero_factor(m, n, p, after)
            assert after.shape[0] <= r
            assert tensor_ok(m, n, p, ring, after)
            done += 1
            if done == 3:
                break
        assert done > 0, perm
    assert hit_pairs == {(0, 1), (0, 2), (1, 2)}


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_local_reduce_merges_split_pair_in_every_role_pair(orc, ring):
    """R12 after a flip checks the touched rows against all rows with the same
    two-shared-factor predicate: local_reduce(i, r) right after a split at (i, j)
    must merge the split pair back whatever role pair it shares."""
    m = n = p = 3
    base = _walked(orc, (m, n, p), ring, 250, 0x77, R=64)
    rows = base.rows()
    r = rows.shape[0]
    rng = np.random.default_rng(5)
    for perm in range(6):
        done = 0
        for _ in range(200):
            i, j = (int(x) for x in rng.choice(r, 2, replace=False))
            w = orc.walker(m, n, p, ring, 64)
            w.seed_rows(rows)
            if not w.apply_expand(0, i, j, perm):
                continue
            w.local_reduce(i, r)
            after = w.rows()
            assert after.shape[0] <= r
            assert tensor_ok(m, n, p, ring, after)
            # no reducible pair may involve the rows local_reduce finished on: the
            # merge target min(i, r) = i survives unless it vanished
            if after.shape[0] == r and not has_zero_factor(m, n, p, after):
                assert all(i not in (a, b) for a, b, _, _ in reducible_pairs(m, n, p, ring, after))
            done += 1
            if done == 2:
                break
        assert done > 0, perm


# ------------------------- 3. Alg. 1 step order ------------------------------

def _split_seed(m, n, p):
    """Naive (m,n,p) with term 0 = u0 (x) v0 (x) e_c written as two terms
    u0 (x) v0 (x) (e_c + e_d) + u0 (x) v0 (x) (-e_d): a valid scheme of rank mnp+1
    with exactly one reducible pair (sharing u and v)."""
    mn, np_, pm = m * n, n * p, p * m
    rows = []
    for i in range(m):
        for j in range(n):
            for k in range(p):
                u = np.zeros(mn, np.int8); u[i * n + j] = 1
                v = np.zeros(np_, np.int8); v[j * p + k] = 1
                w = np.zeros(pm, np.int8); w[k * m + i] = 1
                rows.append(np.concatenate([u, v, w]))
    rows = np.array(rows)
    # e_d = the w of terms (i,j,k) = (1, *, 1): none shares u0 = a_11 or v0 = b_11
    d = 1 * m + 1
    extra = rows[0].copy()
    rows[0, mn + np_ + d] = 1
    extra[mn + np_:] = 0
    extra[mn + np_ + d] = -1
    return np.concatenate([rows, extra[None]], axis=0)


def _one_step(orc, rows, wid, **kw):
    m = n = p = 3
    w = orc.walker(m, n, p, ZT, 40, walker_id=wid)
    assert w.seed_rows(rows) == 0
    prm = OracleParams.default(**kw)
    w.walk(1, 0x0DE5, prm)
    return w, prm


def _clean_flip_walkers(orc, rows, count):
    """Walker ids whose step 0 is a successful flip that local reduction does not
    touch (with reduce and expand switched off the rank stays mnp+1)."""
    r0 = rows.shape[0]
    out = []
    for wid in range(200):
        w, _ = _one_step(orc, rows, wid, thr_accept_eq=0, thr_reduce=0, thr_expand=0)
        if w.cnt[C_FLIPS] == 1 and w.r == r0 and reducible_pairs(3, 3, 3, ZT, w.rows()):
            out.append(wid)
            if len(out) == count:
                break
    assert len(out) == count
    return out


def test_seed_has_exactly_one_reducible_pair(orc):
    rows = _split_seed(3, 3, 3)
    assert orc.verify(3, 3, 3, ZT, rows)[0] == 0
    assert reducible_pairs(3, 3, 3, ZT, rows.astype(np.int64)) == [(0, 27, 0, 1)]


def test_accept_runs_before_reduce(orc):
    """PAPER:310-313 precede PAPER:315-317: in a step whose flip leaves the pair
    alone, reduce() lowers the rank AFTER the acceptance test, so best_rank keeps
    the seeded rank until the next successful flip accepts the lower rank."""
    rows = _split_seed(3, 3, 3)
    r0 = rows.shape[0]
    for wid in _clean_flip_walkers(orc, rows, 4):
        w, prm = _one_step(orc, rows, wid, thr_accept_eq=0, thr_reduce=0xFFFFFFFF, thr_expand=0)
        assert w.r == r0 - 1 and w.cnt[C_MERGES] == 1
        assert w.best_r == r0 and w.cnt[C_IMPROVEMENTS] == 0
        # the next successful flip sees rank < best_rank
        for _ in range(50):
            flips = int(w.cnt[C_FLIPS])
            w.walk(1, 0x0DE5, prm)
            if w.cnt[C_FLIPS] > flips:
                break
        assert w.best_r <= r0 - 1 and w.cnt[C_IMPROVEMENTS] >= 1


def test_expand_gate_sees_rank_after_reduce(orc):
    """PAPER:319 "scheme.rank <= best_rank + 2" is evaluated after reduce()
    (PAPER:315-317).  With slack -1 the gate passes only at rank mnp, which the
    step reaches only through that reduce: an expand must be attempted."""
    rows = _split_seed(3, 3, 3)
    r0 = rows.shape[0]
    for wid in _clean_flip_walkers(orc, rows, 4):
        w, _ = _one_step(orc, rows, wid, thr_accept_eq=0, thr_reduce=0xFFFFFFFF,
                         thr_expand=0xFFFFFFFF, expand_slack=-1)
        assert w.cnt[C_MERGES] >= 1
        assert w.cnt[C_EXPAND_OK] + w.cnt[C_EXPAND_REJECT] == 1
        assert w.best_r == r0
        # without the reduce the gate must stay shut
        w2, _ = _one_step(orc, rows, wid, thr_accept_eq=0, thr_reduce=0,
                          thr_expand=0xFFFFFFFF, expand_slack=-1)
        assert w2.cnt[C_EXPAND_OK] + w2.cnt[C_EXPAND_REJECT] == 0 and w2.r == r0


def test_expand_gate_sees_best_after_accept(orc):
    """PAPER:319's best_rank is the one PAPER:310-313 just updated: with slack -1,
    a step whose flip is accepted at equal rank keeps the gate shut, and a step
    whose rank drops below best (local merge) opens it only after acceptance."""
    rows = _split_seed(3, 3, 3)
    r0 = rows.shape[0]
    # accepted at equal rank (thr_eq max): best = r0, gate r0 <= r0 - 1 shut
    for wid in _clean_flip_walkers(orc, rows, 3):
        w, _ = _one_step(orc, rows, wid, thr_accept_eq=0xFFFFFFFF, thr_reduce=0,
                         thr_expand=0xFFFFFFFF, expand_slack=-1)
        assert w.cnt[C_EXPAND_OK] + w.cnt[C_EXPAND_REJECT] == 0
    # find steps where the flip's local reduction merges the pair: r0-1 < best r0 is
    # accepted first, best becomes r0-1, so the gate r0-1 <= r0-2 is shut
    n_seen = 0
    for wid in range(300):
        w, _ = _one_step(orc, rows, wid, thr_accept_eq=0, thr_reduce=0,
                         thr_expand=0xFFFFFFFF, expand_slack=-1)
        if w.cnt[C_FLIPS] == 1 and w.cnt[C_MERGES] >= 1:
            assert w.best_r == w.r < r0
            assert w.cnt[C_IMPROVEMENTS] == 1
            assert w.cnt[C_EXPAND_OK] + w.cnt[C_EXPAND_REJECT] == 0
            n_seen += 1
    assert n_seen > 0


def test_fallback_expand_has_no_rank_gate(orc):
    """PAPER:305-307 "if not scheme.try_flip(): scheme.expand(); continue" carries
    no rank condition (unlike PAPER:319): on the rank-7 example of PAPER:467-497,
    which has no flip candidate, every step attempts an expand even when the
    p_expand gate could never pass (slack -5)."""
    from golden_io import load_scheme
    m, n, p, c = load_scheme("sec36_after.txt")
    applied = 0
    for wid in range(16):
        w = orc.walker(m, n, p, ZT, 32, walker_id=wid)
        assert w.seed_rows(c) == 0
        w.walk(1, 3, OracleParams.default(expand_slack=-5, thr_expand=0xFFFFFFFF))
        assert w.cnt[C_FLIPS] == 0 and w.cnt[C_EXPAND_OK] + w.cnt[C_EXPAND_REJECT] == 1
        assert w.r == 7 + int(w.cnt[C_EXPAND_OK])
        applied += w.r == 8
    assert applied > 0
