"""Pins of the CPU oracle against what PAPER.md and mathematics fix (T1-T6).

Citations are lines of /root/reference/PAPER.md (read-only; not read at run time:
the printed values live in tests/golden/).
"""
import itertools

import numpy as np
import pytest

from golden_io import load_philox_kat, load_scheme
from numpy_ref import first_failing, matmul_tensor, scheme_tensor
from oracle import Oracle

ZT, Z2 = 0, 1


@pytest.fixture(scope="module")
def orc():
    return Oracle()


# ---------------- T1: layout + verify ----------------
def test_t1_paper_2x2x3_scheme_verifies_in_ct_layout(orc):
    m, n, p, c = load_scheme("scheme_2x2x3_r11.txt")
    assert (m, n, p, c.shape[0]) == (2, 2, 3, 11)
    rc, ff = orc.verify(m, n, p, ZT, c)
    assert rc == 0 and ff == (-1, -1, -1)
    # the printed tensor equals the matmul tensor computed independently
    assert np.array_equal(scheme_tensor(m, n, p, c), matmul_tensor(m, n, p))


def test_t1_row_major_w_reading_fails(orc):
    """Read the printed W columns as row-major C (c11,c12,c13,c21,...) instead of
    the stated C^T order: the scheme must then FAIL (pins R2's w index k*m+i)."""
    m, n, p, c = load_scheme("scheme_2x2x3_r11.txt")
    mn, np_ = m * n, n * p
    W = c[:, mn + np_:]
    W2 = np.zeros_like(W)
    for q in range(p * m):
        i, k = divmod(q, p)          # row-major reading of column q
        W2[:, k * m + i] = W[:, q]
    c2 = np.concatenate([c[:, :mn + np_], W2], axis=1)
    rc, ff = orc.verify(m, n, p, ZT, c2)
    assert rc == 1
    assert ff == first_failing(m, n, p, c2)


def test_t1_paper_first_product_and_c11(orc):
    """m1 = (a11 + a22)(b11 + b22); c11 = m1 - m3 + m4 + m5."""
    m, n, p, c = load_scheme("scheme_2x2x3_r11.txt")
    U, V, W = c[:, :4], c[:, 4:10], c[:, 10:]
    assert list(U[0]) == [1, 0, 0, 1]
    assert list(V[0]) == [1, 0, 0, 0, 1, 0]        # b11 + b22 (b22 is column 4)
    assert list(W[:, 0]) == [1, 0, -1, 1, 1, 0, 0, 0, 0, 0, 0]


@pytest.mark.parametrize("fmt", [(1, 1, 1), (2, 2, 2), (2, 2, 3), (2, 3, 4), (3, 3, 3),
                                 (4, 4, 4), (3, 2, 5), (4, 5, 3)])
def test_naive_schemes_verify(orc, fmt):
    m, n, p = fmt
    c = orc.naive(m, n, p)
    assert c.shape[0] == m * n * p
    assert orc.verify(m, n, p, ZT, c) == (0, (-1, -1, -1))
    assert orc.verify(m, n, p, Z2, c) == (0, (-1, -1, -1))
    assert np.array_equal(scheme_tensor(m, n, p, c), matmul_tensor(m, n, p))


def test_verify_single_perturbations_fail_at_first_index(orc):
    """Every single-coefficient perturbation of the printed (2,2,3:11) scheme and of
    the (2,2,2:7) example fails, at the lexicographically first wrong equation."""
    rng = np.random.default_rng(1)
    for name in ["scheme_2x2x3_r11.txt", "sec36_after.txt"]:
        m, n, p, c = load_scheme(name)
        for l in range(c.shape[0]):
            for e in range(c.shape[1]):
                for val in (-1, 0, 1):
                    if val == c[l, e]:
                        continue
                    c2 = c.copy()
                    c2[l, e] = val
                    rc, ff = orc.verify(m, n, p, ZT, c2)
                    exp = first_failing(m, n, p, c2)
                    if exp is None:
                        assert rc == 0
                    else:
                        assert rc == 1 and ff == exp
    # Z_2: perturbations of the naive scheme
    m, n, p = 3, 3, 3
    c = orc.naive(m, n, p)
    for _ in range(50):
        c2 = c.copy()
        l, e = rng.integers(c.shape[0]), rng.integers(c.shape[1])
        c2[l, e] ^= 1
        rc, ff = orc.verify(m, n, p, Z2, c2)
        assert rc == 1 and ff == first_failing(m, n, p, c2, ring=1)


def test_verify_rejects_out_of_ring(orc):
    m, n, p = 2, 2, 2
    c = orc.naive(m, n, p)
    c[0, 0] = 2
    assert orc.verify(m, n, p, ZT, c)[0] == -3
    c = orc.naive(m, n, p)
    c[0, 0] = -1
    assert orc.verify(m, n, p, Z2, c)[0] == -3


# ---------------- T2: sign symmetry breaking ----------------
def test_t2_both_examples_verify(orc):
    for name in ["sec36_before.txt", "sec36_after.txt"]:
        m, n, p, c = load_scheme(name)
        assert (m, n, p, c.shape[0]) == (2, 2, 2, 7)
        assert orc.verify(m, n, p, ZT, c)[0] == 0


def test_t2_normalize_reproduces_printed_example(orc):
    m, n, p, before = load_scheme("sec36_before.txt")
    _, _, _, after = load_scheme("sec36_after.txt")
    got = orc.normalize(m, n, p, before)
    assert np.array_equal(got, after)
    # idempotent
    assert np.array_equal(orc.normalize(m, n, p, got), got)


# ---------------- T3: bit formulas PAPER:403-422 vs integers ----------------
def _encode(vals):
    d = np.zeros(len(vals), np.uint64)
    s = np.zeros(len(vals), np.uint64)
    for e in range(vals.shape[1]):
        d |= (vals[:, e] != 0).astype(np.uint64) << np.uint64(e)
        s |= (vals[:, e] < 0).astype(np.uint64) << np.uint64(e)
    return d, s


def _decode(d, s, L):
    out = np.zeros((len(d), L), np.int64)
    for e in range(L):
        nz = (d >> np.uint64(e)) & np.uint64(1)
        ng = (s >> np.uint64(e)) & np.uint64(1)
        out[:, e] = nz.astype(np.int64) * (1 - 2 * ng.astype(np.int64))
    return out


def test_t3_bit_arithmetic_exhaustive_length6(orc):
    L = 6
    vecs = np.array(list(itertools.product([-1, 0, 1], repeat=L)), dtype=np.int64)
    A = np.repeat(vecs, len(vecs), axis=0)
    B = np.tile(vecs, (len(vecs), 1))
    da, sa = _encode(A)
    db, sb = _encode(B)
    for op, sign in ((0, 1), (1, -1)):
        d, s, valid, eq, neg = orc.bits_batch(da, sa, db, sb, op)
        ref = A + sign * B
        ref_valid = np.all(np.abs(ref) <= 1, axis=1)
        assert np.array_equal(valid.astype(bool), ref_valid)
        got = _decode(d[ref_valid], s[ref_valid], L)
        assert np.array_equal(got, ref[ref_valid])
        assert np.all((s & ~d) == 0)            # signs subset of digits
        assert np.array_equal(eq.astype(bool), np.all(A == B, axis=1))
        nz = np.any(A != 0, axis=1)
        assert np.array_equal(neg.astype(bool), np.all(A == -B, axis=1) & nz)


def test_t3_spec_examples(orc):
    """SPEC:41-58 examples: [1,0,-1] -> digits 0b101 signs 0b100; [1]+[1] invalid."""
    d, s = _encode(np.array([[1, 0, -1]]))
    assert int(d[0]) == 0b101 and int(s[0]) == 0b100
    one_d, one_s = _encode(np.array([[1]]))
    _, _, valid, _, _ = orc.bits_batch(one_d, one_s, one_d, one_s, 0)
    assert valid[0] == 0
    _, _, valid, _, _ = orc.bits_batch(one_d, one_s, one_d, one_s, 1)
    assert valid[0] == 1


# ---------------- T4: naive additive complexity PAPER:656 ----------------
def test_t4_additions(orc):
    m, n, p, c = load_scheme("sec36_after.txt")
    assert int(np.count_nonzero(c)) == 36
    assert orc.additions(m, n, p, c) == 18       # 36 - 2*7 - 2*2 (Strassen's 18)
    for (m, n, p) in [(2, 2, 2), (3, 3, 3), (2, 3, 4), (4, 4, 4), (5, 5, 5)]:
        assert orc.additions(m, n, p, orc.naive(m, n, p)) == m * p * (n - 1)


# ---------------- T5: type invariant PAPER:515-517 ----------------
def test_t5_type_invariant_strassen(orc):
    for name in ["sec36_before.txt", "sec36_after.txt"]:
        m, n, p, c = load_scheme(name)
        assert orc.type_invariant(m, n, p, c) == {(2, 2, 2): 1, (1, 1, 1): 6}
    m, n, p = 3, 3, 3
    assert orc.type_invariant(m, n, p, orc.naive(m, n, p)) == {(1, 1, 1): 27}


# ---------------- symmetrised polynomial PAPER:519-521 ----------------
def _add(acc, d):
    for k, v in d.items():
        acc[k] = acc.get(k, 0) + v
    return acc


def test_sym_invariant_strassen_and_group_orbit(orc):
    """f on the rank-7 example = 6 x^2y^2z^2 + 36 xyz (the S_3 orbit of X^2Y^2Z^2 + 6XYZ,
    PAPER:515-517).  On walked schemes with an asymmetric type, f equals the sum of the
    type polynomials of the six schemes the meta operators produce from the scheme --
    rotations (cyclic (x,y,z)) and rotations of its transpose (a transposition) generate
    S_3 (R25/R26) -- and f is unchanged by those operators."""
    m, n, p, c = load_scheme("sec36_after.txt")
    assert orc.sym_invariant(m, n, p, c) == {(2, 2, 2): 6, (1, 1, 1): 36}
    asym = 0
    for fmt, seed in [((2, 3, 4), 3), ((3, 3, 3), 5), ((2, 2, 3), 9), ((3, 4, 2), 11)]:
        w = orc.walker(*fmt, 0, 32, walker_id=seed)
        w.seed_naive()
        w.walk(6000, seed)
        s = w.rows()
        f = orc.sym_invariant(*fmt, s)
        assert sum(f.values()) == 6 * s.shape[0]
        orbit = []
        for start in [(fmt, s), orc.meta("transpose", fmt, s)]:
            cur = start
            for _ in range(3):
                orbit.append(cur)
                cur = orc.meta("rotate", *cur)
        acc = {}
        for g_fmt, g_s in orbit:
            _add(acc, orc.type_invariant(*g_fmt, g_s))
            assert orc.sym_invariant(*g_fmt, g_s) == f
        assert acc == f, fmt
        t = orc.type_invariant(*fmt, s)
        asym += any(t.get((b, a, cc), 0) != v for (a, b, cc), v in t.items())
    assert asym >= 1        # the pin saw a scheme whose type polynomial is not symmetric


def test_matrix_rank_vs_numpy(orc):
    rng = np.random.default_rng(7)
    for _ in range(300):
        r, c = rng.integers(1, 9, size=2)
        a = rng.integers(-1, 2, size=(r, c)).astype(np.int8)
        if rng.random() < 0.3 and r > 1:
            a[-1] = np.clip(a[0] + a[-1] * 0, -1, 1)   # force dependence sometimes
        assert orc.matrix_rank(a) == np.linalg.matrix_rank(a.astype(np.float64))


# ---------------- T6: Philox4x32-10 known answers ----------------
def test_t6_philox_kat(orc):
    for ctr, key, out in load_philox_kat():
        assert list(orc.philox(ctr, key)) == out


def test_word_slot_addressing(orc):
    """R8: word t of step s = Philox(key=seed, ctr=(s_lo, s_hi, walker, t>>2))[t & 3]."""
    seed = 0x2511203170000002
    for s in (0, 1, 2**32 + 5):
        for wid in (0, 7, 16383):
            for t in range(23):
                block = orc.philox([s & 0xFFFFFFFF, s >> 32, wid, t >> 2],
                                   [seed & 0xFFFFFFFF, seed >> 32])
                assert orc.word(seed, s, wid, t) == block[t & 3]
