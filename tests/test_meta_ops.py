"""Meta operators: libfg's host implementation (bit-plane index maps)
against the oracle's (int8 definitions), byte-exact; every result verifies; ranks
follow the stated formulas; paper / closed-form pins."""
import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle

ZT, Z2 = 0, 1


@pytest.fixture(scope="module")
def fg():
    from paper_2511_20317_b200.build import build_libfg
    build_libfg()
    from paper_2511_20317_b200 import fg as mod
    return mod


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _schemes(orc):
    _, _, _, strassen = load_scheme("sec36_after.txt")
    _, _, _, s223 = load_scheme("scheme_2x2x3_r11.txt")
    w = orc.walker(3, 3, 3, ZT, 32, walker_id=2)
    w.seed_naive()
    w.walk(4000, 5)
    out = [((2, 2, 2), ZT, strassen), ((2, 2, 3), ZT, s223), ((3, 3, 3), ZT, w.rows()),
           ((2, 3, 4), ZT, orc.naive(2, 3, 4)), ((3, 2, 4), Z2, orc.naive(3, 2, 4))]
    wz = orc.walker(2, 3, 3, Z2, 32, walker_id=4)
    wz.seed_naive()
    wz.walk(3000, 8)
    out.append(((2, 3, 3), Z2, wz.rows()))
    return out


@pytest.mark.parametrize("op", ["transpose", "rotate", "swap_sizes", "project", "extend", "double"])
def test_unary_ops_match_oracle_and_verify(fg, orc, op):
    for fmt, ring, c in _schemes(orc):
        if op == "project" and fmt[2] < 2:
            continue
        nf, got = fg.fg_meta(op, fmt, c, ring)
        nf2, ref = orc.meta(op, fmt, c)
        assert nf == nf2 and np.array_equal(got, ref), (op, fmt)
        assert orc.verify(*nf, ring, got)[0] == 0, (op, fmt)
        r = c.shape[0]
        m, n, p = fmt
        if op == "extend":
            assert got.shape[0] == r + m * n
        elif op == "double":
            assert got.shape[0] == 2 * r
        elif op == "project":
            assert got.shape[0] <= r
        else:
            assert got.shape[0] == r


def test_merge_strassen_with_naive_gives_the_printed_rank(fg, orc):
    """merge((2,2,2:7), naive (2,2,1:4)) is a (2,2,3:11) scheme -- the rank of the
    example printed at PAPER:130-175."""
    _, _, _, strassen = load_scheme("sec36_after.txt")
    nf, got = fg.fg_meta("merge", (2, 2, 2), strassen, ZT, (2, 2, 1), orc.naive(2, 2, 1))
    assert nf == (2, 2, 3) and got.shape[0] == 11
    assert orc.verify(2, 2, 3, ZT, got)[0] == 0
    assert np.array_equal(got, orc.meta("merge", (2, 2, 2), strassen, (2, 2, 1), orc.naive(2, 2, 1))[1])


def test_product_strassen_squared(fg, orc):
    """Strassen x Strassen = (4,4,4:49), the Z_T rank of PAPER:699 (Table 5)."""
    _, _, _, strassen = load_scheme("sec36_after.txt")
    nf, got = fg.fg_meta("product", (2, 2, 2), strassen, ZT, (2, 2, 2), strassen)
    assert nf == (4, 4, 4) and got.shape[0] == 49
    assert orc.verify(4, 4, 4, ZT, got)[0] == 0
    assert np.array_equal(got, orc.meta("product", (2, 2, 2), strassen, (2, 2, 2), strassen)[1])
    # mixed formats and Z_2
    for (f1, c1, f2, c2, ring) in [((2, 3, 1), orc.naive(2, 3, 1), (3, 1, 2), orc.naive(3, 1, 2), ZT),
                                   ((2, 2, 2), strassen, (1, 2, 3), orc.naive(1, 2, 3), ZT),
                                   ((2, 2, 2), np.abs(strassen), (2, 1, 2), orc.naive(2, 1, 2), Z2)]:
        if ring == Z2 and orc.verify(*f1, Z2, c1)[0] != 0:
            continue
        nf, got = fg.fg_meta("product", f1, c1, ring, f2, c2)
        assert np.array_equal(got, orc.meta("product", f1, c1, f2, c2)[1])
        assert orc.verify(*nf, ring, got)[0] == 0


def test_swap_is_an_involution_on_the_format_and_project_of_naive(fg, orc):
    for fmt in [(2, 3, 4), (3, 3, 2)]:
        c = orc.naive(*fmt)
        nf, s1 = fg.fg_meta("swap_sizes", fmt, c)
        nf2, s2 = fg.fg_meta("swap_sizes", nf, s1)
        assert nf2 == fmt and orc.verify(*fmt, ZT, s2)[0] == 0
        nf, pr = fg.fg_meta("project", fmt, c)
        assert pr.shape[0] == fmt[0] * fmt[1] * (fmt[2] - 1)          # naive (m,n,p-1)
        assert orc.additions(*nf, pr) == nf[0] * nf[2] * (nf[1] - 1)


def test_capacity_and_domain_errors(fg, orc):
    c = orc.naive(4, 4, 4)
    with pytest.raises(fg.FgError):
        fg.fg_meta("product", (4, 4, 4), c, ZT, (3, 3, 3), orc.naive(3, 3, 3))   # 12x12 > 64 elements
    bad = orc.naive(2, 2, 2)
    bad[0, 0] = 2
    with pytest.raises(fg.FgError):
        fg.fg_meta("transpose", (2, 2, 2), bad)


def test_invariants_match_oracle_and_paper(fg, orc):
    """PAPER:515-524 on the rank-7 example: type X^2Y^2Z^2 + 6XYZ, rank sums (8,8,8);
    libfg (rank over GF(2^31-1)) equals the oracle (Bareiss over Q) everywhere."""
    m, n, p, s = load_scheme("sec36_after.txt")
    t, sums = fg.fg_type_invariant(m, n, p, ZT, s)
    assert t == {(2, 2, 2): 1, (1, 1, 1): 6} and sums == (8, 8, 8)
    for fmt, ring, c in _schemes(orc):
        t, sums = fg.fg_type_invariant(*fmt, ring, c)
        if ring == ZT:
            assert t == orc.type_invariant(*fmt, c)
        assert sum(t.values()) == c.shape[0]
    nf, sq = fg.fg_meta("product", (2, 2, 2), s, ZT, (2, 2, 2), s)
    assert fg.fg_type_invariant(*nf, ZT, sq)[0] == orc.type_invariant(*nf, sq)


def test_sym_invariant_matches_oracle(fg, orc):
    """libfg's symmetrised polynomial equals the oracle's on every scheme."""
    m, n, p, s = load_scheme("sec36_after.txt")
    assert fg.fg_sym_invariant(m, n, p, ZT, s) == {(2, 2, 2): 6, (1, 1, 1): 36}
    for fmt, ring, c in _schemes(orc):
        if ring == ZT:
            assert fg.fg_sym_invariant(*fmt, ring, c) == orc.sym_invariant(*fmt, c), fmt


def test_scheme_key_is_invariant_under_row_order_and_sign(fg, orc):
    m, n, p, before = load_scheme("sec36_before.txt")
    _, _, _, after = load_scheme("sec36_after.txt")
    k = fg.fg_scheme_key(m, n, p, ZT, after)
    assert fg.fg_scheme_key(m, n, p, ZT, before) == k          # same scheme
    rng = np.random.default_rng(0)
    assert fg.fg_scheme_key(m, n, p, ZT, after[rng.permutation(7)]) == k
    assert fg.fg_scheme_key(m, n, p, ZT, orc.naive(2, 2, 2)) != k


def test_resize_alg2_matches_oracle(fg, orc):
    """Alg. 2 (R31): libfg and the oracle take the same decisions from
    the same Philox words and produce byte-identical schemes, which verify; the op
    mix follows PAPER:378 (swap 1/2; project/product/double/extend 5/50/30/15)."""
    _, _, _, strassen = load_scheme("sec36_after.txt")
    _, _, _, s223 = load_scheme("scheme_2x2x3_r11.txt")
    bests = [((2, 2, 2), strassen), ((2, 2, 3), s223), ((2, 2, 1), orc.naive(2, 2, 1)),
             ((2, 3, 2), orc.naive(2, 3, 2))]
    starts = [((2, 2, 2), strassen), ((2, 2, 3), s223), ((3, 2, 2), orc.naive(3, 2, 2)),
              ((2, 3, 3), orc.naive(2, 3, 3))]
    ops = np.zeros(6, int)
    for t in range(400):
        fmt, c = starts[t % len(starts)]
        got = fg.fg_resize(fmt, c, bests, 160, 0x5EED, t, t * 7 + 1, thr_resize=3 << 30)
        ref = orc.resize(fmt, c, bests, 160, 0x5EED, t, t * 7 + 1, thr_resize=3 << 30)
        assert got[0] == ref[0] and got[2] == ref[2] and np.array_equal(got[1], ref[1]), t
        nf, out, op = got
        assert orc.verify(*nf, ZT, out)[0] == 0
        ops[op >> 1] += 1
    assert ops[1] > 0 and ops[2] + ops[3] + ops[4] + ops[5] > 50
    assert ops[3] > ops[4] > ops[2]             # product > double > project (50 / 30 / 5)


def test_registry_archive_deduplicates(fg, orc):
    """The archive (PAPER:291 persistent storage) holds each scheme once up to row order
    and sign rescaling (fg_scheme_key); invariants come with it."""
    from paper_2511_20317_b200.explore import Registry
    m, n, p, before = load_scheme("sec36_before.txt")
    _, _, _, after = load_scheme("sec36_after.txt")
    reg = Registry(0)
    reg.offer((2, 2, 2), 7, orc.additions(2, 2, 2, after), after)
    reg.offer((2, 2, 2), 7, orc.additions(2, 2, 2, before), before)             # same scheme
    reg.offer((2, 2, 2), 7, 18, after[np.random.default_rng(1).permutation(7)])  # row order
    assert len(reg.archive[(2, 2, 2)]) == 1
    reg.offer((2, 2, 2), 8, 4, orc.naive(2, 2, 2))
    assert len(reg.archive[(2, 2, 2)]) == 2 and reg.best[(2, 2, 2)][0] == 7
    key = next(iter(reg.archive[(2, 2, 2)]))
    t, sums, sym = reg.invariants((2, 2, 2), key)
    assert t == {(2, 2, 2): 1, (1, 1, 1): 6} and sums == (8, 8, 8)
    assert sym == {(2, 2, 2): 6, (1, 1, 1): 36}
