"""R24 naive-complexity minimisation (Table 4) in the oracle:
pinned by the paper's additions metric and by invariants of the mode."""
import numpy as np
import pytest

from golden_io import load_scheme
from numpy_ref import matmul_tensor, scheme_tensor
from oracle import Oracle, OracleParams

CM = OracleParams.default(mode=1)


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def test_strassen_has_no_move(orc):
    """The rank-7 example of PAPER:467-497 has no flip: nothing changes, 18 stays."""
    m, n, p, c = load_scheme("sec36_after.txt")
    w = orc.walker(m, n, p, 0, 16)
    w.seed_rows(c)
    w.walk(500, 3, CM)
    assert w.best_adds == 18 and w.r == 7 and np.array_equal(w.rows(1), c)
    assert w.cnt[2] == 0 and w.cnt[3] == 500


@pytest.mark.parametrize("fmt", [(2, 2, 2), (2, 3, 2), (3, 3, 3)])
def test_naive_is_at_the_lower_bound(orc, fmt):
    """Every row has >= 3 nonzeros, so additions >= 3r - 2r - mp = r - mp; the naive
    scheme meets it (m p (n-1)): the mode can never report fewer."""
    m, n, p = fmt
    w = orc.walker(m, n, p, 0, 32, walker_id=1)
    w.seed_naive()
    w.walk(3000, 5, CM)
    r = m * n * p
    assert w.r == r and w.best_adds == r - m * p == m * p * (n - 1)


@pytest.mark.parametrize("ring", [0, 1])
def test_walked_scheme_gets_cheaper_and_stays_correct(orc, ring):
    m, n, p = 3, 3, 3
    w = orc.walker(m, n, p, ring, 32, walker_id=5)
    w.seed_naive()
    w.walk(20000, 99)
    start = w.rows(0)
    a0 = orc.additions(m, n, p, start)
    c = orc.walker(m, n, p, ring, 32, walker_id=5)
    c.seed_rows(start)
    assert c.best_adds == a0
    for _ in range(10):
        c.walk(1500, 7, CM)
        assert c.r == start.shape[0]                         # no reduction, no expand
        cur, best = c.rows(0), c.rows(1)
        T = scheme_tensor(m, n, p, cur) - matmul_tensor(m, n, p)
        assert not np.any(T % 2 if ring else T)
        assert orc.verify(m, n, p, ring, best)[0] == 0
        assert c.best_adds == orc.additions(m, n, p, best) <= a0
        assert not np.any([np.all(cur[l] == 0) for l in range(len(cur))])
    cnt = c.cnt
    assert cnt[4] == cnt[5] == cnt[6] == cnt[7] == cnt[10] == 0    # expands, merges, reduce calls
    assert cnt[11] == 0
    if ring == 0:
        assert c.best_adds < a0                              # flips do sparsify this scheme
