"""Z_2 -> Z_T lifting (reading R32): libfg's pruned depth-first search
against the oracle's exhaustive enumeration of sign patterns."""
import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle


@pytest.fixture(scope="module")
def fg():
    from paper_2511_20317_b200.build import build_libfg
    build_libfg()
    from paper_2511_20317_b200 import fg as mod
    return mod


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def test_naive_lifts_to_itself(fg, orc):
    c = orc.naive(2, 2, 3)
    rc, out, _ = fg.fg_lift(2, 2, 3, c)
    assert rc == 0 and np.array_equal(out, c)


def test_strassen_mod2_lifts(fg, orc):
    """The printed rank-7 scheme with its signs erased (a Z_2 scheme) lifts back to a
    Z_T scheme with the same support."""
    _, _, _, s = load_scheme("sec36_after.txt")
    z = np.abs(s)
    assert orc.verify(2, 2, 2, 1, z)[0] == 0
    rc, out, nodes = fg.fg_lift(2, 2, 2, z)
    assert rc == 0 and orc.verify(2, 2, 2, 0, out)[0] == 0
    assert np.array_equal(np.abs(out), z)
    assert orc.lift_exhaustive(2, 2, 2, z)[0] == 1


def _free_signs(fmt, z):
    m, n, p = fmt
    return int(z.sum()) - 2 * len(z)          # nonzeros minus the pinned u and v signs


def test_lift_agrees_with_exhaustive_oracle(fg, orc):
    seen = {0: 0, 1: 0}
    # Z_2 walk outputs of small formats, plus one rank-6 (1,2,3) scheme (walker 573,
    # 4211 steps, key 3, its best) that has NO Z_T lift: 26 free signs, ~15 s of
    # exhaustive enumeration in the oracle
    cases = [(f, wid, 500 + wid * 13, 5, 22) for f in [(2, 2, 2), (1, 2, 3), (2, 1, 3), (3, 1, 2)]
             for wid in range(25)]
    cases += [((1, 2, 3), 573, 200 + 573 * 7, 3, 26)]
    for fmt, wid, steps, key, maxfree in cases:
            w = orc.walker(*fmt, 1, 32, walker_id=wid)
            w.seed_naive()
            w.walk(steps, key)
            for which in (0, 1):
                z = w.rows(which)
                if _free_signs(fmt, z) > maxfree:
                    continue
                ex, exout = orc.lift_exhaustive(*fmt, z)
                if ex < 0:
                    continue
                rc, out, _ = fg.fg_lift(*fmt, z, 5_000_000)
                assert (rc == 0) == (ex == 1), (fmt, wid, which)
                if rc == 0:
                    assert orc.verify(*fmt, 0, out)[0] == 0 and np.array_equal(np.abs(out), z)
                else:
                    assert rc == -4
                seen[ex] += 1
    assert seen[1] > 50 and seen[0] >= 1             # both outcomes exercised


def test_budget_and_domain(fg, orc):
    w = orc.walker(3, 3, 3, 1, 32, walker_id=3)
    w.seed_naive()
    w.walk(20000, 5)
    rc, _, nodes = fg.fg_lift(3, 3, 3, w.rows(), node_budget=10)
    assert rc in (0, -6, -4) and nodes <= 11
    bad = orc.naive(2, 2, 2)
    bad[0, 0] = -1
    assert fg.fg_lift(2, 2, 2, bad)[0] == -3


def test_parity_system_decides_dense_cases(fg, orc):
    """The GF(2) parity constraints (R32): on dense (3,3,3) Z_2 walk outputs the search
    ends quickly either way -- a lift that the oracle's Brent check accepts with the same
    support, or a proof that none exists -- where round 1's plain search ran out of its
    budget."""
    outcomes = set()
    for wid in range(6):
        w = orc.walker(3, 3, 3, 1, 32, walker_id=wid)
        w.seed_naive()
        w.walk(30000, 11)
        z = w.rows(1)
        rc, out, nodes = fg.fg_lift(3, 3, 3, z, 1_000_000)
        assert rc in (0, -4) and nodes < 1_000_000
        if rc == 0:
            assert orc.verify(3, 3, 3, 0, out)[0] == 0 and np.array_equal(np.abs(out), z)
        outcomes.add(rc)
    assert outcomes == {0, -4}
