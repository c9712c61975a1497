"""The C ABI library (libfg.so) without a GPU: it loads, exports every symbol that
include/fg.h declares, and its host-only functions behave (checked against the
oracle and the paper fixtures)."""
import os
import re

import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fg():
    from paper_2511_20317_b200.build import build_libfg
    build_libfg()
    from paper_2511_20317_b200 import fg as mod
    return mod


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "fg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fg_[a-z_]+)\s*\(", txt)))


def test_every_header_symbol_is_exported(fg):
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(fg._lib, name), name
    assert set(names) == set(fg.EXPORTED)


def test_strerror_and_defaults(fg):
    for s in range(-7, 1):
        assert fg.fg_strerror(s)
    p = fg.params_default()
    assert (p.k_flip, p.thr_accept_eq, p.thr_reduce, p.thr_expand, p.expand_slack) == \
        (16, 42949672, 2147483648, 42949672, 2)


def test_host_verify_matches_oracle(fg, orc):
    rng = np.random.default_rng(5)
    for name in ["scheme_2x2x3_r11.txt", "sec36_before.txt", "sec36_after.txt"]:
        m, n, p, c = load_scheme(name)
        assert fg.fg_verify(m, n, p, 0, c) == (0, (-1, -1, -1))
        for _ in range(200):
            c2 = c.copy()
            c2[rng.integers(c.shape[0]), rng.integers(c.shape[1])] = rng.integers(-1, 2)
            rc, ff = fg.fg_verify(m, n, p, 0, c2)
            orc_rc, orc_ff = orc.verify(m, n, p, 0, c2)
            assert (rc == 0) == (orc_rc == 0) and ff == orc_ff
    for fmt in [(1, 1, 1), (2, 3, 4), (4, 4, 4), (3, 5, 4)]:
        c = orc.naive(*fmt)
        assert fg.fg_verify(*fmt, 0, c)[0] == 0
        assert fg.fg_verify(*fmt, 1, c)[0] == 0
        c[0, 0] = 2
        assert fg.fg_verify(*fmt, 0, c)[0] == -3
    assert fg.fg_verify(9, 9, 9, 0, np.zeros((1, 243), np.int8))[0] == -2


def test_create_without_gpu_fails_cleanly(fg):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(fg.FgError) as e:
        fg.FlipGraph(3, 3, 3, 0, 32, 16)
    assert e.value.status == -5
    with pytest.raises(fg.FgError) as e:
        fg.FlipGraph(9, 9, 9, 0, 32, 16)
    assert e.value.status == -2


def test_records_pack_merge_unpack(fg, orc):
    m, n, p, strassen = load_scheme("sec36_after.txt")
    naive = orc.naive(2, 2, 2)
    R = 32
    recs = [fg.fg_record_pack(m, n, p, 0, R, naive, 5),
            fg.fg_record_pack(m, n, p, 0, R, strassen, 9),
            fg.fg_record_pack(m, n, p, 0, R, strassen, 3)]
    assert all(len(r) == fg.fg_record_bytes(R) for r in recs)
    out = fg.fg_record_merge(np.concatenate(recs), 3)
    u = fg.fg_record_unpack(out, R)
    assert (u["rank"], u["additions"], u["walker_id"]) == (7, 18, 3)   # R20 tie -> lower id
    assert np.array_equal(u["coeffs"], strassen)
    u0 = fg.fg_record_unpack(recs[0], R)
    assert (u0["rank"], u0["additions"]) == (8, orc.additions(2, 2, 2, naive))


def test_explorer_registers_seed_additions(fg, orc):
    """the exploratory registry starts from each seed's true naive
    additions, so an equal-rank walk result with fewer additions can
    replace it."""
    from paper_2511_20317_b200.explore import Explorer
    m, n, p, c = load_scheme("scheme_2x2x3_r11.txt")
    pop = [((2, 2, 2), orc.naive(2, 2, 2)), ((m, n, p), c)]
    ex = Explorer(pop)
    assert ex.registry.best[(2, 2, 2)][1] == orc.additions(2, 2, 2, orc.naive(2, 2, 2)) == 4
    assert ex.registry.best[(m, n, p)][1] == orc.additions(m, n, p, c)
    r, adds, _ = ex.registry.best[(2, 2, 2)]
    ex.registry.offer((2, 2, 2), r, adds - 1, orc.naive(2, 2, 2))
    assert ex.registry.best[(2, 2, 2)][1] == adds - 1
