"""Every R <= 32 walk kernel against the CPU oracle (FG_WALK_KERNEL selects it at
fg_create): one walker per warp (w32) and one per quad (q4, the default).  Same bar as test_gpu_parity.py: bit-exact final and
best schemes, ranks, counters and the per-step event digest.

Walker counts that are not multiples of 8 / 32 exercise the tail quads and warps.
"""
import os

import numpy as np
import pytest

from oracle import Oracle, OracleParams
from paper_2511_20317_b200.inputs import WORKLOADS, sample_walkers

pytestmark = pytest.mark.gpu
ZT, Z2 = 0, 1
KERNELS = {"w32": "walk_w32", "q4": "walk_q4"}
KERNEL_PREFIX = dict(KERNELS, ql="walk_ql", wm="walk_wm", wl="walk_wl")


@pytest.fixture(scope="module")
def fg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20317_b200 import fg as mod
    return mod


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _ctx(fg, kernel, m, n, p, ring, R, W):
    import torch
    old = os.environ.get("FG_WALK_KERNEL")
    os.environ["FG_WALK_KERNEL"] = kernel
    try:
        g = fg.FlipGraph(m, n, p, ring, R, W, 0, 0, torch.cuda.current_stream().cuda_stream)
    finally:
        if old is None:
            del os.environ["FG_WALK_KERNEL"]
        else:
            os.environ["FG_WALK_KERNEL"] = old
    assert g.kernel_name.startswith(KERNEL_PREFIX[kernel]), g.kernel_name
    return g


def _check(got, ref, ids):
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        g = got[k][ids] if ids is not None else got[k]
        assert np.array_equal(g, ref[k]), f"{k} differs"


@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("kernel", list(KERNELS))
def test_kernel_c1_all_walkers(fg, orc, kernel, ring):
    """(2,2,2) naive -> 7, 61 walkers (a partial last quad / warp), 20000 steps."""
    W, steps, seed = 61, 20000, WORKLOADS["c1_222_zt"].seed + 7
    g = _ctx(fg, kernel, 2, 2, 2, ring, 32, W)
    g.seed_naive()
    g.walk(steps, seed)
    got = g.get_walkers()
    ref = orc.run_walkers(2, 2, 2, ring, 32, W, 0, steps, seed)
    _check(got, ref, None)
    st = g.stats()
    assert st["verify_fail"] == 0


@pytest.mark.parametrize("ring", [ZT, Z2])
@pytest.mark.parametrize("kernel", list(KERNELS))
def test_kernel_c2_sampled(fg, orc, kernel, ring):
    """(3,3,3) naive 27, 2051 walkers, 1500 steps in three launches; 32 sampled
    trajectories bit-exact."""
    W, steps, seed = 2051, 1500, WORKLOADS["c2_333_zt"].seed + 7
    g = _ctx(fg, kernel, 3, 3, 3, ring, 32, W)
    g.seed_naive()
    p = fg.params_default(phase_steps=500)
    g.walk(steps, seed, p)
    got = g.get_walkers()
    ids = sample_walkers(W, 32, seed=3 + ring)
    ref = orc.run_walkers(3, 3, 3, ring, 32, 0, 0, steps, seed, ids=ids)
    _check(got, ref, ids)
    assert g.stats()["verify_fail"] == 0


@pytest.mark.parametrize("kernel", ["w32", "q4"])
def test_kernel_small_rcap_and_edge(fg, orc, kernel):
    """R < 32 (expand hits the row cap) and a format with 1-element factors."""
    for (m, n, p, R, steps) in [((2), 2, 2, 9, 6000), (1, 2, 3, 8, 4000), (2, 3, 2, 14, 5000)]:
        W, seed = 37, 0x5EED + R
        g = _ctx(fg, kernel, m, n, p, ZT, R, W)
        g.seed_naive()
        g.walk(steps, seed)
        got = g.get_walkers()
        ref = orc.run_walkers(m, n, p, ZT, R, W, 0, steps, seed)
        _check(got, ref, None)


@pytest.mark.parametrize("kernel", ["w32", "q4"])
def test_kernel_k_flip_round_boundaries(fg, orc, kernel):
    """K (draws per try_flip, R11) below, at and across the quad kernel's 4-draw rounds,
    with a high expand rate so flip failures and expands are frequent."""
    for kf in (1, 3, 5, 7):
        W, steps, seed = 203, 800, 0xF11 + kf
        p = fg.params_default(k_flip=kf, thr_expand=1 << 29, expand_slack=3)
        g = _ctx(fg, kernel, 3, 3, 3, ZT, 32, W)
        g.seed_naive()
        g.walk(steps, seed, p)
        got = g.get_walkers()
        ids = sample_walkers(W, 12, seed=kf)
        op = OracleParams.default(k_flip=kf, thr_accept_eq=p.thr_accept_eq, thr_reduce=p.thr_reduce,
                                  thr_expand=p.thr_expand, expand_slack=p.expand_slack)
        ref = orc.run_walkers(3, 3, 3, ZT, 32, 0, 0, steps, seed, params=op, ids=ids)
        _check(got, ref, ids)


QL_CASES = [((3, 3, 4), ZT, 48, 45, 3000), ((2, 4, 5), Z2, 64, 37, 3000), ((3, 4, 4), ZT, 64, 29, 2500),
            ((4, 4, 4), ZT, 96, 61, 2000), ((4, 4, 4), Z2, 96, 40, 2000), ((4, 4, 4), ZT, 128, 17, 1500),
            ((3, 4, 5), Z2, 72, 23, 2000), ((4, 4, 6), Z2, 128, 9, 1000), ((2, 4, 4), ZT, 40, 33, 3000)]


@pytest.mark.parametrize("case", QL_CASES, ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-R{c[2]}")
def test_ql_linked_class_kernel(fg, orc, case):
    """The linked-class quad kernel (33 <= R <= 128) against the oracle, every walker."""
    (m, n, p), ring, R, W, steps = case
    seed = 0x51 + R + ring
    g = _ctx(fg, "ql", m, n, p, ring, R, W)
    g.seed_naive()
    g.walk(steps, seed, fg.params_default(phase_steps=steps // 2 + 1))
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed)
    _check(got, ref, None)
    assert g.stats()["verify_fail"] == 0


@pytest.mark.parametrize("case", [((4, 4, 4), ZT, 96, 61, 2000), ((3, 3, 3), ZT, 33, 45, 3000), ((3, 4, 4), ZT, 64, 29, 2500),
                                  ((4, 4, 4), Z2, 96, 40, 2000), ((3, 3, 3), Z2, 64, 45, 2500)],
                         ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-R{c[2]}")
def test_wm_forced_for_one_word(fg, orc, case):
    """One-word formats with 33 <= R <= 128 default to walk_ql; the multi-row kernel
    stays covered for them through FG_WALK_KERNEL=wm."""
    (m, n, p), ring, R, W, steps = case
    seed = 0x3A + R
    g = _ctx(fg, "wm", m, n, p, ring, R, W)
    g.seed_naive()
    g.walk(steps, seed)
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed)
    _check(got, ref, None)


def test_ql_chunked_tasks(fg, orc):
    """walk_ql's persistent (walker group, step chunk) tasks: forcing 3 chunks per group
    (FG_QL_CHUNKS) leaves every trajectory unchanged -- the chunks hand the state over
    through HBM in order."""
    (m, n, p), ring, R, W, steps = (4, 4, 4), ZT, 96, 83, 1500
    old = os.environ.get("FG_QL_CHUNKS")
    os.environ["FG_QL_CHUNKS"] = "3"
    try:
        g = _ctx(fg, "ql", m, n, p, ring, R, W)
        g.seed_naive()
        g.walk(steps, 0xC4C4)
    finally:
        if old is None:
            del os.environ["FG_QL_CHUNKS"]
        else:
            os.environ["FG_QL_CHUNKS"] = old
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, 0xC4C4)
    _check(got, ref, None)
    assert np.all(got["step"] == steps)


@pytest.mark.parametrize("case", [((4, 4, 4), ZT, 96, 61, 2000), ((3, 3, 3), ZT, 33, 45, 3000), ((3, 4, 4), ZT, 64, 29, 2500),
                                  ((4, 4, 4), Z2, 96, 40, 2000), ((3, 3, 3), Z2, 64, 45, 2500)],
                         ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-R{c[2]}")
def test_wl_forced_for_one_word(fg, orc, case):
    """The linked-class one-walker-per-warp kernel (default for wide factors and R > 128)
    on one-word formats through FG_WALK_KERNEL=wl, every walker, across two launches
    (the second resumes from the class image)."""
    (m, n, p), ring, R, W, steps = case
    seed = 0x3B + R
    g = _ctx(fg, "wl", m, n, p, ring, R, W)
    g.seed_naive()
    g.walk(steps, seed, fg.params_default(phase_steps=steps // 3 + 1))
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed)
    _check(got, ref, None)


@pytest.mark.parametrize("case", [((5, 5, 5), ZT, 160, 96, 600), ((4, 5, 12), ZT, 256, 40, 300),
                                  ((4, 5, 12), Z2, 256, 40, 300), ((4, 4, 4), Z2, 160, 64, 800)],
                         ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-R{c[2]}")
def test_wm_forced_for_wide(fg, orc, case):
    """The round-1 multi-row kernel stays covered on the C4 / C5 layouts (P32, P64, PZ64,
    PZ2 with R > 128) through FG_WALK_KERNEL=wm."""
    (m, n, p), ring, R, W, steps = case
    seed = 0x3C + R
    g = _ctx(fg, "wm", m, n, p, ring, R, W)
    g.seed_naive()
    g.walk(steps, seed)
    got = g.get_walkers()
    ids = sample_walkers(W, 8, seed=R)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, seed, ids=ids)
    _check(got, ref, ids)


@pytest.mark.parametrize("case", [((2, 2, 16), ZT, 96, 70, 2500), ((2, 3, 20), ZT, 160, 50, 1500),
                                  ((1, 1, 40), ZT, 64, 64, 2000), ((1, 2, 30), Z2, 96, 64, 2000),
                                  ((1, 1, 40), Z2, 80, 64, 2000)],
                         ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-R{c[2]}")
def test_wl_large_classes(fg, orc, case):
    """Flip classes longer than one ballot round of walk_wl's sorted arrays (16 entries
    each way) and longer than a warp (32): naive (2,2,16) has U classes of 16 rows,
    (2,3,20) of 20, (1,1,40) one U class of all 40 rows.  Every walker, two launches
    (the second resumes from the class image), with the structure self-check on."""
    (m, n, p), ring, R, W, steps = case
    seed = 0x3D + R
    os.environ["FG_DBG"] = "1"
    try:
        g = _ctx(fg, "wl", m, n, p, ring, R, W)
        g.seed_naive()
        g.walk(steps, seed, fg.params_default(phase_steps=steps // 2 + 1))
    finally:
        del os.environ["FG_DBG"]
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed)
    _check(got, ref, None)


@pytest.mark.parametrize("case", [((3, 3, 3), ZT, 32, 203, 2600, "5"), ((3, 3, 3), Z2, 32, 517, 1800, "7"),
                                  ((2, 2, 2), ZT, 12, 64, 3000, "4"), ((3, 3, 3), ZT, 32, 1000, 900, "64")],
                         ids=lambda c: f"{c[0]}-{'zt' if c[1] == ZT else 'z2'}-W{c[3]}-C{c[5]}")
def test_q4_chunked_tasks(fg, orc, case):
    """walk_q4's completion-ordered (walker group, step chunk) tasks (FG_Q4_CHUNKS forces
    the chunk count; the C2 bench configuration chunks by default): every trajectory is
    unchanged, across two launches, with ragged chunk lengths and a count above the
    steps of a launch (64 chunks of a 450-step launch)."""
    (m, n, p), ring, R, W, steps, chunks = case
    seed = 0xC5C5 + W
    old = os.environ.get("FG_Q4_CHUNKS")
    os.environ["FG_Q4_CHUNKS"] = chunks
    try:
        g = _ctx(fg, "q4", m, n, p, ring, R, W)
        g.seed_naive()
        g.walk(steps, seed, fg.params_default(phase_steps=steps // 2))
    finally:
        if old is None:
            del os.environ["FG_Q4_CHUNKS"]
        else:
            os.environ["FG_Q4_CHUNKS"] = old
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed)
    _check(got, ref, None)
    assert np.all(got["step"] == steps)
    assert g.stats()["verify_fail"] == 0


def test_q4_chunked_complexity_mode(fg, orc):
    """R24 (naive-complexity mode) through walk_q4's chunked tasks (FG_Q4_CHUNKS=6):
    every walker bit-exact, the best-by-additions image handed over between chunks."""
    m, n, p, R, W, steps, seed = 3, 3, 3, 32, 203, 1800, 0xCAFE
    w = orc.walker(m, n, p, ZT, R, walker_id=3)
    w.seed_naive()
    w.walk(5000, 77)
    start = w.rows(0)
    old = os.environ.get("FG_Q4_CHUNKS")
    os.environ["FG_Q4_CHUNKS"] = "6"
    try:
        g = _ctx(fg, "q4", m, n, p, ZT, R, W)
        g.seed_pool(start)
        g.walk(steps, seed, fg.params_default(flags=fg.FG_FLAG_COMPLEXITY))
    finally:
        if old is None:
            del os.environ["FG_Q4_CHUNKS"]
        else:
            os.environ["FG_Q4_CHUNKS"] = old
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ZT, R, W, 0, steps, seed, seed_coeffs=start,
                          params=OracleParams.default(mode=1))
    _check(got, ref, None)
    assert np.all(got["r"] == start.shape[0])


@pytest.mark.parametrize("kernel,fmt,R,W", [("q4", (2, 2, 8), 32, 203), ("w32", (2, 2, 8), 32, 203),
                                            ("ql", (2, 2, 8), 48, 203), ("wl", (3, 4, 12), 160, 48),
                                            ("wm", (3, 4, 12), 160, 48)],
                         ids=lambda v: str(v) if not isinstance(v, tuple) else ",".join(map(str, v)))
def test_large_flip_budget(fg, orc, kernel, fmt, R, W):
    """K = 64 flip draws per step (R11, draws beyond 16 from Philox slots 23..70): formats
    with wide V/W factors, where all 16 draws of a step overflow {-1,0,1} a few % of the time
    (witness: the K = 16 oracle run on the same walkers has failed flips), every kernel
    family bit-exact with the oracle."""
    m, n, p = fmt
    steps, seed = 3000, 0x5EED64
    ids = sample_walkers(W, 8, seed=11)
    ref16 = orc.run_walkers(m, n, p, ZT, R, 0, 0, steps, seed, params=OracleParams.default(k_flip=16), ids=ids)
    assert ref16["cnt"][:, 3].sum() > 0
    g = _ctx(fg, kernel, m, n, p, ZT, R, W)
    g.seed_naive()
    g.walk(steps, seed, fg.params_default(k_flip=64, phase_steps=1000))
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ZT, R, 0, 0, steps, seed, params=OracleParams.default(k_flip=64), ids=ids)
    _check(got, ref, ids)
    assert g.stats()["verify_fail"] == 0
    with pytest.raises(fg.FgError):
        g.walk(10, seed, fg.params_default(k_flip=65))
    g.close()
