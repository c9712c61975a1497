"""Seeded random configurations (format, ring, row cap, Alg. 1 parameters, walker
count, step count) through the default R <= 32 kernel and the one-walker-per-warp
kernel, every walker bit-exact against the oracle.  The configurations come from a
fixed numpy seed, so a failure is reproducible by its index."""
import os

import numpy as np
import pytest

from oracle import Oracle, OracleParams

pytestmark = pytest.mark.gpu


def _configs(n=14, seed=20251120):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        m, nn, p = (int(x) for x in rng.integers(1, 4, size=3))
        ring = int(rng.integers(0, 2))
        naive = m * nn * p
        if naive + 1 > 32:
            continue
        R = int(min(32, naive + rng.integers(1, 9)))
        prm = dict(k_flip=int(rng.integers(1, 17)), thr_accept_eq=int(rng.integers(0, 1 << 31)),
                   thr_reduce=int(rng.integers(0, 1 << 32)), thr_expand=int(rng.integers(0, 1 << 30)),
                   expand_slack=int(rng.integers(0, 4)))
        W = int(rng.integers(9, 120))
        steps = int(rng.integers(300, 2500))
        out.append(((m, nn, p), ring, R, prm, W, steps, int(rng.integers(1, 1 << 62))))
    return out


def _extreme_configs(n=8, seed=7):
    """Extreme Alg. 1 parameters: thresholds at 0 / 2^32-1, negative expand slack
    (PAPER:319 gate never open), K = 1 and 16."""
    rng = np.random.default_rng(seed)
    out = []
    fmts = [(2, 2, 2), (3, 3, 3), (2, 3, 4), (1, 2, 2)]
    edges = [0, 1, 1 << 31, (1 << 32) - 1]
    for k in range(n):
        m, nn, p = fmts[k % len(fmts)]
        ring = k & 1
        naive = m * nn * p
        R = min(32, naive + 1 + k % 5)
        prm = dict(k_flip=[1, 16][k % 2], thr_accept_eq=int(rng.choice(edges)), thr_reduce=int(rng.choice(edges)),
                   thr_expand=int(rng.choice(edges)), expand_slack=int(rng.integers(-3, 6)))
        out.append(((m, nn, p), ring, R, prm, int(rng.integers(9, 70)), int(rng.integers(300, 1500)),
                    int(rng.integers(1, 1 << 62))))
    return out


CONFIGS = _configs() + _extreme_configs()


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


@pytest.mark.parametrize("kernel", ["q4", "w32"])
@pytest.mark.parametrize("idx", range(len(CONFIGS)))
def test_fuzz_config(fg, orc, kernel, idx):
    import torch
    (m, n, p), ring, R, prm, W, steps, seed = CONFIGS[idx]
    old = os.environ.get("FG_WALK_KERNEL")
    os.environ["FG_WALK_KERNEL"] = kernel
    try:
        g = fg.FlipGraph(m, n, p, ring, R, W, 0, 0, torch.cuda.current_stream().cuda_stream)
    finally:
        if old is None:
            del os.environ["FG_WALK_KERNEL"]
        else:
            os.environ["FG_WALK_KERNEL"] = old
    g.seed_naive()
    fp = fg.params_default(**prm)
    g.walk(steps, seed, fp)
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed, params=OracleParams.default(**prm))
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        assert np.array_equal(got[k], ref[k]), f"config {idx} {CONFIGS[idx]}: {k} differs"
    assert g.stats()["verify_fail"] == 0


def _ql_configs(n=8, seed=33):
    """Formats and row caps for the linked-class quad kernel (33 <= R <= 128, one-word factors)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        m, nn, p = (int(x) for x in rng.integers(2, 5, size=3))
        ring = int(rng.integers(0, 2))
        naive = m * nn * p
        maxlen = max(m * nn, nn * p, p * m)
        if naive + 2 > 128 or (ring == 0 and maxlen > 16):
            continue
        R = int(min(128, max(33, naive + int(rng.integers(2, 12)))))
        prm = dict(k_flip=int(rng.integers(1, 17)), thr_accept_eq=int(rng.integers(0, 1 << 31)),
                   thr_reduce=int(rng.integers(0, 1 << 32)), thr_expand=int(rng.integers(0, 1 << 30)),
                   expand_slack=int(rng.integers(0, 4)))
        out.append(((m, nn, p), ring, R, prm, int(rng.integers(9, 40)), int(rng.integers(300, 1200)),
                    int(rng.integers(1, 1 << 62))))
    return out


QL_CONFIGS = _ql_configs()


@pytest.mark.parametrize("idx", range(len(QL_CONFIGS)))
def test_fuzz_ql(fg, orc, idx):
    import torch
    (m, n, p), ring, R, prm, W, steps, seed = QL_CONFIGS[idx]
    old = os.environ.get("FG_WALK_KERNEL")
    os.environ["FG_WALK_KERNEL"] = "ql"
    try:
        g = fg.FlipGraph(m, n, p, ring, R, W, 0, 0, torch.cuda.current_stream().cuda_stream)
    finally:
        if old is None:
            del os.environ["FG_WALK_KERNEL"]
        else:
            os.environ["FG_WALK_KERNEL"] = old
    assert g.kernel_name.startswith("walk_ql"), g.kernel_name
    g.seed_naive()
    g.walk(steps, seed, fg.params_default(**prm))
    got = g.get_walkers()
    ref = orc.run_walkers(m, n, p, ring, R, W, 0, steps, seed, params=OracleParams.default(**prm))
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        assert np.array_equal(got[k], ref[k]), f"ql config {idx} {QL_CONFIGS[idx]}: {k} differs"


def _wide_configs(n=10, seed=4242):
    """Formats with two-word factors (Z_T > 16 or Z_2 > 32 elements) or R > 128: the
    walk_wl (default) / walk_wm layouts.  Some walker counts exceed the resident warps,
    so the persistent walker queue hands several walkers to one warp."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        m, nn, p = (int(x) for x in rng.integers(2, 8, size=3))
        ring = int(rng.integers(0, 2))
        naive = m * nn * p
        maxlen = max(m * nn, nn * p, p * m)
        if maxlen > 64 or naive + 4 > 512 or naive > 260:
            continue
        wide = maxlen > (16 if ring == 0 else 32) or naive + 8 > 128
        if not wide:
            continue
        R = int(min(512, naive + int(rng.integers(4, 40))))
        prm = dict(k_flip=int(rng.integers(1, 17)), thr_accept_eq=int(rng.integers(0, 1 << 31)),
                   thr_reduce=int(rng.integers(0, 1 << 32)), thr_expand=int(rng.integers(0, 1 << 29)),
                   expand_slack=int(rng.integers(-1, 4)))
        W = int(rng.choice([37, 160, 2600]))
        steps = int(rng.integers(150, 500))
        out.append(((m, nn, p), ring, R, prm, W, steps, int(rng.integers(1, 1 << 62))))
    return out


WIDE_CONFIGS = _wide_configs()


@pytest.mark.parametrize("kernel", ["wl", "wm"])
@pytest.mark.parametrize("idx", range(len(WIDE_CONFIGS)))
def test_fuzz_wide(fg, orc, kernel, idx):
    import torch
    from paper_2511_20317_b200.inputs import sample_walkers
    (m, n, p), ring, R, prm, W, steps, seed = WIDE_CONFIGS[idx]
    old = os.environ.get("FG_WALK_KERNEL")
    os.environ["FG_WALK_KERNEL"] = kernel
    try:
        g = fg.FlipGraph(m, n, p, ring, R, W, 0, 0, torch.cuda.current_stream().cuda_stream)
    finally:
        if old is None:
            del os.environ["FG_WALK_KERNEL"]
        else:
            os.environ["FG_WALK_KERNEL"] = old
    assert g.kernel_name.startswith("walk_" + kernel), g.kernel_name
    g.seed_naive()
    half = steps // 2
    g.walk(half, seed, fg.params_default(**prm))
    g.walk(steps - half, seed, fg.params_default(**prm))
    got = g.get_walkers()
    ids = sample_walkers(W, 10, seed=idx)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, seed, params=OracleParams.default(**prm), ids=ids)
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        assert np.array_equal(got[k][ids], ref[k]), f"wide config {idx} {WIDE_CONFIGS[idx]}: {k} differs"
    assert g.stats()["verify_fail"] == 0
