"""GPU (libfg.so, sm_100a) against the CPU oracle, through the C ABI.

The bar: every walker trajectory is bit-exact -- final
scheme, best scheme, ranks, step index, 12 counters and the 64-bit event digest
that folds (rank, best, flags, touched rows, draws) of EVERY step.
"""
import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle, OracleParams
from paper_2511_20317_b200.inputs import WORKLOADS, perturbations, sample_walkers

pytestmark = pytest.mark.gpu
ZT, Z2 = 0, 1


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


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _ctx(fg, m, n, p, ring, R, W, base=0):
    return fg.FlipGraph(m, n, p, ring, R, W, base, 0, _stream())


def _oparams(fp):
    return OracleParams.default(k_flip=fp.k_flip, thr_accept_eq=fp.thr_accept_eq,
                                thr_reduce=fp.thr_reduce, thr_expand=fp.thr_expand,
                                expand_slack=fp.expand_slack)


def _assert_same(got, ref, idx=None, what=""):
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        g = got[k] if idx is None else got[k][idx]
        if not np.array_equal(g, ref[k]):
            bad = np.nonzero(np.any((g != ref[k]).reshape(len(g), -1), axis=1))[0]
            raise AssertionError(f"{what}: {k} differs for walkers {bad[:10]} "
                                 f"(gpu {g[bad[0]] if k in ('r','best_r','digest') else ''} "
                                 f"oracle {ref[k][bad[0]] if k in ('r','best_r','digest') else ''})")


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_c1_all_64_walkers_to_strassen(fg, orc, ring):
    """Config C1: (2,2,2) naive -> 7, all 64 trajectories bit-exact."""
    wl = WORKLOADS["c1_222_zt"]
    steps = 60000
    g = _ctx(fg, 2, 2, 2, ring, wl.r_cap, 64)
    g.seed_naive()
    g.walk(steps, wl.seed + ring)
    got = g.get_walkers()
    ref = orc.run_walkers(2, 2, 2, ring, wl.r_cap, 64, 0, steps, wl.seed + ring)
    _assert_same(got, ref, what="c1")
    assert np.all(got["best_r"] == 7)
    assert np.all(got["step"] == steps)
    st = g.stats()
    assert st["verify_fail"] == 0 and st["queue_overflow"] == 0
    assert st["verified"] == int(got["cnt"][:, 9].sum())
    b = g.best()
    assert b["rank"] == 7 and fg.fg_verify(2, 2, 2, ring, b["coeffs"])[0] == 0


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_c2_sampled_walkers(fg, orc, ring):
    """Config C2: (3,3,3) with 16384 walkers at full size; 96 sampled trajectories
    bit-exact against the oracle; every walker's scheme verifies on the device."""
    wl = WORKLOADS["c2_333_zt"]
    steps = 3000
    W = wl.walkers
    g = _ctx(fg, 3, 3, 3, ring, wl.r_cap, W)
    g.seed_naive()
    g.walk(steps, wl.seed + ring)
    got = g.get_walkers()
    ids = sample_walkers(W, 96, seed=ring)
    ref = orc.run_walkers(3, 3, 3, ring, wl.r_cap, 0, 0, steps, wl.seed + ring, ids=ids)
    _assert_same(got, ref, idx=ids, what="c2")
    st = g.stats()
    assert st["verify_fail"] == 0 and st["queue_overflow"] == 0
    # property at full size: every current scheme satisfies the Brent equations
    cur = [got["rows"][k][: got["r"][k]] for k in range(0, W, 7)]
    ok, _ = g.verify_batch(cur)
    assert np.all(ok == 1)
    assert np.all(got["r"] <= wl.r_cap) and np.all(got["best_r"] <= 27)


def test_phase_split_and_params(fg, orc):
    """Counter-based RNG: one call of 2400 steps == calls of 1000+900+500 with
    phase_steps 333 inside; non-default parameters are honoured identically."""
    p = fg.params_default(k_flip=4, thr_reduce=1 << 30, thr_expand=1 << 28, expand_slack=1)
    a = _ctx(fg, 3, 3, 3, ZT, 32, 256, base=1000)
    b = _ctx(fg, 3, 3, 3, ZT, 32, 256, base=1000)
    a.seed_naive()
    b.seed_naive()
    a.walk(2400, 77, p)
    p.phase_steps = 333
    for s in (1000, 900, 500):
        b.walk(s, 77, p)
    ga, gb = a.get_walkers(), b.get_walkers()
    _assert_same(ga, gb, what="split")
    ids = sample_walkers(256, 24, seed=3)
    ref = orc.run_walkers(3, 3, 3, ZT, 32, 0, 0, 2400, 77, params=_oparams(p), ids=ids + 1000)
    _assert_same(ga, ref, idx=ids, what="params")


def test_edge_formats(fg, orc):
    """Degenerate and ragged cases: (1,1,1:1) (no flip, no expand), capacity
    R = naive rank (every expand rejected), non-square (2,3,4), Strassen seed
    (no candidates: expand fallback), R below 32 and a ragged walker count."""
    cases = [((1, 1, 1), ZT, 4, 37, None), ((2, 2, 2), ZT, 8, 33, None),
             ((2, 3, 4), ZT, 32, 70, None), ((2, 3, 4), Z2, 32, 70, None),
             ((2, 2, 2), ZT, 12, 40, "sec36_after.txt"), ((3, 2, 3), ZT, 30, 65, None),
             ((2, 4, 2), ZT, 32, 31, None)]
    for (m, n, p), ring, R, W, seedfile in cases:
        g = _ctx(fg, m, n, p, ring, R, W, base=5)
        seedc = None
        if seedfile:
            _, _, _, seedc = load_scheme(seedfile)
            g.seed_pool(seedc)
        else:
            g.seed_naive()
        g.walk(1500, 4242)
        got = g.get_walkers()
        ref = orc.run_walkers(m, n, p, ring, R, W, 5, 1500, 4242, seed_coeffs=seedc)
        _assert_same(got, ref, what=f"{(m, n, p)} ring {ring} R {R}")


def test_zero_steps_and_best(fg, orc):
    g = _ctx(fg, 3, 3, 3, ZT, 32, 50)
    g.seed_naive()
    g.walk(0, 1)
    b = g.best()
    assert b["rank"] == 27 and b["walker_id"] == 0
    assert b["additions"] == orc.additions(3, 3, 3, orc.naive(3, 3, 3))


def test_verify_batch_matches_oracle(fg, orc):
    rng = np.random.default_rng(11)
    g = _ctx(fg, 3, 3, 3, ZT, 32, 64)
    g.seed_naive()
    g.walk(4000, 9)
    got = g.get_walkers()
    schemes = [got["best"][k][: got["best_r"][k]] for k in range(64)]
    for (l, e, v) in perturbations(20, 27, ZT, 60, seed=1):
        k = int(rng.integers(64))
        c = schemes[k].copy()
        c[l % len(c), e] = v
        schemes.append(c)
    ok, ff = g.verify_batch(schemes)
    for k, c in enumerate(schemes):
        rc, off = orc.verify(3, 3, 3, ZT, c)
        assert ok[k] == (1 if rc == 0 else 0)
        assert tuple(ff[k]) == off
    # Z2
    g2 = _ctx(fg, 2, 3, 4, Z2, 32, 4)
    base = orc.naive(2, 3, 4)
    sch = [base]
    for (l, e, v) in perturbations(24, base.shape[1], Z2, 30, seed=2):
        c = base.copy()
        c[l, e] = v
        sch.append(c)
    ok, ff = g2.verify_batch(sch)
    for k, c in enumerate(sch):
        rc, off = orc.verify(2, 3, 4, Z2, c)
        assert ok[k] == (1 if rc == 0 else 0) and tuple(ff[k]) == off


def test_state_roundtrip_resumes_exactly(fg):
    a = _ctx(fg, 3, 3, 3, ZT, 32, 128)
    a.seed_naive()
    a.walk(700, 5)
    img = a.save_state()
    a.walk(800, 5)
    b = _ctx(fg, 3, 3, 3, ZT, 32, 128)
    b.load_state(img)
    b.walk(800, 5)
    _assert_same(a.get_walkers(), b.get_walkers(), what="resume")


def test_restart_matches_oracle(fg, orc):
    """R23: walkers whose best is worse than pool best + slack are re-seeded."""
    m, n, p, strassen = load_scheme("sec36_after.txt")
    g = _ctx(fg, 2, 2, 2, ZT, 32, 40)
    g.seed_naive()
    g.walk(200, 3)
    rec = fg.fg_record_pack(2, 2, 2, ZT, 32, strassen, 999)
    g.import_best(rec, 1)
    pool = g.best()                      # the scheme restart will use (R20 minimum)
    before = g.get_walkers()
    n = g.restart(0)
    assert n == int(np.sum(before["best_r"] > pool["rank"]))
    g.walk(300, 3)
    got = g.get_walkers()
    for k in range(40):
        w = orc.walker(2, 2, 2, ZT, 32, walker_id=k)
        w.seed_naive()
        w.walk(200, 3)
        if w.best_r > pool["rank"]:
            w.restart(pool["coeffs"])
        w.walk(300, 3)
        assert w.digest == got["digest"][k] and w.r == got["r"][k]
        assert np.array_equal(w.rows(), got["rows"][k][: w.r])


# ---------------- the multi-row kernels (33 <= R <= 512): configs C3-C5 ----------------
MULTI_CASES = [
    # (format, ring, R, walkers, sampled, steps)
    ((4, 4, 4), ZT, 96, 512, 24, 2500),      # C3 Z_T, layout P16, NS 3
    ((4, 4, 4), Z2, 96, 512, 24, 2500),      # C3 Z_2, layout PZ2
    ((5, 5, 5), ZT, 160, 256, 12, 1200),     # C4, layout P32, NS 5
    ((3, 3, 3), ZT, 33, 300, 24, 3000),      # ragged R (NS 2), ranks cross 32
    ((3, 3, 3), Z2, 64, 300, 24, 3000),
    ((4, 4, 4), ZT, 64, 200, 16, 2000),      # R = naive rank: every expand rejected
    ((4, 5, 12), ZT, 256, 64, 6, 400),       # C5 formats, layout P64
    ((6, 7, 9), ZT, 416, 48, 4, 250),
    ((4, 5, 12), Z2, 256, 64, 6, 400),       # layout PZ64
]


@pytest.mark.parametrize("case", MULTI_CASES, ids=lambda c: f"{c[0]}-{'ZT' if c[1] == 0 else 'Z2'}-R{c[2]}")
def test_multi_row_kernel_parity(fg, orc, case):
    (m, n, p), ring, R, W, k, steps = case
    g = _ctx(fg, m, n, p, ring, R, W, base=77)
    # one-word factors with R <= 128 run on the linked-class quad kernel (walk_ql)
    maxlen = max(m * n, n * p, p * m)
    assert g.kernel_name.startswith("walk_ql" if R <= 128 and maxlen <= (16 if ring == ZT else 32) else "walk_wl")
    g.seed_naive()
    seed = 0x2511203170000000 + 2 + ring
    half = steps // 2
    g.walk(half, seed)
    g.walk(steps - half, seed)                 # phase split inside the comparison
    got = g.get_walkers()
    ids = sample_walkers(W, k, seed=R + ring)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, seed, ids=ids + 77)
    _assert_same(got, ref, idx=ids, what=f"multi {(m, n, p)} ring {ring} R {R}")
    st = g.stats()
    assert st["verify_fail"] == 0 and st["queue_overflow"] == 0
    cur = [got["rows"][w][: got["r"][w]] for w in range(0, W, max(1, W // 16))]
    ok, _ = g.verify_batch(cur)
    assert np.all(ok == 1)


def test_multi_row_seeded_pool_and_restart(fg, orc):
    """Strassen seed (rank 7, no flip candidates) in the multi-row kernel (R = 40),
    then an import + restart: trajectories still match the oracle."""
    _, _, _, strassen = load_scheme("sec36_after.txt")
    g = _ctx(fg, 2, 2, 2, ZT, 40, 20, base=3)
    g.seed_pool(strassen)
    g.walk(800, 11)
    got = g.get_walkers()
    ref = orc.run_walkers(2, 2, 2, ZT, 40, 20, 3, 800, 11, seed_coeffs=strassen)
    _assert_same(got, ref, what="multi seed_pool")


# ---------------- R24 naive-complexity minimisation ----------------
@pytest.mark.parametrize("case", [((3, 3, 3), ZT, 32, 256), ((3, 3, 3), Z2, 32, 128),
                                  ((4, 4, 4), ZT, 96, 64), ((2, 3, 4), ZT, 32, 96)],
                         ids=lambda c: f"{c[0]}-{'ZT' if c[1] == 0 else 'Z2'}-R{c[2]}")
def test_complexity_mode_parity(fg, orc, case):
    """Seed every walker with a walked (dense) scheme, run R24 on the GPU and in the
    oracle: trajectories bit-exact; best additions only fall; rank constant."""
    (m, n, p), ring, R, W = case
    w = orc.walker(m, n, p, ring, R, walker_id=5)
    w.seed_naive()
    w.walk(6000, 99)
    start = w.rows(0)
    a0 = orc.additions(m, n, p, start)
    g = _ctx(fg, m, n, p, ring, R, W, base=11)
    g.seed_pool(start)
    prm = fg.params_default(flags=fg.FG_FLAG_COMPLEXITY)
    g.walk(1500, 4242, prm)
    got = g.get_walkers()
    ids = sample_walkers(W, 16, seed=5)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, 1500, 4242, seed_coeffs=start,
                          params=OracleParams.default(mode=1), ids=ids + 11)
    _assert_same(got, ref, idx=ids, what=f"R24 {(m, n, p)}")
    assert np.all(got["r"] == start.shape[0])
    for k in range(W):
        b = got["best"][k][: got["best_r"][k]]
        assert got["best_adds"][k] == orc.additions(m, n, p, b) <= a0
    st = g.stats()
    # improvements are frequent in R24: those that overflow the queue are covered by
    # verifying the walker's final best
    assert st["verify_fail"] == 0 and st["verified"] > 0
    bb = g.best()
    assert bb["additions"] == int(got["best_adds"].min()) and fg.fg_verify(m, n, p, ring, bb["coeffs"])[0] == 0


@pytest.mark.parametrize("case", [((5, 5, 5), ZT, 160, 40, None), ((5, 5, 5), Z2, 144, 40, None),
                                  ((3, 4, 12), ZT, 160, 24, None), ((4, 4, 4), ZT, 96, 40, "wm")],
                         ids=lambda c: f"{c[0]}-{'ZT' if c[1] == 0 else 'Z2'}-R{c[2]}-{c[4] or 'default'}")
def test_complexity_mode_wide_and_mode_switch(fg, orc, monkeypatch, case):
    """R24 on walk_wl's formats (R > 128, wide factors; walk_ql contexts too) and on the
    forced round-1 kernel: two R24 launches (the second resumes walk_wl's class image),
    then a plain Alg. 1 walk on the same walkers -- R24 flips skip R12, so the image's
    dirty set must force a full R15 scan; every sampled walker bit-exact with the
    oracle walker run through the same three calls."""
    (m, n, p), ring, R, W, env = case
    if env:
        monkeypatch.setenv("FG_WALK_KERNEL", env)
    w = orc.walker(m, n, p, ring, R, walker_id=7)
    w.seed_naive()
    w.walk(4000, 123)
    start = w.rows(0)
    g = _ctx(fg, m, n, p, ring, R, W, base=21)
    g.seed_pool(start)
    cm = fg.params_default(flags=fg.FG_FLAG_COMPLEXITY)
    g.walk(700, 77, cm)
    g.walk(500, 78, cm)
    mid = g.get_walkers()
    g.walk(900, 79)
    got = g.get_walkers()
    a0 = orc.additions(m, n, p, start)
    for k in sample_walkers(W, 6, seed=3):
        o = orc.walker(m, n, p, ring, R, walker_id=21 + int(k))
        o.seed_rows(start)
        o.walk(700, 77, OracleParams.default(mode=1))
        o.walk(500, 78, OracleParams.default(mode=1))
        assert o.digest == mid["digest"][k] and o.best_adds == mid["best_adds"][k] <= a0
        assert mid["r"][k] == start.shape[0]
        o.walk(900, 79)
        assert o.digest == got["digest"][k] and o.r == got["r"][k] and o.best_r == got["best_r"][k]
        assert np.array_equal(o.rows(), got["rows"][k][: o.r])
        assert np.array_equal(o.rows(1), got["best"][k][: o.best_r])
    assert g.stats()["verify_fail"] == 0


def test_best_adds_tracks_best_scheme_in_walk_mode(fg, orc):
    g = _ctx(fg, 3, 3, 3, ZT, 32, 512)
    g.seed_naive()
    g.walk(5000, 21)
    got = g.get_walkers()
    for k in range(0, 512, 5):
        assert got["best_adds"][k] == orc.additions(3, 3, 3, got["best"][k][: got["best_r"][k]])


def test_load_walkers_distinct_schemes(fg, orc):
    """fg_load_walkers (one scheme per walker, used by exploratory search) continues
    each walker exactly like an oracle walker seeded with that scheme."""
    schemes = []
    for k in range(12):
        w = orc.walker(3, 3, 3, ZT, 32, walker_id=100 + k)
        w.seed_naive()
        w.walk(500 + 100 * k, 9)
        schemes.append(w.rows())
    g = _ctx(fg, 3, 3, 3, ZT, 32, 12, base=40)
    g.load_walkers(schemes)
    g.walk(1200, 31)
    got = g.get_walkers()
    for k in range(12):
        w = orc.walker(3, 3, 3, ZT, 32, walker_id=40 + k)
        w.seed_rows(schemes[k])
        w.walk(1200, 31)
        assert w.digest == got["digest"][k] and w.r == got["r"][k]
        assert np.array_equal(w.rows(), got["rows"][k][: w.r])


def test_api_errors_and_stats(fg, orc):
    """Error paths of the ABI (no partial work): walk before seed, bad params,
    unsupported capacity; stats accumulate; fg_get_walker agrees with the bulk call."""
    g = _ctx(fg, 3, 3, 3, ZT, 32, 8)
    with pytest.raises(fg.FgError) as e:
        g.walk(10, 1)
    assert e.value.status == -6                     # FG_E_STATE: not seeded
    g.seed_naive()
    with pytest.raises(fg.FgError) as e:
        g.walk(10, 1, fg.params_default(k_flip=0))
    assert e.value.status == -1
    with pytest.raises(fg.FgError) as e:
        g.walk(10, 1, fg.params_default(flags=8))
    assert e.value.status == -1
    with pytest.raises(fg.FgError) as e:
        fg.FlipGraph(3, 3, 3, ZT, 600, 4, 0, 0, _stream())
    assert e.value.status == -2
    with pytest.raises(fg.FgError) as e:
        g.seed_pool(orc.naive(3, 3, 3)[:5])        # does not verify
    assert e.value.status == -4
    g.walk(300, 2)
    g.walk(200, 2)
    st = g.stats()
    assert st["steps"] == 8 * 500 and st["walk_launches"] == 2 and st["launches"] >= 4
    got = g.get_walkers()
    assert np.all(got["cnt"][:, 0] == 500) and np.all(got["step"] == 500)
    assert int(got["cnt"][:, 2].sum()) == st["flips"]


def test_c2_bench_launch_configuration(fg, orc):
    """The launch configuration bench.py times (C2: 16384 walkers, 10^4-step phases, the
    default kernel with its step-chunk tasks), two phases; 256 sampled trajectories
    bit-exact, every final and best scheme of a 1-in-16 sample satisfies
    the Brent equations on the device."""
    wl = WORKLOADS["c2_333_zt"]
    W, steps = wl.walkers, 20000
    g = _ctx(fg, 3, 3, 3, ZT, wl.r_cap, W)
    g.seed_naive()
    p = fg.params_default(phase_steps=10000)
    g.walk(steps, wl.seed, p)
    got = g.get_walkers()
    ids = sample_walkers(W, 256, seed=2025)
    ref = orc.run_walkers(3, 3, 3, ZT, wl.r_cap, 0, 0, steps, wl.seed, ids=ids)
    _assert_same(got, ref, idx=ids, what="c2-bench")
    st = g.stats()
    assert st["verify_fail"] == 0 and st["walk_launches"] == 2
    sample = list(range(0, W, 16))
    ok, _ = g.verify_batch([got["rows"][k][: got["r"][k]] for k in sample])
    assert np.all(ok == 1)
    ok, _ = g.verify_batch([got["best"][k][: got["best_r"][k]] for k in sample])
    assert np.all(ok == 1)


@pytest.mark.parametrize("ring", [ZT, Z2])
def test_c2_every_walker(fg, orc, ring):
    """C2 at full size, EVERY one of the 16384 walkers (digest, ranks, counters, current
    and best rows) against the oracle over two 600-step launches of the default kernel
    (chunked tasks: 16384 walkers give the 592 schedulers 3-4 warps each)."""
    wl = WORKLOADS["c2_333_zt"]
    W, steps = wl.walkers, 1200
    g = _ctx(fg, 3, 3, 3, ring, wl.r_cap, W)
    g.seed_naive()
    g.walk(steps, wl.seed + 7 * ring, fg.params_default(phase_steps=600))
    got = g.get_walkers()
    ref = orc.run_walkers(3, 3, 3, ring, wl.r_cap, W, 0, steps, wl.seed + 7 * ring)
    _assert_same(got, ref, idx=None, what="c2-all")
    assert g.stats()["verify_fail"] == 0


def test_virtual_ranks_match_single_gpu(fg):
    """SURVEY 4.3 multi-GPU: G ranks owning disjoint global walker-id ranges produce,
    walker by walker, the states of one context over all ids (the trajectory depends
    only on (seed, global id, step)); the merge of the per-rank best records equals the
    single context's best.  Two "virtual ranks" on one GPU, with a restart from the
    merged pool in between (R23), as bench.py's multi-rank path does."""
    from paper_2511_20317_b200.pool_sync import merge_gathered
    W, half, steps, seed = 3000, 1500, 2500, 0x2511203170000009
    one = _ctx(fg, 3, 3, 3, ZT, 32, W, base=0)
    ranks = [_ctx(fg, 3, 3, 3, ZT, 32, half, base=0), _ctx(fg, 3, 3, 3, ZT, 32, half, base=half)]
    for g in [one] + ranks:
        g.seed_naive()
    for phase in range(2):
        one.walk(steps, seed + phase)
        for g in ranks:
            g.walk(steps, seed + phase)
        # pool sync: all-gather of the per-rank records, identical merge on every rank
        recs = np.stack([g.export_best() for g in ranks])
        merged = merge_gathered(recs, 2, 32)
        b1 = one.best()
        assert merged["rank"] == b1["rank"] and merged["walker_id"] == b1["walker_id"]
        for g in ranks:
            g.import_best(recs.reshape(-1), 2)
        one.import_best(np.stack([one.export_best()]).reshape(-1), 1)
        got1 = one.get_walkers()
        for k, g in enumerate(ranks):
            gk = g.get_walkers()
            sl = slice(k * half, (k + 1) * half)
            for key in ("r", "best_r", "digest", "cnt", "rows", "best"):
                assert np.array_equal(gk[key], got1[key][sl]), (phase, k, key)
        # restart stagnant walkers from the merged pool on every context (same pool)
        n1 = one.restart(0)
        nr = sum(g.restart(0) for g in ranks)
        assert n1 == nr
