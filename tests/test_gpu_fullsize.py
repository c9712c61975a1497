"""GPU parity in the launch configurations the bench numbers come from (VERDICT r1
item 2), plus the host-side guards of the ADVICE r1 fixes.

- C3 (Z_T and Z_2), C4 and the C5 formats at their full walker counts and the
  bench's phase length: the default kernel runs its real task schedule (walk_ql's
  chunk hand-over at 1.26 waves, the multi-row kernels' persistent walker queue
  with several walkers per warp), and sampled trajectories must equal the oracle's.
- Seeds that force strict improvements on the two-word layouts (P32, P64, PZ64):
  naive with one term split in two, so the first reduction lowers the rank below
  the seeded best and the improvement goes through the verify queue (R19).
- The batched verifier's failing path at the large formats (mn*np > 256 threads,
  pm = 48 / 54): the first failing (a,b,c) of every corrupted scheme equals the
  oracle's.
"""
import numpy as np
import pytest

from oracle import Oracle
from paper_2511_20317_b200.inputs import WORKLOADS, perturbations, sample_walkers

pytestmark = pytest.mark.gpu
ZT, Z2 = 0, 1
CNT_IMPROVEMENTS, CNT_VERIFY_FAIL = 9, 11


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


def _same(got, ref, ids, what):
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        g = got[k][ids]
        if not np.array_equal(g, ref[k]):
            bad = np.nonzero(np.any((g != ref[k]).reshape(len(g), -1), axis=1))[0]
            raise AssertionError(f"{what}: {k} differs for sampled walkers {ids[bad[:8]]}")


# the phase length bench.py uses for the multi-row configs (bench.PHASE_MULTI)
PHASE_MULTI = 2000

FULL = [
    # (workload, steps, sampled walkers)
    ("c3_444_zt", 2000, 10),
    ("c3_444_z2", 2000, 10),
    ("c4_555_zt", 2000, 8),
    ("c5_4512_zt", 600, 8),
    ("c5_679_zt", 500, 8),
]


@pytest.mark.parametrize("case", FULL, ids=lambda c: c[0])
def test_bench_launch_configuration(fg, orc, case):
    name, steps, k = case
    wl = WORKLOADS[name]
    g = _ctx(fg, *wl.fmt, wl.ring, wl.r_cap, wl.walkers)
    g.seed_naive()
    g.walk(steps, wl.seed, fg.params_default(phase_steps=PHASE_MULTI))
    got = g.get_walkers()
    # the walkers the last tasks of the launch ran, plus a seeded sample
    ids = np.unique(np.concatenate([sample_walkers(wl.walkers, k, seed=wl.config_id),
                                    np.arange(wl.walkers - 3, wl.walkers)]))
    ref = orc.run_walkers(*wl.fmt, wl.ring, wl.r_cap, 0, 0, steps, wl.seed, ids=ids)
    _same(got, ref, ids, f"{name} ({g.kernel_name})")
    st = g.stats()
    assert st["verify_fail"] == 0 and st["queue_overflow"] == 0
    assert np.all(got["step"] == steps)
    sample = list(range(0, wl.walkers, max(1, wl.walkers // 24)))
    ok, _ = g.verify_batch([got["best"][w][: got["best_r"][w]] for w in sample])
    assert np.all(ok == 1)
    b = g.best()
    assert b["rank"] == int(got["best_r"].min())
    assert fg.fg_verify(*wl.fmt, wl.ring, b["coeffs"])[0] == 0


def split_seed(orc, m, n, p, ring):
    """Naive (m,n,p) with term 0 = u0 (x) v0 (x) e_c written as u0 (x) v0 (x) (e_c + e_d)
    + u0 (x) v0 (x) (-e_d) (Z_2: + e_d): rank mnp + 1 with one reducible pair."""
    c = orc.naive(m, n, p)
    mn, np_ = m * n, n * p
    d = 1 * m + 1                      # w of terms (1, *, 1): shares neither u0 nor v0
    extra = c[0].copy()
    c[0, mn + np_ + d] = 1
    extra[mn + np_:] = 0
    extra[mn + np_ + d] = 1 if ring == Z2 else -1
    out = np.concatenate([c, extra[None]], axis=0)
    assert orc.verify(m, n, p, ring, out)[0] == 0
    return out


IMPROVE = [((5, 5, 5), ZT, 160, 300), ((4, 5, 12), ZT, 256, 200), ((6, 7, 9), ZT, 416, 160),
           ((4, 5, 12), Z2, 256, 200), ((4, 4, 4), ZT, 96, 300), ((4, 4, 4), Z2, 96, 300)]


@pytest.mark.parametrize("case", IMPROVE, ids=lambda c: f"{c[0]}-{'ZT' if c[1] == 0 else 'Z2'}")
def test_forced_strict_improvements_through_the_queue(fg, orc, case):
    (m, n, p), ring, R, W = case
    seedc = split_seed(orc, m, n, p, ring)
    g = _ctx(fg, m, n, p, ring, R, W, base=900)
    g.seed_pool(seedc)
    steps = 300
    g.walk(steps, 0x51EED)
    got = g.get_walkers()
    impr = int(got["cnt"][:, CNT_IMPROVEMENTS].sum())
    st = g.stats()
    # most walkers reduce the split pair within the first steps: strict improvements
    assert impr >= W // 2, impr
    assert st["verified"] == impr and st["verify_fail"] == 0 and st["queue_overflow"] == 0
    ids = sample_walkers(W, 6, seed=R)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, 0x51EED, seed_coeffs=seedc, ids=ids + 900)
    _same(got, ref, ids, f"improve {(m, n, p)}")


@pytest.mark.parametrize("fmt,R", [((4, 5, 12), 256), ((6, 7, 9), 416), ((5, 5, 5), 160)])
@pytest.mark.parametrize("ring", [ZT, Z2])
def test_verifier_failing_path_large_formats(fg, orc, fmt, R, ring):
    m, n, p = fmt
    g = _ctx(fg, m, n, p, ring, R, 32)
    g.seed_naive()
    g.walk(400, 0xBAD + ring)
    got = g.get_walkers()
    schemes = [got["best"][k][: got["best_r"][k]] for k in range(0, 32, 4)]
    width = m * n + n * p + p * m
    for (l, e, v) in perturbations(400, width, ring, 48, seed=R + ring):
        c = schemes[l % 8].copy()
        row = l % len(c)
        if c[row, e] == v:                  # always change the coefficient
            v = 1 - v if ring == Z2 else (v + 2) % 3 - 1
        c[row, e] = v
        schemes.append(c)
    ok, ff = g.verify_batch(schemes)
    nfail = 0
    for k, c in enumerate(schemes):
        rc, off = orc.verify(m, n, p, ring, c)
        assert ok[k] == (1 if rc == 0 else 0), k
        assert tuple(ff[k]) == off, (k, tuple(ff[k]), off)
        nfail += rc != 0
    assert nfail >= 30


# ---------------- ADVICE r1 guards (host side of libfg) ----------------

def test_partial_seed_is_not_walkable(fg, orc):
    """A context whose walkers are only partly seeded has no best and cannot walk;
    once every walker is covered it behaves like a fully seeded one."""
    g = _ctx(fg, 3, 3, 3, ZT, 32, 40)
    naive = orc.naive(3, 3, 3)
    g.seed_pool(naive, 0, 20)
    with pytest.raises(fg.FgError) as e:
        g.walk(10, 1)
    assert e.value.status == -6
    with pytest.raises(fg.FgError):
        g.best()
    g.seed_pool(naive, 20, 40)
    g.walk(500, 1)
    b = g.best()
    assert 1 <= b["rank"] <= 27 and fg.fg_verify(3, 3, 3, ZT, b["coeffs"])[0] == 0


HDR = 128          # fg_whdr bytes: r, best_r, step, digest, cnt[12], best_adds, pad


def _state_views(buf, W, R):
    """Views of fg_save_state's image (include/fg.h): 64-byte header (word 10 = bytes per
    plane word), walker headers, then the current and the best planes packed to that width."""
    bw = int(np.frombuffer(bytes(buf[40:44]), np.uint32)[0])
    hdr = buf[64: 64 + HDR * W].reshape(W, HDR)
    words = 6 * R * bw
    cur = buf[64 + HDR * W: 64 + HDR * W + words * W].reshape(W, words)
    best = buf[64 + HDR * W + words * W: 64 + HDR * W + 2 * words * W].reshape(W, words)
    return hdr, cur, best


def test_unverified_best_never_becomes_the_local_best(fg, orc):
    """R19: a walker whose best scheme fails the Brent equations cannot supply the
    local best.  A state image whose lowest-rank walker holds a broken scheme is
    rejected (FG_E_INVALID_SCHEME); the same walker flagged with a failed
    verification (cnt[VERIFY_FAIL] > 0) is skipped and the best comes from the others."""
    W, R = 16, 32
    a = _ctx(fg, 3, 3, 3, ZT, R, W)
    a.seed_naive()
    a.walk(3000, 5)
    good = a.best()
    img = np.array(a.save_state(), dtype=np.uint8).copy()
    hdr, cur, best = _state_views(img, W, R)
    k = (good["walker_id"] + 1) % W
    hdr[k, 4:8] = np.frombuffer(np.int32(5).tobytes(), np.uint8)      # best_r = 5: beats everyone
    best[k, :] = 0
    best[k, :1] = 1                                                    # not a scheme
    b = _ctx(fg, 3, 3, 3, ZT, R, W)
    with pytest.raises(fg.FgError) as e:
        b.load_state(img)
    assert e.value.status == -4
    hdr[k, 24 + 8 * CNT_VERIFY_FAIL: 32 + 8 * CNT_VERIFY_FAIL] = np.frombuffer(np.uint64(1).tobytes(), np.uint8)
    c = _ctx(fg, 3, 3, 3, ZT, R, W)
    c.load_state(img)
    got = c.best()
    assert got["rank"] == good["rank"] and got["walker_id"] != k
    assert fg.fg_verify(3, 3, 3, ZT, got["coeffs"])[0] == 0


def test_local_best_keeps_fewer_additions(fg, orc):
    """R20: the local best only changes for a lexicographically smaller (rank,
    additions, id); a later walk whose walkers' bests drifted to more additions at
    the same rank (plateau acceptance) does not replace it."""
    g = _ctx(fg, 3, 3, 3, ZT, 32, 64)
    g.seed_naive()
    seen = []
    for ph in range(6):
        g.walk(2000, 0x77)
        b = g.best()
        seen.append((b["rank"], b["additions"], b["walker_id"]))
    for x, y in zip(seen, seen[1:]):
        assert y <= x, seen


def test_rank_first_steps_match_oracle(fg, orc):
    """Exact time-to-rank (fg_rank_first_steps): on C1, the first step index at which
    any walker's best reaches each rank equals the oracle's, found by stepping every
    oracle walker one iteration at a time."""
    wl = WORKLOADS["c1_222_zt"]
    W, steps = 64, 30000
    g = _ctx(fg, 2, 2, 2, ZT, wl.r_cap, W)
    g.seed_naive()
    g.walk(steps, wl.seed, fg.params_default(phase_steps=7000))
    first = g.rank_first_steps(8)
    U = (1 << 64) - 1
    exp = [U] * 9
    exp[8] = 0
    for k in range(W):
        w = orc.walker(2, 2, 2, ZT, wl.r_cap, walker_id=k)
        w.seed_naive()
        b = 8
        for s in range(steps):
            w.walk(1, wl.seed)
            if w.best_r < b:
                b = w.best_r
                exp[b] = min(exp[b], s)
            if b == 7:
                break
    assert [int(x) for x in first] == exp, (first, exp)
