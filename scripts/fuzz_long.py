"""Long seeded parity fuzz on the GPU (not part of the default suite): random formats,
rings, row capacities, Alg. 1 parameters, walker counts and step counts through every
built walk kernel (default selection and the FG_WALK_KERNEL / chunk overrides), sampled
walkers compared bit for bit with the oracle (rows, best rows, ranks, counters, per-step
digest).  Prints one line per configuration and a final tally.

  python scripts/fuzz_long.py [n_per_family] [seed] [seconds]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Oracle, OracleParams  # noqa: E402
from paper_2511_20317_b200 import fg  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
SEED = int(sys.argv[2]) if len(sys.argv) > 2 else 777
BUDGET = float(sys.argv[3]) if len(sys.argv) > 3 else 900.0
rng = np.random.default_rng(SEED)
orc = Oracle()
st = torch.cuda.current_stream().cuda_stream


def draw_format(family):
    while True:
        if family in ("q4", "w32"):
            m, n, p = (int(x) for x in rng.integers(1, 4, size=3))
        elif family == "ql":
            m, n, p = (int(x) for x in rng.integers(2, 5, size=3))
        else:
            m, n, p = (int(x) for x in rng.integers(1, 8, size=3))
        ring = int(rng.integers(0, 2))
        naive = m * n * p
        maxlen = max(m * n, n * p, p * m)
        if maxlen > 64 or naive > 300:
            continue
        if family in ("q4", "w32"):
            if naive + 1 > 32 or (family == "q4" and maxlen > (16 if ring == 0 else 32)):
                continue
            R = int(min(32, naive + rng.integers(1, 9)))
        elif family == "ql":
            if maxlen > (16 if ring == 0 else 32) or naive < 20 or naive + 8 > 128:
                continue
            R = int(min(128, naive + rng.integers(4, 30)))
        else:
            if naive < 8:
                continue
            R = int(min(512, naive + rng.integers(4, 40)))
            if R <= 32:
                continue
        return (m, n, p), ring, R


def env_for(family):
    e = {"q4": {"FG_WALK_KERNEL": "q4"}, "w32": {"FG_WALK_KERNEL": "w32"}, "ql": {"FG_WALK_KERNEL": "ql"},
         "wl": {"FG_WALK_KERNEL": "wl"}, "wm": {"FG_WALK_KERNEL": "wm"}}[family]
    if family == "q4" and rng.random() < 0.5:
        e["FG_Q4_CHUNKS"] = str(int(rng.integers(2, 12)))
    if family == "ql" and rng.random() < 0.5:
        e["FG_QL_CHUNKS"] = str(int(rng.integers(2, 9)))
    if family == "wl" and rng.random() < 0.3:
        e["FG_DBG"] = "1"
    return e


t_start = time.time()
bad = tot = 0
for family in ("q4", "w32", "ql", "wl", "wm"):
    for it in range(N):
        if time.time() - t_start > BUDGET:
            break
        (m, n, p), ring, R = draw_format(family)
        prm = dict(k_flip=int(rng.integers(1, 17) if rng.random() < 0.75 else rng.integers(17, 65)), thr_accept_eq=int(rng.integers(0, 1 << 31)),
                   thr_reduce=int(rng.integers(0, 1 << 32)), thr_expand=int(rng.integers(0, 1 << 29)),
                   expand_slack=int(rng.integers(-1, 4)))
        cm = rng.random() < 0.2          # R24 (naive-complexity) mode on a fifth of the runs
        W = int(rng.choice([17, 64, 203, 600, 2100]))
        steps = int(rng.integers(200, 1500))
        seed = int(rng.integers(1, 1 << 62))
        env = env_for(family)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            g = fg.FlipGraph(m, n, p, ring, R, W, 0, 0, st)
            kname = g.kernel_name
            g.seed_naive()
            params = fg.params_default(phase_steps=steps // 2 + 1, flags=fg.FG_FLAG_COMPLEXITY if cm else 0, **prm)
            g.walk(steps, seed, params)
            got = g.get_walkers()
            g.close()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        ids = np.array(sorted(set([0, W - 1] + [int(x) for x in rng.integers(0, W, size=6)])), dtype=np.int64)
        op = OracleParams.default(mode=1 if cm else 0, **prm)
        ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, seed, params=op, ids=ids)
        diff = [k for k in ("r", "best_r", "digest", "cnt", "rows", "best") if not np.array_equal(got[k][ids], ref[k])]
        tot += 1
        bad += bool(diff)
        print(f"{family:3s} {(m, n, p)} ring {ring} R {R:3d} W {W:5d} steps {steps:5d} {kname:16s} "
              f"env {env} params {prm}{' R24' if cm else ''}: {'OK' if not diff else 'DIFF ' + ','.join(diff)}", flush=True)
print(f"{tot - bad}/{tot} configurations bit-exact ({time.time() - t_start:.0f} s)")
sys.exit(1 if bad else 0)
