"""Exploratory search at scale (the lifecycle of PAPER:266-293): a population
seeded with Strassen (2,2,2:7) and naive schemes of a few small formats, R rounds of
(GPU walk -> registry sync -> Resize on the host, Alg. 2).  Records the registry's best
(rank, additions) per format after every round and re-verifies every best on the host.

  python scripts/explore_run.py <walkers> <rounds> <steps_per_round> <out.json>
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_io import load_scheme  # noqa: E402
from paper_2511_20317_b200 import fg  # noqa: E402
from paper_2511_20317_b200.explore import Explorer  # noqa: E402


def naive(m, n, p):
    rows = []
    for i in range(m):
        for j in range(n):
            for k in range(p):
                u = np.zeros(m * n, np.int8); u[i * n + j] = 1
                v = np.zeros(n * p, np.int8); v[j * p + k] = 1
                w = np.zeros(p * m, np.int8); w[k * m + i] = 1
                rows.append(np.concatenate([u, v, w]))
    return np.array(rows, dtype=np.int8)


def main():
    W, rounds, steps, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    _, _, _, strassen = load_scheme("sec36_after.txt")
    seeds = [((2, 2, 2), strassen), ((2, 2, 3), naive(2, 2, 3)), ((2, 3, 3), naive(2, 3, 3)),
             ((3, 3, 3), naive(3, 3, 3)), ((2, 2, 4), naive(2, 2, 4))]
    pop = [seeds[k % len(seeds)] for k in range(W)]
    ex = Explorer(pop, seed=0x2511, stream=torch.cuda.current_stream().cuda_stream, thr_resize=1 << 30)
    trace = []
    t0 = time.time()
    for rnd in range(rounds):
        ops = ex.round(steps)
        best = {f"{f[0]},{f[1]},{f[2]}": [int(r), int(a)] for f, (r, a, _) in sorted(ex.registry.best.items())}
        trace.append({"round": rnd, "wall_s": round(time.time() - t0, 1), "formats": len(ex.formats()),
                      "diversity": ex.diversity(), "applied_resizes": int(sum(1 for o in ops if o >> 1)),
                      "best": best})
        print(json.dumps(trace[-1]), flush=True)
    checks = {}
    for f, (r, a, c) in sorted(ex.registry.best.items()):
        rc, _ = fg.fg_verify(*f, fg.FG_ZT, c)
        checks[f"{f[0]},{f[1]},{f[2]}"] = {"rank": int(r), "additions": int(a), "naive_rank": f[0] * f[1] * f[2],
                                           "host_brent_check": "ok" if rc == 0 else "FAIL"}
    archive = {f"{f[0]},{f[1]},{f[2]}": len(v) for f, v in sorted(ex.registry.archive.items())}
    with open(out, "w") as fh:
        json.dump({"walkers": W, "rounds": rounds, "steps_per_round": steps, "wall_s": round(time.time() - t0, 1),
                   "final": checks, "archive_sizes": archive, "trace": trace}, fh)
    print(json.dumps(checks))


if __name__ == "__main__":
    main()
