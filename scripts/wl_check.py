"""Quick walk_wl check on the GPU: structure self-check (FG_DBG=1) and sampled parity
against the oracle on several formats.  Usage: FG_DBG=1 python scripts/wl_check.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle  # noqa: E402
from paper_2511_20317_b200 import fg  # noqa: E402

orc = Oracle()
cases = [((5, 5, 5), 0, 160, 64, 3000), ((6, 7, 9), 0, 416, 16, 1500), ((4, 5, 12), 1, 256, 32, 2000),
         ((5, 5, 5), 0, 160, 64, 300), ((4, 4, 4), 0, 96, 64, 600), ((3, 3, 3), 0, 40, 64, 1500),
         ((4, 5, 12), 0, 256, 32, 200), ((4, 5, 12), 1, 256, 32, 200), ((6, 7, 9), 0, 416, 16, 150),
         ((4, 4, 4), 1, 160, 32, 500), ((2, 3, 4), 0, 64, 64, 2000),
         ((2, 2, 16), 0, 96, 64, 2000), ((2, 3, 20), 0, 160, 32, 1500), ((1, 1, 40), 0, 64, 32, 1500),
         ((1, 2, 30), 1, 96, 32, 1500)]
only = sys.argv[1:] and int(sys.argv[1])
st = torch.cuda.current_stream().cuda_stream
bad = 0
for ci, ((m, n, p), ring, R, W, steps) in enumerate(cases):
    if only and ci != only - 1:
        continue
    g = fg.FlipGraph(m, n, p, ring, R, W, 7, 0, st)
    g.seed_naive()
    t0 = time.time()
    h = steps // 2
    g.walk(h, 12345)
    g.walk(steps - h, 12345)
    torch.cuda.synchronize()
    got = g.get_walkers()
    ids = np.array(sorted(set([0, W - 1, W // 2, 3])), dtype=np.int64)
    ref = orc.run_walkers(m, n, p, ring, R, 0, 0, steps, 12345, ids=ids + 7)
    res = []
    for k in ("r", "best_r", "digest", "cnt", "rows", "best"):
        ok = np.array_equal(got[k][ids], ref[k])
        res.append(f"{k}={'ok' if ok else 'DIFF'}")
        bad += not ok
    print(f"{(m, n, p)} ring {ring} R {R} {g.kernel_name}: {' '.join(res)} "
          f"r={got['r'][ids].tolist()} oracle r={ref['r'].tolist()} ({time.time() - t0:.2f}s)", flush=True)
    g.close()
print("BAD" if bad else "ALL OK")
