"""Per-step event rates of a workload on the GPU (draws, flips, expands, merges)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_20317_b200 import fg  # noqa: E402
from paper_2511_20317_b200.inputs import WORKLOADS  # noqa: E402

for name in sys.argv[1:]:
    wl = WORKLOADS[name]
    W = min(wl.walkers, 2048)
    g = fg.FlipGraph(*wl.fmt, wl.ring, wl.r_cap, W, 0, 0, torch.cuda.current_stream().cuda_stream)
    g.seed_naive()
    for ph in range(3):
        g.walk(2000, wl.seed)
        got = g.get_walkers(rows=False)
        c = got["cnt"].sum(axis=0).astype(float)
        steps = c[0]
        names = ["steps", "draws", "flips", "flip_fail", "expand_ok", "expand_reject", "merges",
                 "zero_removed", "best_copies", "improvements", "reduce_calls", "verify_fail"]
        print(name, g.kernel_name, f"after {int(steps / W)} steps: r mean {got['r'].mean():.1f} best min {got['best_r'].min()}",
              " ".join(f"{n}/step={c[k] / steps:.4f}" for k, n in enumerate(names) if k), flush=True)
