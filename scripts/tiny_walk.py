"""Tiny walk for debugging tools (compute-sanitizer): 64 walkers x N steps."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_20317_b200 import fg
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
m, n, p = (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,2,2").split(","))
g = fg.FlipGraph(m, n, p, 0, 32, 64, 0, 0, torch.cuda.current_stream().cuda_stream)
g.seed_naive()
g.walk(steps, 12345)
print("ok", g.kernel_name, g.get_walkers(rows=False)["r"][:8])
