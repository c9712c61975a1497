"""Pool-sync cost on the device: export / all-gather (NCCL) / import / best, per phase.
  python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 scripts/xchg_time.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
torch.cuda.set_device(0)
from paper_2511_20317_b200 import fg
from paper_2511_20317_b200.pool_sync import PoolSync
from paper_2511_20317_b200.inputs import WORKLOADS
wl = WORKLOADS["c2_333_zt"]
st = torch.cuda.current_stream()
g = fg.FlipGraph(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, wl.walkers, 0, 0, st.cuda_stream)
g.seed_naive(); g.walk(2000, wl.seed)
sync = PoolSync(g)
T = {k: [] for k in ("export", "gather", "import", "best", "exchange", "walk100")}
for it in range(30):
    torch.cuda.synchronize(); t0 = time.perf_counter(); rec = g.export_best(); torch.cuda.synchronize(); T["export"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); recs = sync.gather_records(rec); torch.cuda.synchronize(); T["gather"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); g.import_best(np.ascontiguousarray(recs.reshape(-1)), 1); torch.cuda.synchronize(); T["import"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); g.best(); torch.cuda.synchronize(); T["best"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); sync.exchange(); torch.cuda.synchronize(); T["exchange"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); g.walk(100, wl.seed); torch.cuda.synchronize(); T["walk100"].append(time.perf_counter() - t0)
for k, v in T.items():
    v = np.array(v[5:]) * 1e6
    print(f"{k:9s} median {np.median(v):8.1f} us  min {v.min():8.1f}")
dist.destroy_process_group()
