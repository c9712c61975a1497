"""Long walk on one workload: the time-to-rank ladder and the best scheme after a fixed
device-time budget ("best rank reached in a fixed budget").  Plain Alg. 1
phases from naive seeds (no restarts, no Resize); the ladder is exact (verified strict
improvements' step indices, fg_rank_first_steps), the best scheme is re-verified on the
host (fg_verify, exact integer Brent check) and written with its invariants.

  python scripts/long_run.py <workload | m,n,p,ring,R,walkers[,target]> <seconds> <out.json>
                             [restart_every_phases slack [k_flip]]

With a restart period, every that many phases the box-wide best becomes the pool
(fg_export_best -> fg_import_best) and walkers whose best rank exceeds it by more than
`slack` are re-seeded from it (fg_restart, R23; PAPER:290 population synchronisation).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import PHASE_MULTI, ladder_from_first  # noqa: E402
from paper_2511_20317_b200 import fg  # noqa: E402
from paper_2511_20317_b200.inputs import WORKLOADS  # noqa: E402


def main():
    key, budget, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    every = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    slack = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    k_flip = int(sys.argv[6]) if len(sys.argv) > 6 else 0       # 0: the default K (R11)
    run(key, budget, out, every, slack, k_flip)


def run(key, budget, out, every=0, slack=2, k_flip=0, seed_coeffs=None, seed_note="naive"):
    params = fg.params_default(k_flip=k_flip) if k_flip else None
    restarted = 0
    if key in WORKLOADS:
        wl = WORKLOADS[key]
    else:
        # an ad-hoc format "m,n,p,ring,R,walkers[,target]" (PAPER tables' formats)
        from paper_2511_20317_b200.inputs import Workload
        f = [int(x) for x in key.split(",")]
        wl = Workload(f"({f[0]},{f[1]},{f[2]}) {'Z_T' if f[3] == 0 else 'Z_2'} naive {f[0] * f[1] * f[2]}",
                      f[0], f[1], f[2], f[3], f[4], f[5], f[6] if len(f) > 6 else None, 99)
    S = 10000 if wl.r_cap <= 32 else PHASE_MULTI
    stream = torch.cuda.current_stream()
    g = fg.FlipGraph(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, wl.walkers, 0, 0, stream.cuda_stream)
    if seed_coeffs is None:
        g.seed_naive()
    else:
        g.seed_pool(seed_coeffs)
    phase_ms, trace = [], []
    t0 = time.time()
    while sum(phase_ms) < budget * 1000.0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.walk(S, wl.seed, params)
        e1.record(stream)
        torch.cuda.synchronize()
        phase_ms.append(e0.elapsed_time(e1))
        if every and len(phase_ms) % every == 0:
            g.import_best(g.export_best(), 1)
            restarted += g.restart(slack)
        if len(phase_ms) % 25 == 1:
            b = g.best()
            trace.append({"device_s": round(sum(phase_ms) / 1000.0, 3), "best_rank": b["rank"],
                          "best_additions": b["additions"]})
    first = [int(x) for x in g.rank_first_steps(wl.r_cap)]
    naive = wl.m * wl.n * wl.p
    seeded = naive if seed_coeffs is None else int(seed_coeffs.shape[0])
    lad = ladder_from_first(first, phase_ms, S, naive, seeded_rank=seeded)
    b = g.best()
    rc, ff = fg.fg_verify(wl.m, wl.n, wl.p, wl.ring, b["coeffs"])
    t, sums = fg.fg_type_invariant(wl.m, wl.n, wl.p, wl.ring, b["coeffs"])
    st = g.stats()
    res = {"workload": wl.name, "walkers": wl.walkers, "phase_steps": S, "phases": len(phase_ms),
           "device_s": round(sum(phase_ms) / 1000.0, 3), "wall_s": round(time.time() - t0, 1),
           "walker_steps_per_s": wl.walkers * S * len(phase_ms) / (sum(phase_ms) / 1000.0),
           "seed": seed_note, "kernel": g.kernel_name, "k_flip": k_flip or 16, "restart": {"every_phases": every, "slack": slack, "restarted": restarted},
           "time_to_rank_s": {str(k): round(v[0], 4) for k, v in sorted(lad.items())},
           "steps_to_rank": {str(k): v[1] for k, v in sorted(lad.items())},
           "best": {"rank": b["rank"], "additions": b["additions"], "walker_id": b["walker_id"],
                    "host_brent_check": "ok" if rc == 0 else f"FAIL {list(ff)}",
                    "type_invariant": {f"{a},{bb},{c}": v for (a, bb, c), v in sorted(t.items())},
                    "rank_sums": list(sums), "coeffs": np.asarray(b["coeffs"]).astype(int).tolist()},
           "target_rank_context": wl.target_rank, "trace": trace,
           "verify": {k: st[k] for k in ("verified", "verify_fail", "queue_overflow")}}
    with open(out, "w") as fh:
        json.dump(res, fh)
    print(json.dumps({k: v for k, v in res.items() if k not in ("best", "trace")}))
    print("best", res["best"]["rank"], res["best"]["additions"], res["best"]["host_brent_check"])
    g.close()


if __name__ == "__main__":
    main()
