"""bench.py -- flip-steps/s of the B200 flip-graph walker (BASELINE.json metric).

One bench "step" = one walk phase: every walker runs `--phase-steps` iterations of
Algorithm 1 on the device, the batched verifier checks every strict
improvement, and (N > 1) the per-rank best records are all-gathered over NCCL and
merged.  value = walker-steps of all ranks / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2_333_zt]
  python bench.py --impl reference ...   # the CPU oracle on the host cores
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "flip-steps/sec per box (1/2/4/8 B200) and time-to-target-rank; % int-issue peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2_333_zt")
    ap.add_argument("--phase-steps", type=int, default=10000)
    ap.add_argument("--walkers", type=int, default=0, help="walkers per GPU (0 = workload's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: total oracle time budget over warmup + steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for tests")
    return ap.parse_args()


# ---------------- integer roofline ----------------
# (kernel, workload) -> (dram bytes per launch, profile it comes from)
# and the capture's issue / ALU-pipe utilisation (the north star's "% int-issue" figures)
NCU_TRAFFIC = {
    ("walk_q4<P16>", "c2_333_zt"): (52.551424e6 + 7.051776e6, "profiles/r01_ncu_walk_q4.txt", 58.89, 50.5),
}


def model_ops_per_step(ring: int, r: float) -> float:
    """SURVEY.md 8(d) per-step algorithmic int32 ops: Z_T 30 r + 200, Z_2 15 r + 180."""
    return 30.0 * r + 200.0 if ring == 0 else 15.0 * r + 180.0


def int_peak_tops(sm_mhz: float, sms: int = 148) -> float:
    """Integer ALU pipe peak: 4 SMSPs x 16 lanes/clk (ALU rt = 2 cycles per warp
    instruction per SMSP, B300_MICROARCH.md 'Pipe rates') = 64 lanes/clk/SM."""
    return sms * 64 * sm_mhz * 1e6 / 1e12


# ---------------- clocks sampler (B200_PROFILING.md clocks line) ----------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# ---------------- CPU oracle (cpu_baseline / --impl reference) ----------------
def run_oracle_sample(wl, seconds: float):
    """Time the oracle as it stands on all host cores: walkers with global ids
    0..C*4-1 from naive, a step count calibrated to ~`seconds` of wall time."""
    from oracle import Oracle
    orc = Oracle()
    cores = os.cpu_count() or 1
    count = cores * 4
    t0 = time.perf_counter()
    orc.run_walkers(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, count, 0, 500, wl.seed, threads=cores,
                    want_rows=False)
    dt = time.perf_counter() - t0
    steps = max(500, int(500 * seconds / max(dt, 1e-3)))
    t0 = time.perf_counter()
    orc.run_walkers(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, count, 0, steps, wl.seed, threads=cores,
                    want_rows=False)
    dt = time.perf_counter() - t0
    return {"value": count * steps / dt, "unit": "flip-steps/s", "cores": cores, "kind": "oracle",
            "sample": f"{count} walkers x {steps} steps of {wl.name} from naive, "
                      f"{dt:.1f} s wall, OpenMP over walkers"}


def reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per = max(0.2, args.ref_seconds / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        run_oracle_sample(wl, per / 4)
    vals = []
    last = None
    t_all = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = run_oracle_sample(wl, per)
        t_all += time.perf_counter() - t0
        vals.append(last["value"])
    value = statistics.median(vals)
    cpu = dict(last)
    cpu["value"] = value
    out = {"metric": METRIC, "value": value, "unit": "flip-steps/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_all / max(1, args.steps),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": wl.name, "walkers_per_gpu": wl.walkers},
           "cpu_baseline": cpu,
           "e2e": {"value": value, "unit": "flip-steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------- our arm ----------------
def main():
    args = parse()
    from paper_2511_20317_b200.inputs import WORKLOADS
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, wl)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_20317_b200 import fg
    from paper_2511_20317_b200.pool_sync import PoolSync

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % torch.cuda.device_count()     # one GPU per rank (modulo only for tests)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.dist_backend)
    stream = torch.cuda.current_stream()
    W = args.walkers or wl.walkers
    g = fg.FlipGraph(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, W, rank * W, dev, stream.cuda_stream)
    sync = PoolSync(g, world)
    g.seed_naive()
    S = args.phase_steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    # time-to-rank ladder: device time since seeding until the box best first <= rank
    ladder = {}
    ladder_steps = {}            # box walker-steps done when each rank was first reached
    elapsed = [0.0]
    done_steps = [0]

    def phase(timed_events=None):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        g.walk(S, wl.seed)
        best = sync.exchange()
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        elapsed[0] += ms / 1000.0
        done_steps[0] += W * S * world
        for target in range(best["rank"], wl.m * wl.n * wl.p):
            ladder.setdefault(target, elapsed[0])
            ladder_steps.setdefault(target, done_steps[0])
        return ms

    for _ in range(args.warmup):
        flush.zero_()
        phase()
    st0 = g.stats()
    r_before = g.get_walkers(rows=False)["r"].mean()
    clocks = Clocks(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        flush.zero_()                       # L2 flushed between timed steps (not timed)
        times.append(phase())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st1 = g.stats()
    r_after = g.get_walkers(rows=False)["r"].mean()
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64,
                     device="cuda" if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    walker_steps = float(W) * S * args.steps * world
    value = walker_steps / (total_ms / 1000.0)

    # dominant kernel (walk) timed live with CUDA events inside libfg, on its stream
    walk_ms = (st1["walk_us"] - st0["walk_us"]) / 1000.0
    launches = st1["walk_launches"] - st0["walk_launches"]
    per_launch_ms = walk_ms / max(1, launches)
    r_mean = 0.5 * (r_before + r_after)
    ops = model_ops_per_step(wl.ring, r_mean) * W * S       # per launch
    achieved = ops / (per_launch_ms / 1000.0) / 1e12
    sm_mhz = clk.get("sm_mhz") or 1965.0
    peak = int_peak_tops(sm_mhz)
    # DRAM bytes per launch from the committed `ncu --set full` capture of this kernel
    # on this workload (dram__bytes_read.sum + dram__bytes_write.sum), if there is one
    traffic = NCU_TRAFFIC.get((g.kernel_name, args.workload))
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                "frac": achieved / peak, "traffic": traffic[0] if traffic else None,
                "traffic_unit": "B/launch", "traffic_source": traffic[1] if traffic else None,
                "ncu_issue_active_pct": traffic[2] if traffic else None,
                "ncu_alu_pipe_pct": traffic[3] if traffic else None,
                "kernel": g.kernel_name, "kernel_ms_per_launch": per_launch_ms,
                "kernel_share_of_step": walk_ms / total_ms if total_ms else None,
                "ops_per_step_model": model_ops_per_step(wl.ring, r_mean),
                "peak_basis": f"148 SMs x 64 int32 lanes/clk x {sm_mhz:.0f} MHz (median under load)"}

    # e2e through the C ABI with host buffers: H2D state, walk, D2H state every step
    e2e = None
    if not args.no_e2e:
        nbytes = g.state_bytes()
        host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        g.save_state(host.data_ptr())
        e_times = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.load_state(host.data_ptr())
            g.walk(S, wl.seed)
            sync.exchange()
            g.save_state(host.data_ptr())
            torch.cuda.synchronize()
            e_times.append(time.perf_counter() - t0)
        te = torch.tensor([sum(e_times)], dtype=torch.float64,
                          device="cuda" if args.dist_backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(W) * S * len(e_times) * world / float(te.item()), "unit": "flip-steps/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_oracle_sample(wl, args.cpu_seconds)
        # the trajectories are identical on the CPU (parity), so the oracle reaches each
        # rank after the same walker-steps: time = steps / its measured rate (extrapolated)
        cpu["time_to_rank_s_extrapolated"] = {str(k): round(v / cpu["value"], 1)
                                              for k, v in sorted(ladder_steps.items())}

    best = g.best()
    stats = {k: st1[k] - st0[k] for k in ("verified", "verify_fail", "queue_overflow")}
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "flip-steps/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
               "data": "synthetic",
               "config": {"workload": wl.name, "walkers_per_gpu": W, "phase_steps": S,
                          "seed": hex(wl.seed), "l2": "flushed (256 MB write) between timed steps",
                          "kernel": g.kernel_name},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(st1["launches"] - st0["launches"]),
               "clocks": clk,
               "time_to_rank_s": {str(k): round(v, 4) for k, v in sorted(ladder.items())},
               "best": {"rank": best["rank"], "additions": best["additions"]},
               "verify": stats}
        print(json.dumps(out), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
