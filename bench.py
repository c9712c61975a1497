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
    ap.add_argument("--no-per-config", action="store_true", help="skip the other BASELINE workloads")
    ap.add_argument("--per-config-steps", type=int, default=4, help="timed phases per other workload")
    ap.add_argument("--per-config-ladder-s", type=float, default=3.0,
                    help="device seconds each other workload walks for its time-to-rank ladder")
    return ap.parse_args()


# ---------------- integer roofline ----------------
# (kernel, workload) -> (dram bytes per launch, profile it comes from)
# and the capture's issue / ALU-pipe utilisation (the north star's "% int-issue" figures)
NCU_TRAFFIC = {
    ("walk_q4<P16>", "c2_333_zt"): (54.7328e6 + 28.400896e6, "profiles/r02_ncu_walk_q4_c2_333_zt.txt", 58.84, 52.7),
    ("walk_q4<PZ2>", "c2_333_z2"): (28.868096e6 + 32.758528e6, "profiles/r02_ncu_walk_q4_c2_333_z2.txt", 52.35, 42.6),
    ("walk_ql<P16>", "c3_444_zt"): (76.071424e6 + 60.55424e6, "profiles/r02_ncu_walk_ql_c3_444_zt.txt", 51.59, 51.0),
    ("walk_ql<PZ2>", "c3_444_z2"): (49.316096e6 + 51.712768e6, "profiles/r02_ncu_walk_ql_c3_444_z2.txt", 53.40, 53.5),
    ("walk_wl<P32>", "c4_555_zt"): (180.075264e6 + 136.5504e6, "profiles/r02_ncu_walk_wl_c4_555_zt.txt", 72.77, 76.0),
    ("walk_wl<P64>", "c5_4512_zt"): (203.328512e6 + 96.339968e6, "profiles/r02_ncu_walk_wl_c5_4512_zt.txt", 58.76, 68.2),
    ("walk_wl<P64>", "c5_5610_zt"): (245.70112e6 + 132.997376e6, "profiles/r02_ncu_walk_wl_c5_5610_zt.txt", 53.49, 66.2),
    ("walk_wl<P64>", "c5_679_zt"): (310.14528e6 + 180.666624e6, "profiles/r02_ncu_walk_wl_c5_679_zt.txt", 48.21, 61.5),
}


# phase length of the multi-row configs (C3-C5)
PHASE_MULTI = 2000
# LOP3/IADD chain rate measured on the B200 relative to the ALU-pipe model (2.517 vs 2.0
# warp-instructions per clock per SM, profiles/r01_microbench.txt)
MEASURED_INT_RATIO = 2.517 / 2.0


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


# ---------------- time to rank (exact) ----------------
def ladder_from_first(first, phase_ms, S, naive_rank, seeded_rank=None):
    """Time-to-rank from the first step index of a verified strict improvement to each
    rank (fg_rank_first_steps, min over ranks): rank <= t is first held after step
    s* = min_{k <= t} first[k]; its device time is the phases before s*'s phase plus
    the fraction (s* + 1) / S of that phase (uniform progress within a phase).
    Returns {t: (seconds, steps done per walker)} for every reached t < naive_rank."""
    out = {}
    best = None
    top = min(len(first), naive_rank)
    cum = [0.0]
    for ms in phase_ms:
        cum.append(cum[-1] + ms / 1000.0)
    for t in range(top):
        if first[t] < (1 << 63) and (best is None or first[t] < best):
            best = int(first[t])
        if best is None:
            continue
        p = best // S
        if p >= len(phase_ms):
            continue
        if seeded_rank is not None and t >= seeded_rank:
            continue
        out[t] = (cum[p] + (best - p * S + 1) / S * phase_ms[p] / 1000.0, best + 1)
    return out


def roofline_of(g, wl, W, S, walk_ms, launches, total_ms, r_mean, clk):
    per_launch_ms = walk_ms / max(1, launches)
    ops = model_ops_per_step(wl.ring, r_mean) * W * S       # per launch
    achieved = ops / (per_launch_ms / 1000.0) / 1e12
    sm_mhz = clk.get("sm_mhz") or 1965.0
    peak = int_peak_tops(sm_mhz)
    # DRAM bytes per launch from the committed `ncu --set full` capture of this kernel
    # on this workload (dram__bytes_read.sum + dram__bytes_write.sum), if there is one
    traffic = NCU_TRAFFIC.get((g.kernel_name, wl.key))
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
            "frac": achieved / peak, "traffic": traffic[0] if traffic else None,
            "traffic_unit": "B/launch", "traffic_source": traffic[1] if traffic else None,
            "ncu_issue_active_pct": traffic[2] if traffic else None,
            "ncu_alu_pipe_pct": traffic[3] if traffic else None,
            "kernel": g.kernel_name, "kernel_ms_per_launch": per_launch_ms,
            "kernel_share_of_step": walk_ms / total_ms if total_ms else None,
            "ops_per_step_model": model_ops_per_step(wl.ring, r_mean),
            "frac_vs_measured_int_rate": achieved / (peak * MEASURED_INT_RATIO),
            "peak_basis": f"ALU pipe only: 148 SMs x 64 int32 lanes/clk x {sm_mhz:.0f} MHz (median under "
                          f"load); the LOP3/IADD chain measures {MEASURED_INT_RATIO:.3f}x that "
                          "(profiles/r01_microbench.txt: ptxas moves IADDs to the FMA pipe)"}


class Run:
    """One workload on this rank: seed, warm up, time phases (CUDA events on the libfg
    stream), keep the per-phase times for the time-to-rank ladder."""

    def __init__(self, wl, W, S, rank, world, dev, stream, fg, PoolSync):
        self.wl, self.W, self.S, self.world = wl, W, S, world
        self.stream = stream
        self.g = fg.FlipGraph(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, W, rank * W, dev, stream.cuda_stream)
        self.sync = PoolSync(self.g, world)
        self.g.seed_naive()
        self.phase_ms = []

    def phase(self):
        import torch
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(self.stream)
        self.g.walk(self.S, self.wl.seed)
        best = self.sync.exchange()
        ev1.record(self.stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        self.phase_ms.append(ms)
        return ms, best

    def ladder(self, dist=None, dev="cpu"):
        """Exact time-to-rank, box-wide (min over ranks of the first steps; times are
        the max-over-ranks phase times)."""
        import numpy as np
        import torch
        first = self.g.rank_first_steps(self.wl.r_cap).astype(np.float64)
        ms = list(self.phase_ms)
        if self.world > 1 and dist is not None:
            t = torch.tensor(np.minimum(first, 2.0 ** 62), dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            first = t.cpu().numpy()
            tm = torch.tensor(ms, dtype=torch.float64, device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ms = tm.cpu().tolist()
        first_i = [int(x) if x < 2.0 ** 62 else (1 << 64) - 1 for x in first]
        naive = self.wl.m * self.wl.n * self.wl.p
        return ladder_from_first(first_i, ms, self.S, naive, seeded_rank=naive)


def per_config(args, fg, PoolSync, dev, stream, clk_peak_mhz, skip):
    """Every other BASELINE workload on this GPU (rank 0, N = 1): throughput, roofline
    fraction of its kernel, exact time-to-rank ladder over a fixed device-time budget
    and the best (rank, additions) reached."""
    import torch
    from paper_2511_20317_b200.inputs import WORKLOADS
    out = {}
    for key, wl in WORKLOADS.items():
        if key == skip:
            continue
        S = 10000 if wl.r_cap <= 32 else PHASE_MULTI
        run = Run(wl, wl.walkers, S, 0, 1, dev, stream, fg, PoolSync)
        g = run.g
        for _ in range(2):
            run.phase()
        st0 = g.stats()
        r0 = g.get_walkers(rows=False)["r"].mean()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        times = []
        for _ in range(args.per_config_steps):
            flush.zero_()
            times.append(run.phase()[0])
        st1 = g.stats()
        r1 = g.get_walkers(rows=False)["r"].mean()
        # keep walking (untimed for the value) to extend the time-to-rank ladder
        budget = args.per_config_ladder_s * 1000.0
        while sum(run.phase_ms) < budget:
            run.phase()
        total = sum(times)
        value = float(wl.walkers) * S * len(times) / (total / 1000.0)
        walk_ms = (st1["walk_us"] - st0["walk_us"]) / 1000.0
        launches = st1["walk_launches"] - st0["walk_launches"]
        roof = roofline_of(g, wl, wl.walkers, S, walk_ms, launches, total, 0.5 * (r0 + r1),
                           {"sm_mhz": clk_peak_mhz})
        best = g.best()
        lad = run.ladder()
        out[key] = {"workload": wl.name, "walkers": wl.walkers, "phase_steps": S,
                    "value": value, "unit": "flip-steps/s", "ms_per_phase": total / len(times),
                    "kernel": g.kernel_name, "kernel_ms_per_launch": roof["kernel_ms_per_launch"],
                    "frac": roof["frac"], "traffic": roof["traffic"],
                    "ncu_issue_active_pct": roof["ncu_issue_active_pct"],
                    "best": {"rank": best["rank"], "additions": best["additions"]},
                    "ladder_device_s": round(sum(run.phase_ms) / 1000.0, 3),
                    "time_to_rank_s": {str(k): round(v[0], 6) for k, v in sorted(lad.items())},
                    "target_rank": wl.target_rank,
                    "verify_fail": st1["verify_fail"]}
        g.close()
        del flush
        torch.cuda.synchronize()
    return out


# ---------------- our arm ----------------
def main():
    args = parse()
    from paper_2511_20317_b200.inputs import WORKLOADS
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, wl)
        return

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
    rdev = "cuda" if args.dist_backend == "nccl" else "cpu"
    stream = torch.cuda.current_stream()
    W = args.walkers or wl.walkers
    S = args.phase_steps
    run = Run(wl, W, S, rank, world, dev, stream, fg, PoolSync)
    g = run.g
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    for _ in range(args.warmup):
        flush.zero_()
        run.phase()
    st0 = g.stats()
    r_before = g.get_walkers(rows=False)["r"].mean()
    clocks = Clocks(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        flush.zero_()                       # L2 flushed between timed steps (not timed)
        times.append(run.phase()[0])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st1 = g.stats()
    r_after = g.get_walkers(rows=False)["r"].mean()
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    walker_steps = float(W) * S * args.steps * world
    value = walker_steps / (total_ms / 1000.0)

    # dominant kernel (walk) timed live with CUDA events inside libfg, on its stream
    walk_ms = (st1["walk_us"] - st0["walk_us"]) / 1000.0
    launches = st1["walk_launches"] - st0["walk_launches"]
    roofline = roofline_of(g, wl, W, S, walk_ms, launches, total_ms, 0.5 * (r_before + r_after), clk)
    lad = run.ladder(dist if world > 1 else None, rdev)

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
            run.sync.exchange()
            g.save_state(host.data_ptr())
            torch.cuda.synchronize()
            e_times.append(time.perf_counter() - t0)
        te = torch.tensor([sum(e_times)], dtype=torch.float64, device=rdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(W) * S * len(e_times) * world / float(te.item()), "unit": "flip-steps/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_oracle_sample(wl, args.cpu_seconds)
        # the trajectories are identical on the CPU (parity), so the oracle reaches each
        # rank after the same walker-steps: time = steps / its measured rate (extrapolated)
        cpu["time_to_rank_s_extrapolated"] = {str(k): round(v[1] * W * world / cpu["value"], 2)
                                              for k, v in sorted(lad.items())}

    best = g.best()
    stats = {k: st1[k] - st0[k] for k in ("verified", "verify_fail", "queue_overflow")}
    # attempts per step and accepted flips per second (box-wide: summed over ranks)
    cnt = torch.tensor([float(st1[k] - st0[k]) for k in ("steps", "draws", "flips", "expands", "reductions")],
                       dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    c_steps, c_draws, c_flips, c_exp, c_red = (float(x) for x in cnt.tolist())
    walk_stats = {"draws_per_step": c_draws / max(1.0, c_steps),
                  "flips_accepted_per_s": c_flips / (total_ms / 1000.0),
                  "flip_accept_rate": c_flips / max(1.0, c_steps),
                  "expands_per_step": c_exp / max(1.0, c_steps),
                  "reductions_per_step": c_red / max(1.0, c_steps)}
    g.close()
    pc = None
    if rank == 0 and world == 1 and not args.no_per_config:
        pc = per_config(args, fg, PoolSync, dev, stream, clk.get("sm_mhz") or 1965.0, args.workload)
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "flip-steps/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
               "data": "synthetic",
               "config": {"workload": wl.name, "walkers_per_gpu": W, "phase_steps": S,
                          "seed": hex(wl.seed), "l2": "flushed (256 MB write) between timed steps",
                          "kernel": roofline["kernel"],
                          "alg1": "K=16 flip draws, p_eq=0.01, p_reduce=0.5, p_expand=0.01, slack 2 (DESIGN R11, sec. 10)"},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(st1["launches"] - st0["launches"]),
               "clocks": clk,
               "time_to_rank_s": {str(k): round(v[0], 6) for k, v in sorted(lad.items())},
               "time_to_rank_basis": "exact: first step index of a verified strict improvement "
                                     "(fg_rank_first_steps), device time interpolated within its phase",
               "best": {"rank": best["rank"], "additions": best["additions"]},
               "verify": stats, "walk_stats": walk_stats, "per_config": pc}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
