"""Summarise an ncu report: key throughput / stall / pipe metrics + per-opcode and
per-source-line instruction counts per walker-step.
  python tools/ncu_summary.py <rep> <walker_steps> [cubin kernel-substring]"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__inst_executed.sum", "smsp__warps_active.avg.per_cycle_active",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def main():
    rep, steps = sys.argv[1], float(sys.argv[2])
    v, u = raw(rep)
    for k in KEYS:
        if k in v:
            print(f"{k:60s} {v[k]} {u.get(k, '')}")
    print("-- pipes (% of peak sustained active)")
    for k in sorted(v):
        if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(v[k]) > 0.5:
                    print(f"  {k.split('pipe_')[1].split('.')[0]:12s} {float(v[k]):6.1f}")
            except ValueError:
                pass
    print("-- stalls (cycles per issued instruction)")
    for k in sorted(v):
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio", k)
        if m and float(v[k] or 0) > 0.05:
            print(f"  {m.group(1):22s} {float(v[k]):6.2f}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter()
    tot = 0
    for d in rows[2:]:
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", d[ix["Source"]])
        if not m:
            continue
        e = int(d[ix["Instructions Executed"]] or 0)
        ops[m.group(1)] += e
        tot += e
    print(f"-- {tot / steps:.1f} warp-instructions per walker-step")
    print("  " + "  ".join(f"{o}:{c / steps:.1f}" for o, c in ops.most_common(24)))


if __name__ == "__main__":
    main()
