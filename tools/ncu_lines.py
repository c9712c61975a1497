"""Per-CUDA-source-line instruction counts and stall-sample shares from an ncu report
(needs -lineinfo and --import-source on):  python tools/ncu_lines.py <rep> <walker_steps> [top_n]"""
import csv, io, subprocess, sys
rep, steps = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
f = None; res = []
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": f = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = {h: i for i, h in enumerate(row)}; continue
    if hdr is None or row[0] == "Function Name": continue
    if row[2] != "-": continue
    try:
        e = int(row[hdr["Instructions Executed"]] or 0); smp = int(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    if e: res.append((e, smp, f, row[0], row[1].strip()[:110]))
tot = sum(r[0] for r in res); ts = sum(r[1] for r in res)
print(f"total {tot/steps:.1f} warp-inst/walker-step, samples {ts}")
for e, smp, f, ln, src in sorted(res, reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 60]:
    print(f"{e/steps:7.1f} {100*smp/ts:5.1f}% {f}:{ln}  {src}")
