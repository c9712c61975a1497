#!/bin/bash
# One ncu --set full capture of walk_q4 at C2 Z_T (report returned for per-line analysis).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --workload c2_333_zt --steps 2 --warmup 1 --phase-steps 10000 --no-cpu-baseline --no-e2e --no-per-config"
$B > gpurun_out/c2p.plain.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_ -s 1 -c 1 -o gpurun_out/c2p -f $B > gpurun_out/c2p.ncu.log 2>&1
