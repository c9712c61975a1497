#!/bin/bash
# Every BASELINE config through the full bench contract (CPU baseline included, 5 timed phases).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/all_configs.jsonl
for w in c1_222_zt c2_333_zt c2_333_z2 c3_444_zt c3_444_z2 c4_555_zt c5_4512_zt c5_5610_zt c5_679_zt; do
  ps=10000; [[ $w == c5_* || $w == c4_* ]] && ps=2000
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --phase-steps $ps --cpu-seconds 8 2>/dev/null | grep '^{' >> gpurun_out/all_configs.jsonl
done
