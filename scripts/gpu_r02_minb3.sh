#!/bin/bash
# walk_wl register budget per layout: C5 workloads at FG_WL_MINB in $MBS (0 = default)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/minb3.log
for rep in 1 2; do for w in ${WLS:-c5_4512_zt c5_5610_zt c5_679_zt}; do for mb in ${MBS:-0 14 11}; do
  out=$(FG_WL_MINB=$mb timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --phase-steps 2000 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e6,1), 'M', round(r['kernel_ms_per_launch'],3), 'ms')")
  echo "rep $rep $w minb $mb $out" >> gpurun_out/minb3.log
done; done; done
