#!/bin/bash
# walk_q4 chunked tasks: number of spare (waiting) warps beyond one per walker group, C2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/spare
timeout 600 python -m pytest tests -m gpu -q -x -k "chunk" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
: > $O.timing.log
for rep in 1 2; do
  for sp in all 32 96 192; do
    for wl in c2_333_zt c2_333_z2; do
      if [ $sp = all ]; then unset FG_Q4_SPARE; else export FG_Q4_SPARE=$sp; fi
      out=$(timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,4), 'G', round(r['kernel_ms_per_launch'],3), 'ms frac', round(r['frac'],4))")
      echo "rep $rep $wl spare $sp $out" >> $O.timing.log
    done
  done
done
unset FG_Q4_SPARE
