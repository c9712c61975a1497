#!/bin/bash
# walk_q4 chunked tasks: parity (chunk tests, C2 full-size, q4 kernels), then C2 timing with
# the default (8 chunks) vs FG_Q4_CHUNKS=1 (one task per warp) vs other counts, alternated
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-q4c}
timeout 1500 python -m pytest tests -m gpu -q -x -k "${TESTS_K:-q4 or fullsize or c2 or c1 or parity}" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
: > $O.timing.log
for rep in 1 2; do
  for c in ${CHUNKS:-8 1 4 16}; do
    for wl in ${WLS:-c2_333_zt}; do
      out=$(FG_Q4_CHUNKS=$c timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,4), 'G', r['kernel'], round(r['kernel_ms_per_launch'],3), 'ms frac', round(r['frac'],4))")
      echo "rep $rep $wl chunks $c $out" >> $O.timing.log
    done
  done
done
