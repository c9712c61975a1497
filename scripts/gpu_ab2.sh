#!/bin/bash
# Same-box A/B on one workload per alternative library: pairs "lib:workload" in $PAIRS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab2.log
for rep in 1 2; do
  for pw in $PAIRS; do
    b=${pw%%:*}; w=${pw##*:}
    for lib in "" "build/ab/libfg_${b}.so"; do
      v=$(FG_LIBFG=$lib timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --phase-steps ${PHASE:-2000} --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['kernel'])")
      echo "rep $rep $w ${lib:-base} $v" >> gpurun_out/ab2.log
    done
  done
done
