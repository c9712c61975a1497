#!/bin/bash
# Walker-count sweep (C2 workload otherwise): value and kernel per population.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for k in ${KERNELS:-q4 w32}; do
  for w in 4096 8192 16384 32768 65536 131072; do
    v=$(FG_WALK_KERNEL=$k timeout 300 python bench.py --walkers $w --steps 3 --warmup 3 --phase-steps ${PHASE:-5000} --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G flip-steps/s  frac %.3f  %s' % (d['value']/1e9, d['roofline']['frac'], d['roofline']['kernel']))")
    echo "kernel=$k walkers=$w  $v" >> gpurun_out/sweep.log
  done
done
