#!/bin/bash
# Multi-row configs (C3-C5): throughput with 2000-step phases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/multi.log
for w in c3_444_zt c3_444_z2 c4_555_zt c5_4512_zt c5_5610_zt c5_679_zt; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --phase-steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w %.1f M walker-steps/s %s kernel ms/launch %.1f frac %.3f walkers %d' % (d['value']/1e6, r['kernel'], r['kernel_ms_per_launch'], r['frac'], d['config']['walkers_per_gpu']))" >> gpurun_out/multi.log
done
