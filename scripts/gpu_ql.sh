#!/bin/bash
# walk_ql bring-up: parity, then C3 throughput ql vs wm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "ql" > gpurun_out/ql.log 2>&1; echo rc=$? >> gpurun_out/ql.log
: > gpurun_out/qlb.log
for k in ql wm; do for w in c3_444_zt c3_444_z2; do
  FG_WALK_KERNEL=$k timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --phase-steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k $w', d['value']/1e6, d['roofline']['kernel'], d['roofline']['frac'])" >> gpurun_out/qlb.log
done; done
