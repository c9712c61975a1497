#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-z2chk}
timeout 600 python -m pytest tests/test_pool_sync_nccl.py -q > $O.nccl.log 2>&1; echo "rc=$?" >> $O.nccl.log
: > $O.timing.log
for rep in 1 2; do
  for c in 8 1; do
    for st in "4 2" "10 3"; do
      set -- $st
      out=$(FG_Q4_CHUNKS=$c timeout 300 python bench.py --workload c2_333_z2 --steps $1 --warmup $2 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,4), 'G', round(r['kernel_ms_per_launch'],3), 'ms')")
      echo "rep $rep chunks $c steps/warm $st $out" >> $O.timing.log
    done
  done
done
