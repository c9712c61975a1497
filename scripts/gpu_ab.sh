#!/bin/bash
# Same-box A/B: bench.py with libfg.so vs build/ab/libfg_<b>.so for each b
# in $B, alternating, twice.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab.log
for rep in 1 2; do
  for b in base $B; do
    lib=""; [ "$b" != base ] && lib="build/ab/libfg_${b}.so"
    v=$(FG_LIBFG=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['kernel'])")
    echo "rep $rep $b $v" >> gpurun_out/ab.log
  done
done
