#!/bin/bash
# Profile the walk kernel once (ncu --set full) after a clean plain run.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --phase-steps ${PHASE:-2000} --no-cpu-baseline --no-e2e ${EXTRA:-}"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-walk_} -s 1 -c 1 -o gpurun_out/${NAME:-prof_walk} -f $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
