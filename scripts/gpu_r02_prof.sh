#!/bin/bash
# ncu --set full of the walk kernel on one workload (after a clean plain run) + stats
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WL=${WL:-c4_555_zt}
NAME=${NAME:-prof_${WL}}
timeout 300 python scripts/walk_stats.py $WL > gpurun_out/$NAME.stats.log 2>&1
B="python bench.py --workload $WL --steps 2 --warmup 1 --phase-steps ${PHASE:-2000} --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/$NAME.plain.json 2>gpurun_out/$NAME.plain.err || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_ -s 1 -c 1 -o gpurun_out/$NAME -f $B > gpurun_out/$NAME.ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$NAME.ncu.log
