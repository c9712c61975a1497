#!/bin/bash
# Round-2 measurement pass: GPU suite, default bench (headline + per_config), the ncu
# launch list of the same command, then one `ncu --set full` capture per shipped walk
# kernel (C2 walk_q4, C3 walk_ql, C4 walk_wl P32, C5 (6,7,9) walk_wl P64), each after
# its own plain run exited 0.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-r02m}
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TMO:-2400} python -m pytest tests -m gpu -q ${TESTS_K:+-k "$TESTS_K"} > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
fi
timeout 900 python bench.py > $O.bench.json 2> $O.bench.err; echo "bench rc=$?" >> $O.bench.err
if [ -z "$SKIP_LAUNCH" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O.launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > $O.ncu_launch.log 2>&1; echo "ncu rc=$?" >> $O.ncu_launch.log
fi
for spec in ${PROF:-c2_333_zt:10000 c3_444_zt:2000 c4_555_zt:2000 c5_679_zt:2000}; do
  wl=${spec%%:*}; ph=${spec##*:}
  B="python bench.py --workload $wl --steps 2 --warmup 1 --phase-steps $ph --no-cpu-baseline --no-e2e --no-per-config"
  timeout 300 $B > $O.plain_$wl.json 2> $O.plain_$wl.err || continue
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_ -s 1 -c 1 \
    -o $O.full_$wl -f $B > $O.ncu_$wl.log 2>&1; echo "ncu rc=$?" >> $O.ncu_$wl.log
  # summary on the box (walker-steps per launch from the plain run's config); the report
  # itself comes back only with KEEP_REPS (gpurun_out returns at most 64 MiB)
  ws=$(python -c "import json; d=json.loads(open('$O.plain_$wl.json').read().strip().splitlines()[-1]); print(d['config']['walkers_per_gpu']*d['config']['phase_steps'])")
  python tools/ncu_summary.py $O.full_$wl.ncu-rep $ws > $O.sum_$wl.txt 2>&1
  [ -z "$KEEP_REPS" ] && rm -f $O.full_$wl.ncu-rep
done
