#!/bin/bash
# walk_wl sorted-array bring-up: structure self-check + sampled parity, the wl/wide/fullsize
# GPU tests, then C4/C5 timing at each register budget.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-wlsa}
FG_DBG=1 timeout 900 python scripts/wl_check.py > $O.check.log 2>&1; echo rc=$? >> $O.check.log
FG_DBG=1 FG_WALK_KERNEL=wl timeout 900 python scripts/wl_check.py > $O.check_forced.log 2>&1; echo rc=$? >> $O.check_forced.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "${TESTS_K:-wl or wide or fullsize or multi or state or parity}" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
for mb in ${MINBS:-0}; do
for wl in ${WLS:-c4_555_zt c5_4512_zt c5_5610_zt c5_679_zt}; do
  FG_WL_MINB=$mb timeout 300 python bench.py --workload $wl --phase-steps 2000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-per-config > $O.bench_${wl}_mb$mb.json 2> $O.bench_${wl}_mb$mb.err
done; done
