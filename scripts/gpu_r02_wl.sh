#!/bin/bash
# walk_wl bring-up: structure self-check, forced on one-word formats, C4/C5 bench wl vs wm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-wl2}
FG_DBG=1 timeout 900 python scripts/wl_check.py > $O.check.log 2>&1; echo rc=$? >> $O.check.log
FG_DBG=1 FG_WALK_KERNEL=wl timeout 600 python scripts/wl_check.py > $O.check_forced.log 2>&1; echo rc=$? >> $O.check_forced.log
for wl in c4_555_zt c5_4512_zt c5_679_zt; do
  for k in wl wm; do
    FG_WALK_KERNEL=$k timeout 300 python bench.py --workload $wl --phase-steps 2000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O.bench_${wl}_$k.json 2> $O.bench_${wl}_$k.err
  done
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "multi or wide or wl_forced or wm_forced or fullsize or state" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
