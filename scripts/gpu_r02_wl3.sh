#!/bin/bash
# walk_wl iteration: structure self-check + parity, bench C3-C5 (C3 forced wl too)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-wl3}
FG_DBG=1 timeout 900 python scripts/wl_check.py > $O.check.log 2>&1; echo rc=$? >> $O.check.log
for wl in c4_555_zt c5_4512_zt c5_5610_zt c5_679_zt; do
  timeout 300 python bench.py --workload $wl --phase-steps 2000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O.bench_${wl}.json 2> $O.bench_${wl}.err
done
for wl in c3_444_zt c3_444_z2; do
  FG_WALK_KERNEL=wl timeout 300 python bench.py --workload $wl --phase-steps 2000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O.bench_${wl}_wl.json 2> $O.bench_${wl}_wl.err
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "${TESTS_K:-multi or wide or wl_forced or fullsize or state}" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
