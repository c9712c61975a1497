#!/bin/bash
# Round-2 A/B: for each variant library build/ab/libfg_<v>.so in $VARIANTS, a parity
# check (wl_check structure self-check + sampled oracle parity, and the -k "$TESTS_K"
# GPU tests), then same-box timing alternated with the in-tree library on $WLS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-ab}
for v in $VARIANTS; do
  FG_LIBFG=build/ab/libfg_$v.so FG_DBG=1 timeout 900 python scripts/wl_check.py > $O.check_$v.log 2>&1; echo rc=$? >> $O.check_$v.log
  if [ -n "$TESTS_K" ]; then
    FG_LIBFG=build/ab/libfg_$v.so timeout 1200 python -m pytest tests -m gpu -q -x -k "$TESTS_K" > $O.tests_$v.log 2>&1; echo "tests rc=$?" >> $O.tests_$v.log
  fi
done
: > $O.timing.log
for rep in 1 2; do
  for w in $WLS; do
    for v in base $VARIANTS; do
      lib=""; [ $v != base ] && lib=build/ab/libfg_$v.so
      out=$(FG_LIBFG=$lib timeout 300 python bench.py --workload $w --steps ${STEPS:-3} --warmup 3 --phase-steps ${PHASE:-2000} --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e6,1), 'M', r['kernel'], round(r['kernel_ms_per_launch'],3), 'ms frac', round(r['frac'],4))")
      echo "rep $rep $w $v $out" >> $O.timing.log
    done
  done
done
