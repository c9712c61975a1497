#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-minb}
for mb in 16 1 20 24; do
for wl in c4_555_zt c5_4512_zt c5_679_zt; do
  FG_WL_MINB=$mb timeout 300 python bench.py --workload $wl --phase-steps 2000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O.bench_${wl}_mb$mb.json 2> $O.bench_${wl}_mb$mb.err
done; done
