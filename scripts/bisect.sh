#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/bisect.log
for d in 191 319 575 1087; do
  echo "== dbg=$d" >> gpurun_out/bisect.log
  FG_DBG=$d timeout 30 python scripts/tiny_walk.py 1 >> gpurun_out/bisect.log 2>&1
  echo "rc=$?" >> gpurun_out/bisect.log
done
