#!/bin/bash
# C5 (4,5,12) from the Strassen meta-operator seed (rank 195): plain walk and with restarts.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/meta_seed_run.py 300 gpurun_out/long_meta_4512.json > gpurun_out/long_meta_4512.log 2>&1
timeout 600 python scripts/meta_seed_run.py 300 gpurun_out/long_meta_4512_restart.json 50 1 > gpurun_out/long_meta_4512_restart.log 2>&1
