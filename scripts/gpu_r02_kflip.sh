#!/bin/bash
# K > 16 flip draws (R11): parity of every kernel family at K = 64, then long walks from naive
# with K = 64 on the C5 formats (with K = 16 the (4,5,12) walk sits at the row capacity: ~80 %
# of draws overflow, 3.6 % of steps fail all 16 draws and expand) and on C4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "large_flip_budget or kernel_c1 or kernel_c2" > gpurun_out/kflip.tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/kflip.tests.log
T=${T:-400}
timeout $((T+200)) python scripts/long_run.py c5_4512_zt $T gpurun_out/long_k64_c5_4512.json 0 2 64 > gpurun_out/long_k64_c5_4512.log 2>&1
timeout $((T+200)) python scripts/long_run.py c5_679_zt $T gpurun_out/long_k64_c5_679.json 0 2 64 > gpurun_out/long_k64_c5_679.log 2>&1
timeout $((T+200)) python scripts/long_run.py c4_555_zt $T gpurun_out/long_k64_c4_555.json 0 2 64 > gpurun_out/long_k64_c4_555.log 2>&1
