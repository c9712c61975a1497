#!/bin/bash
# t1 bring-up on the GPU box: smoke, parity tests, bench t1 vs w32.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS_K:+-k "$TESTS_K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_new.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_new.log
FG_WALK_KERNEL=${CMP:-t1} timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cmp.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cmp.log
