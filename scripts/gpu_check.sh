#!/bin/bash
# Run on the GPU box (via gpurun): GPU tests, smoke, short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS_K:+-k "$TESTS_K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3 --cpu-seconds 8} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
