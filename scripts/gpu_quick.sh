#!/bin/bash
# quick check: smoke + parity subset + bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTS_K:-c1 or c2 or edge or split or multi or restart}" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_new.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_new.log
