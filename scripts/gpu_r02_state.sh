#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-state}
timeout 1500 python -m pytest tests -m gpu -q -x -k "${TESTS_K:-state or checkpoint or parity or fullsize or explore}" > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
timeout 600 python bench.py --no-per-config --no-cpu-baseline > $O.bench.json 2> $O.bench.err
