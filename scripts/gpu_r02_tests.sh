#!/bin/bash
# round 2: full GPU suite (or a -k subset) into gpurun_out/$NAME.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NAME=${NAME:-r02_tests}
timeout ${TMO:-2400} python -m pytest tests -m gpu -q ${TESTS_K:+-k "$TESTS_K"} ${PYTEST_ARGS:-} > gpurun_out/$NAME.log 2>&1; echo "tests rc=$?" >> gpurun_out/$NAME.log
