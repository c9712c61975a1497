#!/bin/bash
# Final round-2 validation: the R24 parity tests first (new walk_wl instance), the full GPU
# suite, a bounded long fuzz (all kernels, a fifth of the runs in R24), and the default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${NAME:-r02f}
timeout 900 python -m pytest tests -m gpu -q -k "complexity" > $O.cm.log 2>&1; echo "cm rc=$?" >> $O.cm.log
timeout 2400 python -m pytest tests -m gpu -q > $O.tests.log 2>&1; echo "tests rc=$?" >> $O.tests.log
timeout 700 python scripts/fuzz_long.py ${FUZZ_N:-30} ${FUZZ_SEED:-4242} ${FUZZ_S:-500} > $O.fuzz.log 2>&1; echo "fuzz rc=$?" >> $O.fuzz.log
timeout 900 python bench.py > $O.bench.json 2> $O.bench.err; echo "bench rc=$?" >> $O.bench.err
