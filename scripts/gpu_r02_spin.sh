#!/bin/bash
# Spin-wait A/B: walk_ql sleep variants on C3 (gpu_r02_ab.sh), then the walk_q4 chunk-count
# sweep with the in-tree build (sleep cap 16384 ns) on C2 Z_T / Z_2.
cd "$(dirname "$0")/.."
NAME=ab_qlspin VARIANTS="qs4096 qs16384" TESTS_K="ql and chunk" WLS="c3_444_zt c3_444_z2" PHASE=2000 STEPS=5 bash scripts/gpu_r02_ab.sh
NAME=q4c_spin CHUNKS="8 16 12" WLS="c2_333_zt c2_333_z2" TESTS_K="chunk or c2" bash scripts/gpu_r02_q4c.sh
