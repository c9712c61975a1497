#!/bin/bash
# Build an alternative libfg (build/ab/libfg_<tag>.so, delete after use) in which one
# translation unit is replaced by another source file, for same-box A/B timing:
#   scripts/ab_build.sh <tag> <unit.cu basename> <replacement source>
set -e
cd "$(dirname "$0")/.."
tag=$1; unit=$2; src=$3
objs=$(ls build/libfg/*.o | grep -v "/$unit.o")
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O2 -I include \
     -I paper_2511_20317_b200/csrc -I build/ab -x cu -c "$src" -o /tmp/ab_$tag.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/ab/libfg_$tag.so $objs /tmp/ab_$tag.o
echo build/ab/libfg_$tag.so
