#!/bin/bash
# Build an A/B variant of libcold.so with extra nvcc defines into paper_2007_16122_b200/_ab/<name>.so
# usage: bash tools/ab_build.sh <name> -DFOO ...   then: COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/<name>.so python bench.py ...
set -e
set -o pipefail
NAME=$1; shift
OUT=paper_2007_16122_b200/_ab/$NAME
mkdir -p $OUT
for f in paper_2007_16122_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I include "$@" -c $f -o $OUT/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o paper_2007_16122_b200/_ab/$NAME.so $OUT/*.o
rm -rf $OUT
echo paper_2007_16122_b200/_ab/$NAME.so
