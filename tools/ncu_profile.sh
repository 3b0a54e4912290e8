#!/bin/bash
# Run under gpurun: launch list + one `--set full` capture of the FC2 GEMM and of the gather kernel.
# Usage: bash tools/ncu_profile.sh <tag>
set -x
TAG=${1:-r01}
OUT=gpurun_out
ARGS="--requests 32 --ads 10000 --steps 2 --warmup 1 --no-e2e --no-latency --no-cpu"
python -m paper_2007_16122_b200.build >/dev/null
# 1. launch list (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py $ARGS > $OUT/ncu_launch_bench_$TAG.log 2>&1
# 2. full capture of FC2 (the 2nd gemm launch of a chunk) and of the gather kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 13 -c 1 \
  -o $OUT/prof_fc2_$TAG python bench.py $ARGS > $OUT/ncu_fc2_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 3 -c 1 \
  -o $OUT/prof_gather_$TAG python bench.py $ARGS > $OUT/ncu_gather_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 1 \
  -o $OUT/prof_fc1_$TAG python bench.py $ARGS > $OUT/ncu_fc1_$TAG.log 2>&1
ls -la $OUT
