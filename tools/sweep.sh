#!/bin/bash
# quick perf sweep under gpurun: env-var variants of the library, one bench line each
# usage: bash tools/sweep.sh "<name>:<ENV=..>" ...   (bench args via BENCH_ARGS)
ARGS=${BENCH_ARGS:-"--requests 1024 --no-e2e --no-latency --no-cpu --steps 5"}
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 300 python bench.py $ARGS > gpurun_out/sweep_$name.log 2>&1
done
