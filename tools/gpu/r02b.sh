set -x
timeout 1200 python -m pytest tests -m gpu -x -q -rw > gpurun_out/gpu_tests_r02b.log 2>&1; echo tests rc=$?
timeout 600 python bench.py > gpurun_out/bench_r02b.jsonl 2> gpurun_out/bench_r02b.err; echo bench rc=$?
GIT_SHA=$GIT_SHA bash tools/ncu_profile.sh r02b > gpurun_out/ncu_profile_r02b.log 2>&1; echo ncu rc=$?
tail -c 1500 gpurun_out/bench_r02b.jsonl
