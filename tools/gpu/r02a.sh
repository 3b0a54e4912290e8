set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r02a.log 2>&1; echo tests rc=$?
timeout 600 python bench.py > gpurun_out/bench_r02a.jsonl 2> gpurun_out/bench_r02a.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_r02a.jsonl
