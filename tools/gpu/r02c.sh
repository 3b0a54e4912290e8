set -x
timeout 1500 python -m pytest tests -m gpu -q -rw > gpurun_out/gpu_tests_r02c.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gpu_tests_r02c.log
timeout 600 python bench.py --no-latency > gpurun_out/bench_r02c.jsonl 2> gpurun_out/bench_r02c.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_r02c.jsonl
