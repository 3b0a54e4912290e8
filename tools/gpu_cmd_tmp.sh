python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s37.log 2>&1
BENCH_ARGS="--requests 1 --ads 4000 --no-e2e --no-latency --no-cpu --steps 50 --warmup 5" timeout 900 bash tools/sweep.sh s37L:COLD_TAIL=2
timeout 900 python bench.py --requests 256 --no-e2e --no-cpu --steps 5 > gpurun_out/bench_s37.log 2>&1
python tools/show.py gpurun_out/sweep_s37*.log gpurun_out/bench_s37.log > gpurun_out/sweep_s37.txt 2>&1
