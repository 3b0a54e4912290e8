python -m paper_2007_16122_b200.build >/dev/null
timeout 600 python -m pytest tests -m gpu -q -k "dense" > gpurun_out/gpu_tests_s6.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s6.log
timeout 600 python bench.py --requests 2048 --no-e2e --no-cpu --no-latency --steps 5 --se-dense > gpurun_out/bench_dense_s6.jsonl 2>&1
