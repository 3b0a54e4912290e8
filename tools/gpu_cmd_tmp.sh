python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/gpu_tests_s7.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s7.log
for i in 1 2; do timeout 600 python bench.py --requests 2048 --no-e2e --no-cpu --no-latency --steps 5 > gpurun_out/bench_s7_$i.jsonl 2>&1; done
