python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/gpu_tests_s21.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s21.log
COLD_USER_FORK=0 timeout 300 python tools/probes/latency_profile.py > gpurun_out/latprof_s21_serial.txt 2>&1
timeout 300 python tools/probes/latency_profile.py > gpurun_out/latprof_s21.txt 2>&1
timeout 900 python bench.py --latency-sweep --latency-requests 3000 > gpurun_out/lat_s21.jsonl 2>&1
