python -m paper_2007_16122_b200.build >/dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "host_batch" > gpurun_out/gpu_tests_s26.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s26.log
