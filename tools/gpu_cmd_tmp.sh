python -m paper_2007_16122_b200.build >/dev/null
COLD_GATHER_ORDER=1 timeout 600 python -m pytest tests -m gpu -x -q -k "gather or paper_stack or bag" > gpurun_out/gpu_tests_s24.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s24.log
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s24o0: s24o1:COLD_GATHER_ORDER=1 s24o0b: s24o1b:COLD_GATHER_ORDER=1
python tools/show.py gpurun_out/sweep_s24*.log > gpurun_out/sweep_s24.txt 2>&1
