python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s32.log 2>&1
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" timeout 900 bash tools/sweep.sh s32:COLD_TAIL=2 s32ch1:COLD_CHAIN=1
python tools/show.py gpurun_out/sweep_s32*.log > gpurun_out/sweep_s32.txt 2>&1
