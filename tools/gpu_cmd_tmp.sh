python -m paper_2007_16122_b200.build >/dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or paper_stack or variants or many_small or dense or configs4" > gpurun_out/gpu_tests_s11.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s11.log
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s11a:COLD_CHAIN_GBIAS=0 s11b:COLD_CHAIN_GBIAS=1 s11c:COLD_CHAIN_GBIAS=0 s11d:COLD_CHAIN_GBIAS=1
python tools/show.py gpurun_out/sweep_s11*.log > gpurun_out/sweep_s11.txt 2>&1
