python -m paper_2007_16122_b200.build >/dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "gather or bag or dense or paper_stack" > gpurun_out/gpu_tests_s10.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s10.log
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s10m8:COLD_GATHER_MINB=8 s10m12:COLD_GATHER_MINB=12 s10m16:COLD_GATHER_MINB=16 s10m8b:COLD_GATHER_MINB=8
python tools/show.py gpurun_out/sweep_s10*.log > gpurun_out/sweep_s10.txt 2>&1
