python -m paper_2007_16122_b200.build >/dev/null
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s10.log 2>&1
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" bash tools/sweep.sh s10:COLD_GATHER_MINB=4 s10m8:COLD_GATHER_MINB=8 s10s8m8:"COLD_GATHER_MINB=8 COLD_GSPAN=8"
python tools/show.py gpurun_out/sweep_s10*.log > gpurun_out/sweep_s10.txt 2>&1
timeout 900 python bench.py --se-sweep --steps 5 --warmup 3 > gpurun_out/se_sweep.log 2>&1
