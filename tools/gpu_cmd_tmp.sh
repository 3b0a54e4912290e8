python -m paper_2007_16122_b200.build >/dev/null
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s8.log 2>&1
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" bash tools/sweep.sh s8:COLD_TAIL=2 s8p2:COLD_PAIR=2 s8p2d2:"COLD_PAIR=2 COLD_DBG_GEMM=0:2" s8d2:"COLD_DBG_GEMM=0:2"
python tools/show.py gpurun_out/sweep_s8*.log > gpurun_out/sweep_s8.txt 2>&1
