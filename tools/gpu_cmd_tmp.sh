python -m paper_2007_16122_b200.build >/dev/null
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" bash tools/sweep.sh s26:COLD_TAIL=2 s26d6:COLD_DBG_GEMM=0:6 s26d6d2:COLD_DBG_GEMM=0:6 s26f3d6:COLD_DBG_GEMM=2:6
python tools/show.py gpurun_out/sweep_s26*.log > gpurun_out/sweep_s26.txt 2>&1
