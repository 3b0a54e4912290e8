python -m paper_2007_16122_b200.build >/dev/null
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s21.log 2>&1
COLD_INSTR=1 python tools/probes/epi_instr.py 128 > gpurun_out/epi_instr21.log 2>&1
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" bash tools/sweep.sh s21:COLD_TAIL=2 s21nores:COLD_PAIR_RES=0 s21d1:COLD_DBG_GEMM=0:1 s21d2:COLD_DBG_GEMM=0:2
python tools/show.py gpurun_out/sweep_s21*.log > gpurun_out/sweep_s21.txt 2>&1
