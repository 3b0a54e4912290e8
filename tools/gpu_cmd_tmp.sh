python -m paper_2007_16122_b200.build >/dev/null
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s23m8: s23m7:COLD_GATHER_MINB=7 s23m6:COLD_GATHER_MINB=6 s23m8b: s23m7b:COLD_GATHER_MINB=7 s23m6b:COLD_GATHER_MINB=6
python tools/show.py gpurun_out/sweep_s23*.log > gpurun_out/sweep_s23.txt 2>&1
