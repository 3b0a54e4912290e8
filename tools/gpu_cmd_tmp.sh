python -m paper_2007_16122_b200.build >/dev/null
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" timeout 900 bash tools/sweep.sh s40a4:COLD_GATHER_APT=4 s40a2:COLD_GATHER_APT=2 s40a1:COLD_GATHER_APT=1 s40m4:COLD_GATHER_MINB=4
python tools/show.py gpurun_out/sweep_s40*.log > gpurun_out/sweep_s40.txt 2>&1
