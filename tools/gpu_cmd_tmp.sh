python -m paper_2007_16122_b200.build >/dev/null
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s22a4: s22a2:COLD_GATHER_APT=2 s22g32:COLD_GSPAN=32 s22a4b: s22a2b:COLD_GATHER_APT=2 s22g32b:COLD_GSPAN=32
python tools/show.py gpurun_out/sweep_s22*.log > gpurun_out/sweep_s22.txt 2>&1
