python -m paper_2007_16122_b200.build >/dev/null
AB=COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/llbranchy.so
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s13new1: s13old1:$AB s13new2: s13old2:$AB
python tools/show.py gpurun_out/sweep_s13*.log > gpurun_out/sweep_s13.txt 2>&1
