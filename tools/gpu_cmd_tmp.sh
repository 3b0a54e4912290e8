python -m paper_2007_16122_b200.build >/dev/null
A=COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/oldgroups.so
B=COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/swsmem.so
BENCH_ARGS="--requests 2048 --no-e2e --no-latency --no-cpu --steps 5" timeout 1500 bash tools/sweep.sh s15new1: s15old1:$A s15sw1:$B s15new2: s15old2:$A s15sw2:$B
python tools/show.py gpurun_out/sweep_s15*.log > gpurun_out/sweep_s15.txt 2>&1
