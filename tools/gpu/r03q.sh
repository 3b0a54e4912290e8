set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 300 python -m pytest tests -m gpu -x -q -k "topk or merge or split or serve" > gpurun_out/gpu_tests_r03q.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03q.log
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/topkt.so timeout 120 python tools/probes/lat_ncu.py 4000 4 > gpurun_out/topk_timing_r03q.txt 2>&1
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 > gpurun_out/lat_ab_r03q.jsonl 2>&1
