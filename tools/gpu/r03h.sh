set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03h.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03h.log
timeout 600 python tools/probes/lat_ab.py 0,4096 4000 3000 > gpurun_out/lat_ab_r03h.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_r03h.csv python tools/probes/lat_ncu.py 4000 3 > gpurun_out/lat_ncu_r03h.log 2>&1; echo ncu rc=$?
