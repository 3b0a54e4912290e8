set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03l.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03l.log
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 > gpurun_out/lat_ab_r03l.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_r03l.csv python tools/probes/lat_ncu.py 4000 3 > gpurun_out/lat_ncu_r03l.log 2>&1; echo ncu rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:topk_small -c 1 -o gpurun_out/prof_topk_r03l python tools/probes/lat_ncu.py 4000 2 > gpurun_out/prof_topk_r03l.log 2>&1; echo ncu2 rc=$?
