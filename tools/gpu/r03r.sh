set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 120 python -m pytest tests -m gpu -x -q -k "test_paper_stack_tensor_core" > gpurun_out/gpu_tests_r03r_a.log 2>&1; rc=$?; echo quick rc=$rc; tail -3 gpurun_out/gpu_tests_r03r_a.log
if [ $rc -eq 0 ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03r.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03r.log
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 > gpurun_out/lat_ab_r03r.jsonl 2>&1
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 >> gpurun_out/lat_ab_r03r.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/lat_launches_warm_r03r.csv python tools/probes/lat_ncu.py 4000 8 > /dev/null 2>&1; echo latncuw rc=$?
fi
