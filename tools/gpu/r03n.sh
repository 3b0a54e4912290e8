set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 120 python -m pytest tests -m gpu -x -q -k "test_paper_stack_tensor_core" > gpurun_out/gpu_tests_r03n_a.log 2>&1; rc=$?; echo quick rc=$rc; tail -5 gpurun_out/gpu_tests_r03n_a.log
if [ $rc -eq 0 ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03n.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03n.log
timeout 300 python tools/probes/lat_ab.py 0,8192 4000 3000 > gpurun_out/lat_ab_r03n.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_r03n.csv python tools/probes/lat_ncu.py 4000 3 > gpurun_out/lat_ncu_r03n.log 2>&1; echo ncu rc=$?
fi
