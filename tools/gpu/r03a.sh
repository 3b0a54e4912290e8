set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03a.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03a.log
timeout 600 python bench.py --no-serve > gpurun_out/bench_r03a.jsonl 2> gpurun_out/bench_r03a.err; echo bench rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_r03a.csv python tools/probes/lat_ncu.py 4000 3 > gpurun_out/lat_ncu_r03a.log 2>&1; echo ncu rc=$?
