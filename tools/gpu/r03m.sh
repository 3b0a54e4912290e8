set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "gather or bags or paper or variant or small or chunking" > gpurun_out/gpu_tests_r03m.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03m.log
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 > gpurun_out/lat_ab_r03m.jsonl 2>&1
timeout 600 python tools/probes/lat_ab.py 0 4000 3000 >> gpurun_out/lat_ab_r03m.jsonl 2>&1
