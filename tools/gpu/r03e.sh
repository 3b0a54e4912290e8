set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 300 python -m pytest tests -m gpu -x -q -k "topk or merge or split or serve" > gpurun_out/gpu_tests_r03e.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03e.log
timeout 600 python tools/probes/lat_ab.py 0,68 4000 3000 > gpurun_out/lat_ab_r03e.jsonl 2>&1
timeout 600 python bench.py --no-serve --no-e2e --no-cpu --steps 5 > gpurun_out/bench_r03e.jsonl 2> gpurun_out/bench_r03e.err; echo bench rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:topk_small -c 1 -o gpurun_out/prof_topk_r03e python tools/probes/lat_ncu.py 4000 2 > gpurun_out/prof_topk_r03e.log 2>&1; echo ncu rc=$?
