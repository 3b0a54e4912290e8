python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s39.log 2>&1
timeout 900 python bench.py --precision f32 --requests 64 --ads 4000 --no-e2e --no-latency --no-cpu --steps 3 > gpurun_out/bench_f32.log 2>&1
python tools/show.py gpurun_out/bench_f32.log > gpurun_out/sweep_s39.txt 2>&1
