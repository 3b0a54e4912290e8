set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multi_rank_gpu.py -q -x -k "chain or paper_stack or variants or one_wide or prelu or configs4 or configs2 or many_small or host_batch or bench_rank or server" > gpurun_out/gpu_tests_r02u.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02u.log
bash tools/gpu/ab_multi.sh fc3 paper_2007_16122_b200/_ab/fc3last.so
