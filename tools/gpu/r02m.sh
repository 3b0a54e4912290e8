set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or paper_stack or variants or one_wide or prelu or many_small or configs4 or host_batch" > gpurun_out/gpu_tests_r02m.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02m.log
bash tools/gpu/ab_multi.sh h1t paper_2007_16122_b200/_ab/h1block.so
