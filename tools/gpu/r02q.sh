set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "paper_stack or variants or one_wide or prelu or chain or configs4 or configs2" > gpurun_out/gpu_tests_r02q.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02q.log
bash tools/gpu/ab_multi.sh tl paper_2007_16122_b200/_ab/prevtail.so
