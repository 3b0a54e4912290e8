set -x
python -m paper_2007_16122_b200.build > /dev/null
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/direct.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or paper_stack or variants or one_wide or prelu or configs4" > gpurun_out/gpu_tests_r02t.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02t.log
bash tools/gpu/ab_multi.sh dir paper_2007_16122_b200/_ab/direct.so
