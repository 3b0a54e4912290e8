set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 300 python -m pytest tests -m gpu -x -q -k "chain or paper_stack or variant or prelu or small" > gpurun_out/gpu_tests_r03cc.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests_r03cc.log
bash tools/gpu/ab_multi.sh t45 paper_2007_16122_b200/_ab/t45smem.so
