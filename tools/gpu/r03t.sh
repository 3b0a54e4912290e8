set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03t.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests_r03t.log
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/fc2d.so timeout 300 python -m pytest tests -m gpu -x -q -k "chain or paper_stack" > gpurun_out/gpu_tests_r03t_fc2d.log 2>&1; echo fc2d tests rc=$?; tail -2 gpurun_out/gpu_tests_r03t_fc2d.log
bash tools/gpu/ab_multi.sh fc2d paper_2007_16122_b200/_ab/fc2d.so
