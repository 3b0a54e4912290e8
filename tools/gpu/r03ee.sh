set -x
python -m paper_2007_16122_b200.build > /dev/null
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/gpair.so timeout 300 python -m pytest tests -m gpu -x -q -k "gather or sampled or full or configs" > gpurun_out/gpu_tests_r03ee_gpair.log 2>&1; echo gpair tests rc=$?; tail -2 gpurun_out/gpu_tests_r03ee_gpair.log
bash tools/gpu/ab_multi.sh gp paper_2007_16122_b200/_ab/gpair.so
